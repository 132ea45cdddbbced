"""Cubed-sphere halo update: tile connectivity, edge rotation, corner fill.

The paper runs FV3 on the six tiles of a cubed sphere, one tile per GPU, and
refreshes halos with a Python halo updater that packs edge strips, rotates
them between tiles whose index frames differ by 90 degrees and fills the
halo corners at the cube vertices (SURVEY 8a A21, config
C3).  No implementation of it exists in the reference, so this module is the
specification; ``oracle/cube.py`` applies it with NumPy (the CPU oracle) and
:class:`CubeHalo` with the gather / scatter CUDA kernels
(``fv3b_halo_gather`` / ``fv3b_halo_scatter``).

Connectivity (FV3 tile numbering T = 1..6, mpp cubic-grid layout):

    odd T:  W <- T-2 (rotated, its north edge)   E <- T+1   S <- T-1   N <- T+2 (rotated, its west edge)
    even T: W <- T-1   E <- T+2 (rotated, its south edge)   S <- T-2 (rotated, its east edge)   N <- T+1

Cell (i, j) of an n x n tile is centred at (i, j); a halo cell maps to the
neighbour's interior through one of these affine maps (X, Y) -> (X', Y'):

    plain W/E/S/N     X' = X +/- n  or  Y' = Y +/- n
    odd N, even S     X' = Y - n,     Y' = n - 1 - X      (resp. X' = Y + n)
    odd W, even E     X' = n - 1 - Y, Y' = X + n          (resp. Y' = X - n)

Vector fields are (x, y) component pairs; on a rotated edge the components
are re-expressed in the neighbour's frame (a 90-degree rotation: the
received x component is +/- the neighbour's y component and vice versa).
Staggered components are mapped at their own positions: D-grid (u on south
edges, v on west edges) and C-grid pairs (uc / cx / xfa / mfx on west
edges, vc / cy / yfa / mfy on south edges) land on the neighbour's west /
south edges, which can shift the source index by one along the edge; a
source that falls on the neighbour's outer boundary line (the cube-vertex
line) is clamped to the nearest interior edge.

Corner halo cells (beyond both edges of a tile corner, where three tiles
meet at a cube vertex) are filled after the edge exchange by the FV3
``fill_corners`` X-direction rule, rotating the tile's own west / east halo
strip into the corner (vector components rotated with it):

    SW (-1-a, -1-b) <- (-1-b, a)      SE (n+a, -1-b) <- (n+b, a)
    NE (n+a, n+b)   <- (n+b, n-1-a)   NW (-1-a, n+b) <- (-1-b, n-1-a)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# x / y component pairs among the dycore state (D-grid, C-grid, face fluxes)
VECTOR_PAIRS = {"u": ("v", "D"), "uc": ("vc", "C"), "cx": ("cy", "C"), "xfa": ("yfa", "C"), "mfx": ("mfy", "C")}
_ROLE = {}
for _x, (_y, _g) in VECTOR_PAIRS.items():
    _ROLE[_x] = ("x", _y, _g)
    _ROLE[_y] = ("y", _x, _g)


def role(name: str):
    """('s', None, None) for scalars, ('x'|'y', partner, 'D'|'C') for vector components."""
    return _ROLE.get(name, ("s", None, None))


def _fv3(t: int) -> int:
    return (t - 1) % 6 + 1


@dataclass(frozen=True)
class Side:
    nb: int          # neighbour tile (0-based)
    rot: str         # "plain" | "N" (odd-N / even-S type) | "W" (odd-W / even-E type)


def topology() -> list[dict[str, Side]]:
    """Per tile (0-based), the neighbour and map type of each side."""
    out = []
    for t0 in range(6):
        T = t0 + 1
        if T % 2:
            sides = {"W": Side(_fv3(T - 2) - 1, "W"), "E": Side(_fv3(T + 1) - 1, "plain"),
                     "S": Side(_fv3(T - 1) - 1, "plain"), "N": Side(_fv3(T + 2) - 1, "N")}
        else:
            sides = {"W": Side(_fv3(T - 1) - 1, "plain"), "E": Side(_fv3(T + 2) - 1, "W"),
                     "S": Side(_fv3(T - 2) - 1, "N"), "N": Side(_fv3(T + 1) - 1, "plain")}
        out.append(sides)
    return out


def _point_map(side: str, kind: str, n: int):
    """(X, Y) -> (X', Y') and the Jacobian sign rule (ux, uy) = f(ux', uy')."""
    if kind == "plain":
        d = {"W": (n, 0), "E": (-n, 0), "S": (0, n), "N": (0, -n)}[side]
        return (lambda X, Y: (X + d[0], Y + d[1])), (lambda ux, uy: (ux, uy))
    if kind == "N":  # odd-N (X' = Y - n) or even-S (X' = Y + n); Y' = n - 1 - X
        off = -n if side == "N" else n
        return (lambda X, Y: (Y + off, n - 1 - X)), (lambda ux, uy: (-uy, ux))  # ux = -uy', uy = ux'
    # "W": odd-W (Y' = X + n) or even-E (Y' = X - n); X' = n - 1 - Y
    off = n if side == "W" else -n
    return (lambda X, Y: (n - 1 - Y, X + off)), (lambda ux, uy: (uy, -ux))  # ux = uy', uy = -ux'


def _edge_cells(side: str, n: int, h: int):
    """Halo cells of one side strip (interior span along the edge)."""
    if side in ("W", "E"):
        ii = range(-h, 0) if side == "W" else range(n, n + h)
        return [(i, j) for j in range(n) for i in ii]
    jj = range(-h, 0) if side == "S" else range(n, n + h)
    return [(i, j) for j in jj for i in range(n)]


def _stagger(pos: str):
    """Offset of a component's position from its cell centre."""
    return {"c": (0.0, 0.0), "S": (0.0, -0.5), "W": (-0.5, 0.0)}[pos]


def _position(name: str) -> str:
    r, _, g = role(name)
    if r == "s":
        return "c"
    if g == "D":
        return "S" if r == "x" else "W"  # u on south edges, v on west edges
    return "W" if r == "x" else "S"      # uc on west edges, vc on south edges


def _cell_of(Xp: float, Yp: float, pos_nb: str):
    """Neighbour cell whose `pos_nb` point is (Xp, Yp)."""
    dx, dy = _stagger(pos_nb)
    return int(round(Xp - dx)), int(round(Yp - dy))


@dataclass(frozen=True)
class Entry:
    """dst[name][i, j] = sign * src_tile[src_name][si, sj]"""

    name: str
    i: int
    j: int
    src_tile: int
    src_name: str
    si: int
    sj: int
    sign: float


def edge_entries(tile: int, names, n: int, h: int) -> list[Entry]:
    """Every edge-halo cell of `tile` for the fields `names`."""
    topo = topology()[tile]
    out = []
    clamp = lambda v: min(max(v, 0), n - 1)
    for side in ("W", "E", "S", "N"):
        sd = topo[side]
        pmap, vrule = _point_map(side, sd.rot, n)
        for name in names:
            r, partner, _ = role(name)
            pos = _position(name)
            for (i, j) in _edge_cells(side, n, h):
                dx, dy = _stagger(pos)
                Xp, Yp = pmap(i + dx, j + dy)
                if r == "s" or sd.rot == "plain":
                    src_name, sign = name, 1.0
                    pos_nb = pos
                else:
                    # which neighbour component feeds this one, and its sign:
                    # evaluate the rule on (ux', uy') = (1, 2)
                    cx, cy = vrule(1.0, 2.0)
                    mine = cx if r == "x" else cy
                    comp = "x" if abs(mine) == 1.0 else "y"
                    sign = 1.0 if mine > 0 else -1.0
                    src_name = name if comp == r else partner
                    pos_nb = _position(src_name)
                si, sj = _cell_of(Xp, Yp, pos_nb)
                out.append(Entry(name, i, j, sd.nb, src_name, clamp(si), clamp(sj), sign))
    return out


def corner_entries(names, n: int, h: int) -> list[Entry]:
    """Corner-halo cells filled from the tile's own edge halos (src_tile = -1
    means the same tile)."""
    out = []
    # (target(a, b), source(a, b), rule) ; rule maps (ux', uy') -> (ux, uy)
    rot_a = lambda ux, uy: (-uy, ux)  # SW, NE
    rot_b = lambda ux, uy: (uy, -ux)  # SE, NW
    corners = [
        (lambda a, b: (-1 - a, -1 - b), lambda a, b: (-1 - b, a), rot_a),
        (lambda a, b: (n + a, -1 - b), lambda a, b: (n + b, a), rot_b),
        (lambda a, b: (n + a, n + b), lambda a, b: (n + b, n - 1 - a), rot_a),
        (lambda a, b: (-1 - a, n + b), lambda a, b: (-1 - b, n - 1 - a), rot_b),
    ]
    for tgt, src, rule in corners:
        cx, cy = rule(1.0, 2.0)
        for name in names:
            r, partner, _ = role(name)
            for a in range(h):
                for b in range(h):
                    i, j = tgt(a, b)
                    si, sj = src(a, b)
                    if r == "s":
                        out.append(Entry(name, i, j, -1, name, si, sj, 1.0))
                    else:
                        mine = cx if r == "x" else cy
                        comp = "x" if abs(mine) == 1.0 else "y"
                        out.append(Entry(name, i, j, -1, name if comp == r else partner, si, sj,
                                         1.0 if mine > 0 else -1.0))
    return out


def check_names(names) -> None:
    for nme in names:
        r, partner, _ = role(nme)
        if r != "s" and partner not in names:
            raise ValueError(f"vector component {nme!r} exchanged without its partner {partner!r}")


# ---------------------------------------------------------------------------
# device halo object (one tile per rank)
# ---------------------------------------------------------------------------

class CubeHalo:
    """Cubed-sphere halo update of one tile; ``update(names)`` refreshes the
    halos of the named state fields of ``dycore`` (a Dycore on this tile).

    Per update: one gather launch per neighbour (message in the receiver's
    entry order), the exchange (``parallel.DistTransport`` over NCCL, or a
    loopback), one scatter launch per neighbour (rotation / component swap /
    sign applied on receipt), then the corner fill as a local gather +
    scatter.  Index lists are built once per field list and kept on device.
    """

    def __init__(self, dycore, tile: int, transport=None):
        from .parallel import DistTransport

        self.d = dycore
        self.tile = tile
        g = dycore.grid
        if g.ni != g.nj:
            raise ValueError("cubed-sphere tiles are square")
        self.n, self.h = g.ni, g.halo
        self.transport = transport or DistTransport(tile)
        self.peers = sorted({s.nb for s in topology()[tile].values()})
        self._plans: dict = {}

    def _off(self, i: int, j: int) -> int:
        return i + j * self.d.grid.pitch

    def _plan(self, names: tuple):
        if names in self._plans:
            return self._plans[names]
        import torch

        check_names(names)
        if len(names) > 32:
            raise ValueError("at most 32 fields per cubed-sphere halo update")
        slot = {n: k for k, n in enumerate(names)}
        dev = self.d.cur[names[0]].device
        mine = edge_entries(self.tile, names, self.n, self.h)
        send, recv = {}, {}
        for p in self.peers:
            theirs = [e for e in edge_entries(p, names, self.n, self.h) if e.src_tile == self.tile]
            send[p] = torch.tensor([[slot[e.src_name], self._off(e.si, e.sj)] for e in theirs],
                                   dtype=torch.int32, device=dev).reshape(-1)
            rec = [e for e in mine if e.src_tile == p]
            recv[p] = torch.tensor([[slot[e.name], self._off(e.i, e.j), 1 if e.sign > 0 else -1] for e in rec],
                                   dtype=torch.int32, device=dev).reshape(-1)
        cor = corner_entries(names, self.n, self.h)
        cg = torch.tensor([[slot[e.src_name], self._off(e.si, e.sj)] for e in cor], dtype=torch.int32,
                          device=dev).reshape(-1)
        cs = torch.tensor([[slot[e.name], self._off(e.i, e.j), 1 if e.sign > 0 else -1] for e in cor],
                          dtype=torch.int32, device=dev).reshape(-1)
        L = self.d.cur[names[0]].shape[0]
        nsend = {p: send[p].numel() // 2 for p in self.peers}
        nrecv = {p: recv[p].numel() // 3 for p in self.peers}
        sbuf = {p: torch.empty(nsend[p] * L, dtype=torch.float64, device=dev) for p in self.peers}
        rbuf = {p: torch.empty(nrecv[p] * L, dtype=torch.float64, device=dev) for p in self.peers}
        cbuf = torch.empty(len(cor) * L, dtype=torch.float64, device=dev)
        plan = (send, recv, nsend, nrecv, sbuf, rbuf, cg, cs, len(cor), cbuf)
        self._plans[names] = plan
        return plan

    def _call(self, entry, tensors, buf, idx, n):
        import torch

        from . import _lib

        g = self.d.grid
        fields = [g.abi(t) for t in tensors] + [_lib.tensor_buffer(buf), _lib.tensor_buffer(idx)]
        _lib.call(entry, fields, [float(n)], g.domain(), torch.cuda.current_stream().cuda_stream)

    def pack(self, names) -> list:
        names = tuple(names)
        send, recv, nsend, nrecv, sbuf, rbuf, *_ = self._plan(names)
        tensors = [self.d.cur[n] for n in names]
        for p in self.peers:
            self._call("fv3b_halo_gather", tensors, sbuf[p], send[p], nsend[p])
        return [(names, None, None, [(p, sbuf[p]) for p in self.peers], [(p, rbuf[p]) for p in self.peers])]

    def finish(self, chunks) -> None:
        for names, _, _, _, _ in chunks:
            send, recv, nsend, nrecv, sbuf, rbuf, cg, cs, ncor, cbuf = self._plan(names)
            tensors = [self.d.cur[n] for n in names]
            for p in self.peers:
                self._call("fv3b_halo_scatter", tensors, rbuf[p], recv[p], nrecv[p])
            self._call("fv3b_halo_gather", tensors, cbuf, cg, ncor)
            self._call("fv3b_halo_scatter", tensors, cbuf, cs, ncor)

    def update(self, names) -> None:
        timer = getattr(self.d, "timer", None)
        if timer is not None:
            timer.start("halo")
        chunks = self.pack(names)
        for _, _, _, snd, rcv in chunks:
            self.transport.exchange(snd, rcv)
        self.finish(chunks)
        if timer is not None:
            timer.stop("halo")


class CubePeerHalo:
    """The cubed-sphere halo update of one tile by peer-memory stores
    (``fv3b_halo_peer_idx``): this tile's cells go straight into its four
    neighbours' halos, rotated / component-swapped / sign-flipped on the
    way, one launch for all four; then, once every neighbour's stores have
    landed, the corner fill from the tile's own edge halos (a second launch
    of the same kernel with this tile as the destination).  No message
    buffers, no NCCL.

    ``peers.tensor(tile, name)``: neighbour ``tile``'s current tensor for
    ``name`` (``LoopbackTiles`` in one process; ``parallel.IpcPeers``-style
    mappings across processes).  ``sync(0)`` / ``sync(1)`` order the stores
    against the neighbours when the tiles do not share one stream
    (``parallel.FlagSync``)."""

    direct = True

    def __init__(self, dycore, tile: int, peers, sync=None):
        g = dycore.grid
        if g.ni != g.nj:
            raise ValueError("cubed-sphere tiles are square")
        self.d = dycore
        self.tile = tile
        self.n, self.h = g.ni, g.halo
        self.peers = peers
        self.sync = sync
        self.neighbours = sorted({s.nb for s in topology()[tile].values()})
        self._plans: dict = {}

    def _off(self, i: int, j: int) -> int:
        return i + j * self.d.grid.pitch

    def _plan(self, names: tuple):
        if names in self._plans:
            return self._plans[names]
        import torch

        check_names(names)
        if len(names) > 32:
            raise ValueError("at most 32 fields per cubed-sphere halo update")
        slot = {n: k for k, n in enumerate(names)}
        dev = self.d.cur[names[0]].device
        lists = []
        for p in self.neighbours:  # what neighbour p takes from this tile
            ent = [e for e in edge_entries(p, names, self.n, self.h) if e.src_tile == self.tile]
            lists.append(torch.tensor([[slot[e.src_name], self._off(e.si, e.sj), slot[e.name], self._off(e.i, e.j),
                                        1 if e.sign > 0 else -1] for e in ent], dtype=torch.int32,
                                      device=dev).reshape(-1))
        cor = corner_entries(names, self.n, self.h)
        corner = torch.tensor([[slot[e.src_name], self._off(e.si, e.sj), slot[e.name], self._off(e.i, e.j),
                                1 if e.sign > 0 else -1] for e in cor], dtype=torch.int32, device=dev).reshape(-1)
        self._plans[names] = (lists, corner)
        return self._plans[names]

    def _call(self, names, dst_sets, lists) -> None:
        import torch

        from . import _lib

        g = self.d.grid
        fields = [g.abi(self.d.cur[n]) for n in names] + [g.abi(t) for row in dst_sets for t in row]
        fields += [_lib.tensor_buffer(idx) for idx in lists]  # int32, 5 per entry
        s = [float(len(names)), float(len(lists))]
        _lib.call("fv3b_halo_peer_idx", fields, s, g.domain(), torch.cuda.current_stream().cuda_stream)

    def push(self, names) -> None:
        names = tuple(names)
        lists, _ = self._plan(names)
        self._call(names, [[self.peers.tensor(p, n) for n in names] for p in self.neighbours], lists)

    def corners(self, names) -> None:
        names = tuple(names)
        _, corner = self._plan(names)
        self._call(names, [[self.d.cur[n] for n in names]], [corner])

    def update(self, names) -> None:
        timer = getattr(self.d, "timer", None)
        if timer is not None:
            timer.start("halo")
        if self.sync is not None:
            self.sync(0)
        self.push(names)
        if self.sync is not None:
            self.sync(1)
        self.corners(names)
        if timer is not None:
            timer.stop("halo")


class LoopbackTiles:
    """The six tiles' dycores held in this process (CubePeerHalo peers)."""

    def __init__(self, dycores):
        self.d = dycores

    def tensor(self, tile: int, name: str):
        return self.d[tile].cur[name]
