"""Decomposed doubly periodic domains: the halo update between ranks.

The paper's dycore runs one horizontal block per GPU and refreshes halos with
a Python halo updater that packs edge strips, exchanges them with
non-blocking point-to-point messages and unpacks them (
SURVEY 8e).  Here:

* :class:`HaloPlan` — host logic only: the px x py block decomposition of a
  doubly periodic domain (rank r owns block (r % px, r // px)), the eight
  edge / corner strips each rank sends and receives, and the message layout
  (one contiguous message per peer, strips in a fixed direction order) that
  both sides derive independently.  Corners travel with the diagonal
  neighbours, so one round of messages fills the whole halo ring, exactly the
  values a single-domain periodic fill would write.
* packers — move strips between the field tensors (device Layout,
  ``device.Grid``) and message buffers: :class:`DevicePacker` runs the
  ``fv3b_halo_pack_rects`` / ``fv3b_halo_unpack_rects`` CUDA kernels (one
  launch per halo update for up to 32 fields); :class:`TorchPacker` does the
  same with tensor slicing (CPU tests, the gloo path).
* transports — :class:`DistTransport` posts one ``isend`` / ``irecv`` pair per
  peer through ``torch.distributed.batch_isend_irecv`` (NCCL over NVLink on
  the B200 box, gloo on CPU); messages to the rank itself (a periodic wrap
  along an undecomposed axis) are device copies.
* :class:`DecomposedHalo` — the halo object a :class:`~.dycore.Dycore` calls.
* :class:`PeerHalo` — the same update without messages: one
  ``fv3b_halo_peer_rects`` launch stores this rank's strips straight into
  the neighbours' halos (CUDA-IPC mappings over NVLink, :class:`IpcPeers`,
  or blocks on the same device, :class:`LoopbackPeers`).
* :class:`LoopbackCluster` — several ranks' dycores in one process on one
  GPU, advanced in lockstep with device copies as the transport; it checks
  the decomposed step against the single-domain step without a multi-GPU box.

No region of the shipped programs fires on a doubly periodic block
(placement all-False, ``lower.py:91-93``), so with correct halos every rank
computes bitwise what the single domain computes on its cells.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

DIRS = [(-1, -1), (0, -1), (1, -1), (-1, 0), (1, 0), (-1, 1), (0, 1), (1, 1)]  # (di, dj), message order
MAX_FIELDS = 32


@dataclass(frozen=True)
class Rect:
    """Interior-relative rectangle [i0, i0+w) x [j0, j0+h) (all levels)."""

    i0: int
    j0: int
    w: int
    h: int

    @property
    def cells(self) -> int:
        return self.w * self.h


def _span(d: int, n: int, h: int, send: bool) -> tuple[int, int]:
    if d == 0:
        return 0, n
    if send:
        return (0, h) if d < 0 else (n - h, h)
    return (-h, h) if d < 0 else (n, h)


class HaloPlan:
    """Neighbour strips and message layout of one rank of a px x py
    decomposition (uniform ni x nj blocks, halo width h)."""

    def __init__(self, ni: int, nj: int, h: int, px: int, py: int, rank: int):
        if not 0 <= rank < px * py:
            raise ValueError(f"rank {rank} outside a {px}x{py} decomposition")
        if h > ni or h > nj:
            raise ValueError("halo wider than the block")
        self.ni, self.nj, self.h, self.px, self.py, self.rank = ni, nj, h, px, py, rank
        self.ri, self.rj = rank % px, rank // px
        self.peer = [((self.ri + di) % px) + ((self.rj + dj) % py) * px for di, dj in DIRS]
        self.send = []
        self.recv = []
        for di, dj in DIRS:
            (si, wi), (sj, hj) = _span(di, ni, h, True), _span(dj, nj, h, True)
            self.send.append(Rect(si, sj, wi, hj))
            (ri, wi), (rj, hj) = _span(di, ni, h, False), _span(dj, nj, h, False)
            self.recv.append(Rect(ri, rj, wi, hj))
        self.peers = sorted(set(self.peer))
        # send order: per peer (ascending), directions in DIRS order
        self.send_order = [(p, [d for d in range(8) if self.peer[d] == p]) for p in self.peers]
        # receive order: the sender lists its strips for me in its DIRS order;
        # its direction is the negation of mine
        neg = {d: DIRS.index((-DIRS[d][0], -DIRS[d][1])) for d in range(8)}
        self.recv_order = [(p, sorted([e for e in range(8) if self.peer[e] == p], key=lambda e: neg[e]))
                           for p in self.peers]

    def layout(self, nfields: int, levels: int, recv: bool):
        """[(peer, start, length, [(direction, rect, offset)])] in elements."""
        out, off = [], 0
        for p, dirs in (self.recv_order if recv else self.send_order):
            start, items = off, []
            for d in dirs:
                r = (self.recv if recv else self.send)[d]
                items.append((d, r, off))
                off += r.cells * nfields * levels
            out.append((p, start, off - start, items))
        return out

    def total(self, nfields: int, levels: int) -> int:
        return sum(r.cells for r in self.send) * nfields * levels


def grid_shape(world: int) -> tuple[int, int]:
    """px x py of the weak-scaling decompositions (J split first)."""
    return {1: (1, 1), 2: (1, 2), 4: (2, 2), 6: (2, 3), 8: (2, 4)}.get(world, (1, world))


# ---------------------------------------------------------------------------
# packers
# ---------------------------------------------------------------------------

class TorchPacker:
    """Strip copies by tensor slicing (CPU tests; any device)."""

    def __init__(self, grid):
        self.grid = grid

    def _view(self, t: torch.Tensor, r: Rect) -> torch.Tensor:
        g = self.grid
        return t[:, g.halo + r.j0 : g.halo + r.j0 + r.h, g.i0 + r.i0 : g.i0 + r.i0 + r.w]

    def pack(self, tensors, rects, buf: torch.Tensor) -> None:
        L = tensors[0].shape[0]
        for r, off in rects:
            n = r.cells
            for t, x in enumerate(tensors):
                buf[off + t * L * n : off + (t + 1) * L * n].view(L, r.h, r.w).copy_(self._view(x, r))

    def unpack(self, tensors, rects, buf: torch.Tensor) -> None:
        L = tensors[0].shape[0]
        for r, off in rects:
            n = r.cells
            for t, x in enumerate(tensors):
                self._view(x, r).copy_(buf[off + t * L * n : off + (t + 1) * L * n].view(L, r.h, r.w))


class DevicePacker:
    """``fv3b_halo_pack_rects`` / ``fv3b_halo_unpack_rects``: all strips of
    a halo update for up to 32 fields in one launch each way."""

    def __init__(self, grid, placement=(False, False, False, False)):
        from . import _lib

        self._lib = _lib
        self.grid = grid
        self.dom = grid.domain(placement)

    def _call(self, entry, tensors, rects, buf):
        s = [float(len(rects))]
        for r, off in rects:
            s += [float(r.i0), float(r.j0), float(r.w), float(r.h), float(off)]
        fields = [self.grid.abi(t) for t in tensors] + [self._lib.tensor_buffer(buf)]
        self._lib.call(entry, fields, s, self.dom, torch.cuda.current_stream().cuda_stream)

    def pack(self, tensors, rects, buf):
        self._call("fv3b_halo_pack_rects", tensors, rects, buf)

    def unpack(self, tensors, rects, buf):
        self._call("fv3b_halo_unpack_rects", tensors, rects, buf)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class DistTransport:
    """One message per peer through torch.distributed P2P (grouped
    ncclSend/ncclRecv on NCCL); self messages are copies."""

    def __init__(self, rank: int, group=None):
        self.rank = rank
        self.group = group

    def exchange(self, send: list, recv: list) -> None:
        """send / recv: [(peer, tensor)] in the plan's peer order."""
        import torch.distributed as dist

        ops = []
        rbuf = dict(recv)
        for p, t in send:
            if p == self.rank:
                rbuf[p].copy_(t)
            else:
                ops.append(dist.P2POp(dist.isend, t, p, self.group))
                ops.append(dist.P2POp(dist.irecv, rbuf[p], p, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


# ---------------------------------------------------------------------------
# the halo object of a decomposed dycore
# ---------------------------------------------------------------------------

class DecomposedHalo:
    """Halo update of one rank; ``update(names)`` refreshes the I/J halos of
    the named state fields of ``dycore`` (a :class:`~.dycore.Dycore`)."""

    def __init__(self, dycore, px: int, py: int, rank: int, transport=None, packer=None):
        self.d = dycore
        g = dycore.grid
        self.plan = HaloPlan(g.ni, g.nj, g.halo, px, py, rank)
        self.transport = transport or DistTransport(rank)
        self.packer = packer or (DevicePacker(g) if dycore.device != "cpu" else TorchPacker(g))
        self._bufs: dict[tuple[int, int, int], tuple[torch.Tensor, torch.Tensor]] = {}

    def _buffers(self, chunk: int, nf: int, levels: int, device) -> tuple[torch.Tensor, torch.Tensor]:
        """Send / receive buffers of chunk ``chunk`` of an update (one pair
        per chunk: two equal-size chunks of one update must not share)."""
        key = (chunk, nf, levels)
        if key not in self._bufs:
            n = self.plan.total(nf, levels)
            self._bufs[key] = (torch.empty(n, dtype=torch.float64, device=device),
                               torch.empty(n, dtype=torch.float64, device=device))
        return self._bufs[key]

    def pack(self, names) -> list:
        """Pack every chunk of <= 32 fields; returns per-chunk state for
        :meth:`finish` (send / recv slices per peer)."""
        chunks = []
        for c in range(0, len(names), MAX_FIELDS):
            tensors = [self.d.cur[n] for n in names[c : c + MAX_FIELDS]]
            L = tensors[0].shape[0]
            sbuf, rbuf = self._buffers(c // MAX_FIELDS, len(tensors), L, tensors[0].device)
            slay = self.plan.layout(len(tensors), L, recv=False)
            rlay = self.plan.layout(len(tensors), L, recv=True)
            self.packer.pack(tensors, [(r, off) for _, _, _, items in slay for _, r, off in items], sbuf)
            send = [(p, sbuf[s : s + n]) for p, s, n, _ in slay]
            recv = [(p, rbuf[s : s + n]) for p, s, n, _ in rlay]
            chunks.append((tensors, rlay, rbuf, send, recv))
        return chunks

    def finish(self, chunks) -> None:
        for tensors, rlay, rbuf, _, _ in chunks:
            self.packer.unpack(tensors, [(r, off) for _, _, _, items in rlay for _, r, off in items], rbuf)

    def update(self, names) -> None:
        timer = getattr(self.d, "timer", None)
        if timer is not None:
            timer.start("halo")
        chunks = self.pack(list(names))
        for _, _, _, send, recv in chunks:
            self.transport.exchange(send, recv)
        self.finish(chunks)
        if timer is not None:
            timer.stop("halo")


NEG = [DIRS.index((-di, -dj)) for di, dj in DIRS]


class PeerHalo:
    """Halo update by peer-memory stores (``fv3b_halo_peer_rects``): this
    rank's eight edge / corner strips go straight into its neighbours' halos,
    one launch per update for up to 32 fields -- no message buffers, no
    pack / unpack, no NCCL on the data path.  On a multi-GPU node the
    neighbours' state buffers are CUDA-IPC mappings (:class:`IpcPeers`) and
    the stores travel over NVLink; in one process (:class:`LoopbackCluster`
    with ``direct=True``) they are other blocks on the same device.

    ``peers.tensor(direction, name)`` is the tensor the neighbour in that
    direction currently holds under ``name`` (lockstep ranks share the
    buffer assignment).  ``sync(0)`` / ``sync(1)`` run before and after the
    stores when the ranks do not share one stream: before, every neighbour
    has finished reading its old halo; after, every store into this rank's
    halo has landed.  :class:`FlagSync` does this on the device (graph-
    capturable, no host round trip); :func:`ipc_sync` with host barriers."""

    def __init__(self, dycore, px: int, py: int, rank: int, peers, sync=None, copier=None):
        self.d = dycore
        g = dycore.grid
        self.plan = HaloPlan(g.ni, g.nj, g.halo, px, py, rank)
        self.peers = peers
        self.sync = sync
        self.copier = copier or (DevicePeerCopier(g) if dycore.device != "cpu" else TorchPeerCopier(g))
        # direction d: my send strip -> the recv strip of direction -d of the neighbour peer[d]
        self.rects = []
        for d in range(8):
            s, r = self.plan.send[d], self.plan.recv[NEG[d]]
            self.rects.append((s.i0, s.j0, r.i0, r.j0, s.w, s.h))

    direct = True  # LoopbackCluster: stores into the neighbours, no messages

    def push(self, names) -> None:
        """Store this rank's strips into the neighbours' halos."""
        names = list(names)
        for c in range(0, len(names), MAX_FIELDS):
            chunk = names[c : c + MAX_FIELDS]
            self.copier([self.d.cur[n] for n in chunk],
                        [[self.peers.tensor(d, n) for n in chunk] for d in range(8)], self.rects)

    def corners(self, names) -> None:
        """(Corners travel with the diagonal neighbours: nothing local.)"""

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


class DevicePeerCopier:
    """``fv3b_halo_peer_rects``: every strip of every field, one launch."""

    def __init__(self, grid):
        from . import _lib

        self._lib = _lib
        self.grid = grid
        self.dom = grid.domain()
        self._prepared: dict = {}  # buffer addresses -> ctypes argument arrays

    def __call__(self, src, dst, rects) -> None:
        key = tuple(t.data_ptr() for t in src) + tuple(t.data_ptr() for row in dst for t in row)
        args = self._prepared.get(key)
        if args is None:
            g = self.grid
            fields = [g.abi(t) for t in src] + [g.abi(t) for row in dst for t in row]
            s = [float(len(src)), float(len(rects))] + [float(x) for r in rects for x in r]
            args = self._prepared[key] = self._lib.prepare(fields, s)
        self._lib.call_prepared("fv3b_halo_peer_rects", args, self.dom, torch.cuda.current_stream().cuda_stream)


class TorchPeerCopier:
    """The same strip copies by tensor slicing (CPU tests)."""

    def __init__(self, grid):
        self.grid = grid

    def _view(self, t, i0, j0, w, h):
        g = self.grid
        return t[:, g.halo + j0 : g.halo + j0 + h, g.i0 + i0 : g.i0 + i0 + w]

    def __call__(self, src, dst, rects) -> None:
        for (si, sj, di, dj, w, h), row in zip(rects, dst):
            for s, o in zip(src, row):
                self._view(o, di, dj, w, h).copy_(self._view(s, si, sj, w, h))


class LoopbackPeers:
    """The neighbours of one rank among dycores held in this process."""

    def __init__(self, dycores, plan: HaloPlan):
        self.d = dycores
        self.plan = plan

    def tensor(self, direction: int, name: str) -> torch.Tensor:
        return self.d[self.plan.peer[direction]].cur[name]


class IpcPeers:
    """The neighbours' state buffers mapped into this process with CUDA IPC
    (one process per GPU on an NVLink node; peer access is enabled by the
    IPC open).  Every rank enumerates its state buffers in the same order
    (sorted names, current then alternate), so buffer b of rank p is the one
    rank p holds wherever this rank holds its own buffer b.  The handles
    travel once, at construction, through ``all_gather_object`` on
    ``group`` (any backend)."""

    def __init__(self, dycore, plan: HaloPlan | None, group=None, flags: torch.Tensor | None = None,
                 neighbours=None, rank: int | None = None):
        """``plan``: a px x py decomposition's HaloPlan (neighbours and rank
        from it); otherwise ``neighbours`` (ranks) and ``rank`` (e.g. the
        cubed sphere's four adjacent tiles, :meth:`tiles`)."""
        import pickle
        from multiprocessing.reduction import ForkingPickler

        import torch.distributed as dist
        import torch.multiprocessing  # noqa: F401  (registers the tensor reducers)

        self.d = dycore
        self.plan = plan
        self.rank = plan.rank if plan is not None else rank
        nbrs = set(plan.peer) if plan is not None else set(neighbours)
        mine = self._buffers(dycore)
        if flags is not None:  # the FlagSync array travels as the last buffer
            mine.append(flags)
        # CUDA tensors pickle as IPC handles (CPU tensors move to shared memory)
        shared = [bytes(ForkingPickler.dumps(t)) for t in mine]
        self._index = {t.data_ptr(): b for b, t in enumerate(mine)}
        gathered: list = [None] * dist.get_world_size(group)
        dist.all_gather_object(gathered, shared, group=group)
        self._peer = {}
        for p in nbrs:
            self._peer[p] = mine if p == self.rank else [pickle.loads(b) for b in gathered[p]]
        # neighbours on other GPUs: this device's kernels store into their memory
        if mine and mine[0].is_cuda:
            from . import _lib

            here = mine[0].device.index
            for p, bufs in self._peer.items():
                if bufs and bufs[0].device.index != here:
                    with torch.cuda.device(here):
                        _lib.enable_peer_access(bufs[0].device.index)
        self.flags = flags
        self.neighbours = sorted(nbrs)

    def flag_sync(self) -> FlagSync:
        """The device-side barrier over the shared flag arrays."""
        if self.flags is None:
            raise ValueError("IpcPeers was built without a flag array")
        return FlagSync(self.rank, self.neighbours, self.flags, {p: b[-1] for p, b in self._peer.items()})

    def rank_tensor(self, p: int, name: str) -> torch.Tensor:
        """Rank p's tensor that holds ``name`` in the shared buffer assignment."""
        return self._peer[p][self._index[self.d.cur[name].data_ptr()]]

    def tiles(self):
        """The ``tensor(tile, name)`` view CubePeerHalo takes."""
        ipc = self

        class _Tiles:
            def tensor(self, tile: int, name: str) -> torch.Tensor:
                return ipc.rank_tensor(tile, name)

        return _Tiles()

    @staticmethod
    def _buffers(dycore) -> list:
        out, seen = [], set()
        for table in (dycore.cur, dycore.alt):
            for n in sorted(table):
                t = table[n]
                if t.data_ptr() not in seen:
                    seen.add(t.data_ptr())
                    out.append(t)
        return out

    def tensor(self, direction: int, name: str) -> torch.Tensor:
        return self.rank_tensor(self.plan.peer[direction], name)


def ipc_sync(group=None, device: bool = True):
    """Cross-process ordering for :class:`PeerHalo`: drain this rank's
    stream (``device``), then a barrier on ``group``."""
    import torch.distributed as dist

    def sync(phase: int):
        if device:
            torch.cuda.current_stream().synchronize()
        dist.barrier(group=group)

    return sync


class FlagSync:
    """Stream-ordered barrier of one rank with its neighbours for
    :class:`PeerHalo` (``fv3b_peer_barrier``): every rank owns an int64
    flag array [2, world] (phase 0 = arrived, 1 = stored; column p = rank
    p's word); a barrier bumps (phase 0) or reuses (phase 1) the rank's
    update counter, release-stores it into its column of each neighbour's
    array and spins on its own array until every neighbour has caught up.
    ``peer_flags[p]``: neighbour p's flag array as mapped in this process
    (CUDA IPC across processes, the tensor itself in one process)."""

    def __init__(self, rank: int, neighbours, flags: torch.Tensor, peer_flags: dict):
        from . import _lib

        self._lib = _lib
        world = flags.shape[1]
        self.flags = flags
        self.epoch = torch.zeros(1, dtype=torch.int64, device=flags.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=flags.device)
        self._keep = dict(peer_flags)
        nb = sorted(p for p in set(neighbours) if p != rank)
        self.dom = _lib.Domain()
        self._args = []
        for phase in (0, 1):
            words = [_lib.tensor_buffer(self.epoch), _lib.tensor_buffer(self.err)]
            for p in nb:
                remote = peer_flags[p].data_ptr() + 8 * (phase * world + rank)
                local = flags.data_ptr() + 8 * (phase * world + p)
                words += [_lib.buffer_field(remote, 1), _lib.buffer_field(local, 1)]
            self._args.append(_lib.prepare(words, [1.0 - phase, float(len(nb))]))

    def __call__(self, phase: int) -> None:
        self._lib.call_prepared("fv3b_peer_barrier", self._args[phase], self.dom,
                                torch.cuda.current_stream().cuda_stream)

    def check(self) -> None:
        """Raise if a barrier timed out (reads the device error word)."""
        if int(self.err.item()):
            raise RuntimeError("fv3b_peer_barrier: a neighbour did not arrive within 10 s")


def new_flags(world: int, device) -> torch.Tensor:
    """A rank's zeroed flag array for :class:`FlagSync`."""
    return torch.zeros(2, world, dtype=torch.int64, device=device)


class LoopbackCluster:
    """px x py ranks' dycores in one process, stepped in lockstep; messages
    are device copies between the ranks' buffers (tests / single-GPU
    validation of the decomposed path)."""

    def __init__(self, dycores, px: int = 1, py: int = 1, halos=None, direct: bool = False,
                 flag_sync: bool = False, concurrent: bool = False):
        """``halos``: per-rank halo objects exposing pack / finish (default:
        a px x py doubly periodic decomposition; cubesphere.CubeHalo for
        the six tiles of a cube; ``cubesphere.CubePeerHalo`` for its
        peer-memory form).  ``direct``: the decomposition's halo updates as
        peer-memory stores (:class:`PeerHalo`) instead of pack / copy /
        unpack.  ``flag_sync``: every rank on its own stream, ordered only by
        the device-side neighbour barriers (:class:`FlagSync`; built here for
        ``direct``, supplied with ``halos`` otherwise), as separate
        processes would be.  A measurement mode: in one process the ranks'
        streams must land on distinct hardware queues (at most
        CUDA_DEVICE_MAX_CONNECTIONS streams), or one rank's spinning barrier
        blocks a neighbour's arrival queued behind it until the barrier's
        10 s bound expires.  ``concurrent``: every rank's programs between
        two halo points on its own stream, joined before each exchange and
        forked after it (stream order only, no device barriers), so the
        ranks' kernels share the GPU -- the six small cube tiles of C3 on
        one device fill it together instead of one after another."""
        self.d = dycores
        self.streams = None
        self.cstreams = [torch.cuda.Stream() for _ in dycores] if concurrent and not flag_sync else None
        if direct and halos is None:
            self.halos = []
            flags = [new_flags(len(dycores), d.device) for d in dycores] if flag_sync else None
            for r, d in enumerate(dycores):
                plan = HaloPlan(d.grid.ni, d.grid.nj, d.grid.halo, px, py, r)
                sync = FlagSync(r, plan.peer, flags[r], dict(enumerate(flags))) if flag_sync else None
                self.halos.append(PeerHalo(d, px, py, r, LoopbackPeers(dycores, plan), sync=sync))
        else:
            self.halos = halos or [DecomposedHalo(d, px, py, r, transport=self, packer=None)
                                   for r, d in enumerate(dycores)]
        if flag_sync and not all(getattr(h, "direct", False) and h.sync is not None for h in self.halos):
            raise ValueError("flag_sync needs peer-store halos with device barriers (direct=True, or such halos)")
        if flag_sync:
            self.streams = [torch.cuda.Stream() for _ in dycores]
        for d, h in zip(dycores, self.halos):
            d.halo = h

    def exchange(self, send, recv):  # transports run inside step(); see below
        raise RuntimeError("LoopbackCluster exchanges all ranks at once (use step())")

    def exchange_all(self, reqs) -> None:
        """One halo update on every rank (``reqs[r]``: rank r's field list)."""
        if getattr(self.halos[0], "direct", False):  # peer-memory stores into the neighbours
            if self.streams:  # each rank on its stream, ordered by its device barriers
                for r, (h, names) in enumerate(zip(self.halos, reqs)):
                    with self._on(r):
                        h.update(names)
            else:  # one stream: every rank's stores, then every rank's local corner fill
                for h, names in zip(self.halos, reqs):
                    h.push(names)
                for h, names in zip(self.halos, reqs):
                    h.corners(names)
            return
        chunks = [h.pack(names) for h, names in zip(self.halos, reqs)]
        for r, ch in enumerate(chunks):
            for c, (_, _, _, _, recv) in enumerate(ch):
                for p, rt in recv:
                    rt.copy_(dict(chunks[p][c][3])[r])  # peer p's message to r
        for h, ch in zip(self.halos, chunks):
            h.finish(ch)

    def _assignment(self) -> tuple:
        return tuple(d._assignment() for d in self.d)

    def capture(self) -> None:
        """Capture one lockstep step of every rank (programs and device-copy
        halo exchanges) as a CUDA graph per distinct buffer assignment, as
        Dycore.capture does for one rank.  Captures execute nothing; the
        bookkeeping is restored afterwards."""
        import torch

        from .device import capture_guard

        start = [(dict(d.cur), dict(d.alt)) for d in self.d]
        self._graphs = {}
        with capture_guard():
            while self._assignment() not in self._graphs:
                key = self._assignment()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self.step()
                self._graphs[key] = (g, [(dict(d.cur), dict(d.alt)) for d in self.d])
        for d, (cur, alt) in zip(self.d, start):
            d.cur, d.alt = cur, alt
        torch.cuda.synchronize()

    def replay(self) -> None:
        """Run one captured lockstep step on the current stream."""
        g, post = self._graphs[self._assignment()]
        g.replay()
        for d, (cur, alt) in zip(self.d, post):
            d.cur, d.alt = dict(cur), dict(alt)

    def _on(self, r: int):
        import contextlib

        ranks = self.streams or self.cstreams
        return torch.cuda.stream(ranks[r]) if ranks else contextlib.nullcontext()

    def step(self) -> None:
        gens = [d.phases() for d in self.d]
        main = torch.cuda.current_stream()
        ranks = self.streams or self.cstreams
        if ranks:
            for s in ranks:
                s.wait_stream(main)
        while True:
            reqs = []
            for r, g in enumerate(gens):
                with self._on(r):
                    reqs.append(next(g, None))
            if all(r is None for r in reqs):
                break
            assert all(r is not None for r in reqs), "ranks out of lockstep"
            if self.cstreams:  # join the ranks' programs, exchange on the main stream, fork again
                for s in self.cstreams:
                    main.wait_stream(s)
                self.exchange_all(reqs)
                for s in self.cstreams:
                    s.wait_stream(main)
            else:
                self.exchange_all(reqs)
        if ranks:
            for s in ranks:
                main.wait_stream(s)
