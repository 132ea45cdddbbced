"""Decomposed doubly periodic domains (parallel.py) on CPU: the halo plan's
message layouts agree between every sender / receiver pair, and the halo
update of a px x py decomposition reproduces the single-domain periodic fill
exactly — in process (loopback) and across two gloo ranks."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from paper_2205_04148_b200.device import Grid
from paper_2205_04148_b200.parallel import DIRS, DecomposedHalo, DistTransport, HaloPlan, TorchPacker
from paper_2205_04148_b200.state import periodic_fill

DECOMPS = [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (3, 2), (2, 4), (1, 3)]


@pytest.mark.parametrize("px,py", DECOMPS)
def test_message_layouts_pair_up(px, py):
    ni, nj, h, nf, L = 7, 5, 3, 3, 4
    plans = [HaloPlan(ni, nj, h, px, py, r) for r in range(px * py)]
    for r, pr in enumerate(plans):
        for p, _, n, items in pr.layout(nf, L, recv=False):
            # what r sends to p == what p expects from r, strip by strip
            recv = {q: it for q, _, _, it in plans[p].layout(nf, L, recv=True)}[r]
            assert [(x.w, x.h) for _, x, _ in items] == [(x.w, x.h) for _, x, _ in recv]
            for (ds, _, _), (dr, _, _) in zip(items, recv):
                assert DIRS[ds] == (-DIRS[dr][0], -DIRS[dr][1])
    for pr in plans:  # the receive strips tile the halo ring exactly once
        ring = sum(x.cells for x in pr.recv)
        assert ring == (ni + 2 * h) * (nj + 2 * h) - ni * nj


class _Stub:
    """Just what DecomposedHalo needs from a Dycore: grid, cur, device."""

    def __init__(self, grid, fields):
        self.grid, self.cur, self.device, self.timer = grid, fields, "cpu", None


def _global_fields(nf, NI, NJ, L, h, seed=5):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(nf):
        a = rng.uniform(-1, 1, (NI + 2 * h, NJ + 2 * h, L))
        periodic_fill(a, h)
        out.append(a)
    return out


def _block(a, ri, rj, ni, nj, h):
    """Block (ri, rj) of a periodic global array, halo included (wrapped)."""
    NI, NJ = a.shape[0] - 2 * h, a.shape[1] - 2 * h
    ii = (np.arange(ri * ni - h, (ri + 1) * ni + h) % NI) + h
    jj = (np.arange(rj * nj - h, (rj + 1) * nj + h) % NJ) + h
    return a[np.ix_(ii, jj)]


def _local(grid, a_blk, h, scramble):
    t = grid.new3("cpu", fill=0.0)
    src = a_blk.copy()
    if scramble:  # halos start as garbage
        src[:h] = src[-h:] = np.nan
        src[:, :h] = src[:, -h:] = np.nan
    grid.put(t, src, ("I", "J", "K"), (h, h, 0))
    return t


class _Loopback:
    def __init__(self, halos):
        self.halos = halos

    def run(self, names):
        chunks = [hh.pack(names) for hh in self.halos]
        for r, ch in enumerate(chunks):
            for c, (_, _, _, _, recv) in enumerate(ch):
                for p, rt in recv:
                    rt.copy_(dict(chunks[p][c][3])[r])
        for hh, ch in zip(self.halos, chunks):
            hh.finish(ch)


@pytest.mark.parametrize("px,py", DECOMPS)
def test_loopback_halo_equals_global_periodic_fill(px, py):
    ni, nj, nk, h, nf = 9, 7, 3, 4, 3
    grid = Grid(ni, nj, nk, halo=h)
    glob = _global_fields(nf, px * ni, py * nj, grid.levels, h)
    stubs = []
    for r in range(px * py):
        ri, rj = r % px, r // px
        fields = {f"f{t}": _local(grid, _block(glob[t], ri, rj, ni, nj, h), h, True) for t in range(nf)}
        stubs.append(_Stub(grid, fields))
    halos = [DecomposedHalo(s, px, py, r, transport=object(), packer=TorchPacker(grid)) for r, s in enumerate(stubs)]
    _Loopback(halos).run([f"f{t}" for t in range(nf)])
    for r, s in enumerate(stubs):
        ri, rj = r % px, r // px
        for t in range(nf):
            got = grid.get(s.cur[f"f{t}"], ("I", "J", "K"), (h, h, 0), (ni + 2 * h, nj + 2 * h, grid.levels))
            np.testing.assert_array_equal(got, _block(glob[t], ri, rj, ni, nj, h))


def _gloo_worker(rank, world, port, px, py, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ni, nj, nk, h, nf = 8, 6, 2, 3, 2
        grid = Grid(ni, nj, nk, halo=h)
        glob = _global_fields(nf, px * ni, py * nj, grid.levels, h, seed=11)
        ri, rj = rank % px, rank // px
        fields = {f"f{t}": _local(grid, _block(glob[t], ri, rj, ni, nj, h), h, True) for t in range(nf)}
        halo = DecomposedHalo(_Stub(grid, fields), px, py, rank, transport=DistTransport(rank),
                              packer=TorchPacker(grid))
        halo.update([f"f{t}" for t in range(nf)])
        ok = all(np.array_equal(grid.get(fields[f"f{t}"], ("I", "J", "K"), (h, h, 0),
                                          (ni + 2 * h, nj + 2 * h, grid.levels)),
                                _block(glob[t], ri, rj, ni, nj, h)) for t in range(nf))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("px,py", [(1, 2), (2, 1)])
def test_gloo_two_ranks_halo_exchange(px, py):
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, px, py, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("px,py", DECOMPS)
def test_peer_halo_equals_global_periodic_fill(px, py):
    """PeerHalo's store plan (my send strip of direction d -> the recv strip
    of direction -d of neighbour peer[d]) fills every block's halo ring with
    the single-domain periodic values; strips emulated by tensor slicing."""
    from paper_2205_04148_b200.parallel import LoopbackPeers, PeerHalo, TorchPeerCopier

    ni, nj, nk, h, nf = 9, 7, 3, 4, 3
    grid = Grid(ni, nj, nk, halo=h)
    glob = _global_fields(nf, px * ni, py * nj, grid.levels, h, seed=17)
    stubs = []
    for r in range(px * py):
        ri, rj = r % px, r // px
        fields = {f"f{t}": _local(grid, _block(glob[t], ri, rj, ni, nj, h), h, True) for t in range(nf)}
        stubs.append(_Stub(grid, fields))
    for r, s in enumerate(stubs):
        halo = PeerHalo(s, px, py, r, LoopbackPeers(stubs, HaloPlan(ni, nj, h, px, py, r)),
                        copier=TorchPeerCopier(grid))
        halo.update([f"f{t}" for t in range(nf)])
    for r, s in enumerate(stubs):
        ri, rj = r % px, r // px
        for t in range(nf):
            got = grid.get(s.cur[f"f{t}"], ("I", "J", "K"), (h, h, 0), (ni + 2 * h, nj + 2 * h, grid.levels))
            np.testing.assert_array_equal(got, _block(glob[t], ri, rj, ni, nj, h))


def _ipc_worker(rank, world, port, px, py, q):
    import torch.distributed as dist
    import torch.multiprocessing as tmp

    from paper_2205_04148_b200.parallel import IpcPeers, PeerHalo, TorchPeerCopier, ipc_sync

    tmp.set_sharing_strategy("file_system")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ni, nj, nk, h, nf = 8, 6, 2, 3, 2
        grid = Grid(ni, nj, nk, halo=h)
        glob = _global_fields(nf, px * ni, py * nj, grid.levels, h, seed=23)
        ri, rj = rank % px, rank // px
        fields = {f"f{t}": _local(grid, _block(glob[t], ri, rj, ni, nj, h), h, True) for t in range(nf)}
        stub = _Stub(grid, fields)
        stub.alt = {}
        peers = IpcPeers(stub, HaloPlan(ni, nj, h, px, py, rank))
        halo = PeerHalo(stub, px, py, rank, peers, sync=ipc_sync(device=False), copier=TorchPeerCopier(grid))
        halo.update([f"f{t}" for t in range(nf)])
        ok = all(np.array_equal(grid.get(stub.cur[f"f{t}"], ("I", "J", "K"), (h, h, 0),
                                          (ni + 2 * h, nj + 2 * h, grid.levels)),
                                _block(glob[t], ri, rj, ni, nj, h)) for t in range(nf))
        q.put((rank, ok))
        dist.barrier()  # keep the shared buffers alive until every rank has checked
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("px,py", [(1, 2), (2, 1)])
def test_ipc_peer_halo_two_ranks(px, py):
    """The multi-process PeerHalo plumbing (IpcPeers handle exchange through
    all_gather_object, buffer indexing, barrier ordering) on two gloo ranks,
    with shared CPU tensors standing in for CUDA-IPC mappings."""
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, px, py, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


# ---------------------------------------------------------------------------
# a decomposed timestep across two gloo processes (the oracle programs on each
# rank's block, DecomposedHalo + DistTransport at every halo point) against
# the single-domain oracle step
# ---------------------------------------------------------------------------

class _NumpyGrid:
    """What DecomposedHalo / TorchPacker need from a Grid, for (K, J, I)
    views of the oracle's (I, J, K) state arrays (uniform halo, no pre-pad)."""

    def __init__(self, ni, nj, h):
        self.ni, self.nj, self.halo, self.i0 = ni, nj, h, h


def _step_worker(rank, world, port, px, py, q):
    import torch.distributed as dist

    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.state import initial_state

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ni, nj, nk = 16, 16, 4
        glob_cfg = RunConfig(ni=px * ni, nj=py * nj, nk=nk, n_split=2, dt_atmos=30.0)
        glob = initial_state(glob_cfg)
        h = glob_cfg.halo
        ri, rj = rank % px, rank // px
        local = {n: np.ascontiguousarray(_block(a, ri, rj, ni, nj, h)) if a.ndim == 3 else
                 np.ascontiguousarray(_block(a[..., None], ri, rj, ni, nj, h)[..., 0]) for n, a in glob.items()}
        cfg = RunConfig(ni=ni, nj=nj, nk=nk, n_split=2, dt_atmos=30.0)
        od = OracleDycore(cfg, local)
        stub = _Stub(_NumpyGrid(ni, nj, h), {})
        halo = DecomposedHalo(stub, px, py, rank, transport=DistTransport(rank), packer=TorchPacker(stub.grid))
        for _ in range(2):
            for names in od.phases():
                stub.cur = {n: torch.from_numpy(local[n]).permute(2, 1, 0) for n in names}
                halo.update(names)
        q.put((rank, {n: local[n][h:-h, h:-h] for n in ("u", "v", "w", "delp", "pt", "gz", "q0", "mfx")}))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("px,py", [(1, 2), (2, 1)])
def test_gloo_two_rank_decomposed_timestep_equals_single_domain(px, py):
    """Two timesteps of a 1x2 / 2x1 decomposition on two gloo processes
    (DecomposedHalo, DistTransport, the message layouts of every halo point
    of the step) == the single-domain oracle step on the whole domain."""
    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.state import initial_state

    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port, px, py, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    ni, nj, nk = 16, 16, 4
    cfg = RunConfig(ni=px * ni, nj=py * nj, nk=nk, n_split=2, dt_atmos=30.0)
    st = initial_state(cfg)
    ref = OracleDycore(cfg, st)
    for _ in range(2):
        ref.step()
    h = cfg.halo
    for r in range(2):
        ri, rj = r % px, r // px
        for n, got in res[r].items():
            top = nk + 1 if n == "gz" else nk
            want = st[n][h + ri * ni: h + (ri + 1) * ni, h + rj * nj: h + (rj + 1) * nj, :top]
            assert np.array_equal(got[..., :top], want), (r, n)


def test_loopback_halo_two_equal_chunks():
    """One update of 64 fields = two chunks of 32 with equal message sizes:
    each chunk has its own buffers (keyed by chunk, not size)."""
    px, py = 2, 2
    ni, nj, nk, h, nf = 6, 5, 1, 3, 64
    grid = Grid(ni, nj, nk, halo=h)
    glob = _global_fields(nf, px * ni, py * nj, grid.levels, h, seed=29)
    stubs = []
    for r in range(px * py):
        ri, rj = r % px, r // px
        fields = {f"f{t}": _local(grid, _block(glob[t], ri, rj, ni, nj, h), h, True) for t in range(nf)}
        stubs.append(_Stub(grid, fields))
    halos = [DecomposedHalo(s, px, py, r, transport=object(), packer=TorchPacker(grid)) for r, s in enumerate(stubs)]
    _Loopback(halos).run([f"f{t}" for t in range(nf)])
    for r, s in enumerate(stubs):
        ri, rj = r % px, r // px
        for t in range(nf):
            got = grid.get(s.cur[f"f{t}"], ("I", "J", "K"), (h, h, 0), (ni + 2 * h, nj + 2 * h, grid.levels))
            np.testing.assert_array_equal(got, _block(glob[t], ri, rj, ni, nj, h))
