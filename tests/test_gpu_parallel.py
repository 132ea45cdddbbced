"""Decomposed dycore on one B200: the CUDA pack / unpack kernels
(fv3b_halo_pack_rects / unpack_rects) reproduce the single-rank periodic halo
kernel, and a 2 x 2 (and 1 x 2) decomposition advanced in lockstep with
device-copy transport (parallel.LoopbackCluster) is bitwise the single-domain
dycore on every block."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _block(a, ri, rj, ni, nj, h):
    NI, NJ = a.shape[0] - 2 * h, a.shape[1] - 2 * h
    ii = (np.arange(ri * ni - h, (ri + 1) * ni + h) % NI) + h
    jj = (np.arange(rj * nj - h, (rj + 1) * nj + h) % NJ) + h
    return a[np.ix_(ii, jj)]


class _SelfTransport:
    def exchange(self, send, recv):
        rb = dict(recv)
        for p, t in send:
            assert p == 0
            rb[p].copy_(t)


def test_device_packer_single_rank_equals_periodic_kernel():
    import torch

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import DecomposedHalo

    cfg = RunConfig(ni=40, nj=24, nk=6, nq=2)
    a = Dycore(cfg)
    b = Dycore(cfg)
    g = torch.Generator(device="cuda").manual_seed(3)
    names = ["u", "v", "w", "q0", "q1"]
    for n in names:
        a.cur[n].copy_(torch.rand(a.cur[n].shape, generator=g, device="cuda", dtype=torch.float64))
        b.cur[n].copy_(a.cur[n])
    a.halo.update(names)
    DecomposedHalo(b, 1, 1, 0, transport=_SelfTransport()).update(names)
    torch.cuda.synchronize()
    for n in names:
        assert torch.equal(a.cur[n], b.cur[n]), n


@pytest.mark.parametrize("mode", ["packed", "direct", "direct-graph", "concurrent", "concurrent-graph"])
@pytest.mark.parametrize("px,py", [(2, 2), (1, 2)])
def test_loopback_decomposed_dycore_bitwise(px, py, mode):
    """packed: pack / device copy / unpack; direct: PeerHalo
    (fv3b_halo_peer_rects stores into the neighbours' halos), eager or
    captured as CUDA graphs and replayed.  The device-side neighbour
    barriers (fv3b_peer_barrier) are tested across processes
    (test_ipc_peer_halo_two_processes_bitwise): in one process, spinning
    barrier kernels on streams that happen to share a hardware queue
    (CUDA_DEVICE_MAX_CONNECTIONS) would wait on each other."""
    import torch

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import LoopbackCluster
    from paper_2205_04148_b200.state import initial_state

    ni, nj, nk = 32, 24, 8
    glob_cfg = RunConfig(ni=px * ni, nj=py * nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
    blk_cfg = RunConfig(ni=ni, nj=nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
    st = initial_state(glob_cfg)
    h = glob_cfg.halo
    ref = Dycore(glob_cfg, st)
    blocks = []
    for r in range(px * py):
        ri, rj = r % px, r // px
        blocks.append(Dycore(blk_cfg, {n: _block(a, ri, rj, ni, nj, h) for n, a in st.items()}))
    graph = mode.endswith("-graph")
    conc = mode.startswith("concurrent")  # each rank's programs on its own stream (packed halos)
    cluster = LoopbackCluster(blocks, px, py, direct=mode.startswith("direct"), flag_sync=mode == "flags",
                              concurrent=conc)
    if graph:
        cluster.capture()
    for _ in range(2):
        ref.step()
        cluster.replay() if graph else cluster.step()
    torch.cuda.synchronize()
    if mode == "flags":
        for hal in cluster.halos:
            hal.sync.check()
    names = ["u", "v", "w", "delp", "pt", "gz", "pef", "q0", "q1", "q1_a4", "mfx", "cy"]
    full = ref.download(names)
    for r, d in enumerate(blocks):
        ri, rj = r % px, r // px
        got = d.download(names)
        for n in names:
            want = _block(full[n], ri, rj, ni, nj, h)[h:-h, h:-h]
            assert np.array_equal(got[n][h:-h, h:-h], want), (r, n)


def _ipc_worker(rank, port, q, flags=False):
    """One rank of a 1 x 2 decomposition in its own process on cuda:0; the
    neighbour's state buffers are CUDA-IPC mappings (parallel.IpcPeers)."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import HaloPlan, IpcPeers, PeerHalo, ipc_sync, new_flags
    from paper_2205_04148_b200.state import initial_state

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        ni, nj, nk, px, py = 32, 24, 8, 1, 2
        glob_cfg = RunConfig(ni=px * ni, nj=py * nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
        blk_cfg = RunConfig(ni=ni, nj=nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
        st = initial_state(glob_cfg)
        h = glob_cfg.halo
        ri, rj = rank % px, rank // px
        d = Dycore(blk_cfg, {n: _block(a, ri, rj, ni, nj, h) for n, a in st.items()})
        peers = IpcPeers(d, HaloPlan(ni, nj, h, px, py, rank), flags=new_flags(2, "cuda") if flags else None)
        sync = peers.flag_sync() if flags else ipc_sync()
        d.halo = PeerHalo(d, px, py, rank, peers, sync=sync)
        dist.barrier()
        for _ in range(2):
            d.step()
        torch.cuda.synchronize()
        if flags:
            sync.check()
        names = ["u", "v", "w", "delp", "pt", "gz", "q0", "q1"]
        got = d.download(names)
        q.put((rank, {n: got[n][h:-h, h:-h] for n in names}))
        dist.barrier()  # the neighbour's mappings stay valid until both are done
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("flags", [False, True])
def test_ipc_peer_halo_two_processes_bitwise(flags):
    """Two processes (one per rank, as on an NVLink node) exchanging halos by
    peer-memory stores through CUDA IPC, here both on cuda:0, ordered by
    host barriers or by the device-side neighbour barriers (the contexts
    time-slice; the barrier spin is bounded): bitwise the single-domain
    dycore."""
    import socket

    import torch

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.state import initial_state

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q, flags)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    ni, nj, nk = 32, 24, 8
    glob_cfg = RunConfig(ni=ni, nj=2 * nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
    ref = Dycore(glob_cfg, initial_state(glob_cfg))
    for _ in range(2):
        ref.step()
    torch.cuda.synchronize()
    h = glob_cfg.halo
    full = ref.download(list(res[0]))
    for r in range(2):
        for n, got in res[r].items():
            assert np.array_equal(got, _block(full[n], 0, r, ni, nj, h)[h:-h, h:-h]), (r, n)
