"""Cubed sphere (config C3) on one B200: six tiles advanced in lockstep
with the CUDA index-list halo (CubeHalo: rotated edge strips, vector
component swap and sign, corner fill) moved by device copies, against the
NumPy oracle of the same specification (oracle/cube.py) — the halo update
alone and the full FULL_TILE dycore step, bitwise."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAMES = ["u", "v", "uc", "vc", "delp", "pt", "q0", "cx", "cy", "mfx", "mfy"]


def _cluster(cfg, states, mode="packed"):
    """packed: CubeHalo (gather / device copy / scatter); direct:
    CubePeerHalo (stores into the neighbour tiles, one stream).  ("flags",
    every tile on its own stream ordered by the device-side barriers, is a
    benchmarking mode only: in one process, spinning barrier kernels on
    streams that share a hardware queue wait on each other.)"""
    from paper_2205_04148_b200.cubesphere import CubeHalo, CubePeerHalo, LoopbackTiles
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import FlagSync, LoopbackCluster, new_flags

    tiles = [Dycore(cfg, st, placement=(True, True, True, True)) for st in states]
    if mode in ("packed", "concurrent"):  # concurrent: each tile's programs on its own stream (bench C3)
        return tiles, LoopbackCluster(tiles, halos=[CubeHalo(d, t, transport=None) for t, d in enumerate(tiles)],
                                      concurrent=mode == "concurrent")
    peers = LoopbackTiles(tiles)
    halos = [CubePeerHalo(d, t, peers) for t, d in enumerate(tiles)]
    if mode == "flags":
        flags = [new_flags(6, "cuda") for _ in tiles]
        for t, h in enumerate(halos):
            h.sync = FlagSync(t, h.neighbours, flags[t], dict(enumerate(flags)))
    return tiles, LoopbackCluster(tiles, halos=halos, flag_sync=mode == "flags")


@pytest.mark.parametrize("mode", ["packed", "direct"])
def test_cube_halo_matches_oracle(mode):
    import torch

    from oracle.cube import cube_halo
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig(ni=16, nj=16, nk=5, nq=1)
    rng = np.random.default_rng(9)
    states = []
    for t in range(6):
        st = initial_state(RunConfig(ni=16, nj=16, nk=5, nq=1, seed=100 + t))
        for n in NAMES:
            st[n] = rng.uniform(-1, 1, st["delp"].shape)
        states.append(st)
    tiles, cl = _cluster(cfg, states, mode)
    if cl.streams:
        for st in cl.streams:
            st.wait_stream(torch.cuda.current_stream())
    cl.exchange_all([NAMES] * 6)
    if cl.streams:
        for st in cl.streams:
            torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    ref = [{n: states[t][n].copy() for n in NAMES} for t in range(6)]
    cube_halo(ref, NAMES, cfg.ni, cfg.halo)
    for t, d in enumerate(tiles):
        got = d.download(NAMES)
        for n in NAMES:
            assert np.array_equal(got[n], ref[t][n]), (t, n)


@pytest.mark.parametrize("mode,graph", [("packed", False), ("packed", True), ("direct", False), ("direct", True),
                                        ("concurrent", False), ("concurrent", True)])
def test_cube_dycore_matches_oracle_bitwise(mode, graph):
    import torch

    from oracle.cube import OracleCube
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig(ni=24, nj=24, nk=6, n_split=2, dt_atmos=20.0)
    states = [initial_state(RunConfig(ni=24, nj=24, nk=6, seed=2205 + t)) for t in range(6)]
    tiles, cl = _cluster(cfg, [{k: v.copy() for k, v in st.items()} for st in states], mode)
    ref = OracleCube(cfg, states)
    for it in range(3):
        if graph and it == 1:
            cl.capture()  # (after an eager step: kernel attributes and index lists exist)
        cl.replay() if graph and it >= 1 else cl.step()
        ref.step()
    torch.cuda.synchronize()
    h = cfg.halo
    names = ["u", "v", "w", "delp", "pt", "gz", "pef", "q0", "q7", "q3_a4", "mfx", "cy"]
    for t, d in enumerate(tiles):
        got = d.download(names)
        for n in names:
            # the state: interior columns, layer fields on levels < nk (the top
            # slot of ping-pong layer fields is scratch, as in test_gpu_dycore)
            top = cfg.nk + 1 if n in ("gz", "pef") else cfg.nk
            a, b = got[n][h:-h, h:-h, :top], ref.tiles[t].state[n][h:-h, h:-h, :top]
            assert np.isfinite(b).all(), (t, n)
            assert np.array_equal(a, b), (t, n, float(np.max(np.abs(a - b))))


def _cube_worker(tile, port, q):
    """One tile of the cube per process (cuda:0 for all); the neighbours'
    buffers are CUDA-IPC mappings, stores ordered by host barriers."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.cubesphere import CubePeerHalo, topology
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import IpcPeers, ipc_sync
    from paper_2205_04148_b200.state import initial_state

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=tile, world_size=6)
    try:
        torch.cuda.set_device(0)
        cfg = RunConfig(ni=16, nj=16, nk=5, n_split=1, dt_atmos=20.0)
        d = Dycore(cfg, initial_state(RunConfig(ni=16, nj=16, nk=5, seed=2205 + tile)),
                   placement=(True, True, True, True))
        nbrs = sorted({s.nb for s in topology()[tile].values()})
        ipc = IpcPeers(d, None, neighbours=nbrs, rank=tile)
        d.halo = CubePeerHalo(d, tile, ipc.tiles(), sync=ipc_sync())
        dist.barrier()
        d.step()
        torch.cuda.synchronize()
        names = ["u", "v", "w", "delp", "pt", "gz", "q0", "mfx", "cy"]
        h = cfg.halo
        got = d.download(names)
        q.put((tile, {n: got[n][h:-h, h:-h] for n in names}))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_cube_ipc_six_processes_bitwise():
    """The six tiles as six processes (one per GPU on a node; here all on
    cuda:0) exchanging rotated halos by CUDA-IPC peer stores: one FULL_TILE
    step bitwise the oracle cube."""
    import socket

    import torch

    from oracle.cube import OracleCube
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.state import initial_state

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cube_worker, args=(t, port, q)) for t in range(6)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    cfg = RunConfig(ni=16, nj=16, nk=5, n_split=1, dt_atmos=20.0)
    ref = OracleCube(cfg, [initial_state(RunConfig(ni=16, nj=16, nk=5, seed=2205 + t)) for t in range(6)])
    ref.step()
    h = cfg.halo
    for t in range(6):
        for n, got in res[t].items():
            top = cfg.nk + 1 if n == "gz" else cfg.nk
            want = ref.tiles[t].state[n][h:-h, h:-h, :top]
            assert np.array_equal(got[..., :top], want), (t, n)
