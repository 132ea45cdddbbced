"""Evidence (not a test: minutes of CPU): BASELINE config C2, 10 full
timesteps of the 192 x 192 x 80 doubly periodic domain on the B200 (CUDA-graph
replay) against the CPU oracle running the same global initial state, bitwise
-- north_star's "full-timestep prognostic fields <= 1e-9 after 10 steps" at
the benchmarked size.  The oracle side runs as px x py blocks of the global
state on host processes with the halos exchanged over gloo at every halo point
(DecomposedHalo + DistTransport; tests/test_parallel.py shows the decomposed
oracle step equals the single-domain one bitwise).

    python tools/c2_10step_parity.py [steps]        (on the GPU box)
"""
import os
import socket
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

FIELDS = ["u", "v", "w", "delp", "pt", "gz", "pef", "q0", "q7", "mfx", "cy", "pe", "pk", "pkz", "cvm"]
INTERFACE = ("gz", "pef", "pe", "peln", "pk")


def _block(a, ri, rj, ni, nj, h):
    """Block (ri, rj) of a periodic global array, halo included (wrapped)."""
    NI, NJ = a.shape[0] - 2 * h, a.shape[1] - 2 * h
    ii = (np.arange(ri * ni - h, (ri + 1) * ni + h) % NI) + h
    jj = (np.arange(rj * nj - h, (rj + 1) * nj + h) % NJ) + h
    return a[np.ix_(ii, jj)]


def _rank(rank, world, port, px, py, steps, st, q):
    os.environ.update(OMP_NUM_THREADS="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    from bench import _HostGrid, _HostRank
    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.parallel import DecomposedHalo, DistTransport, TorchPacker

    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = RunConfig()  # C2
        h, ni, nj = g.halo, g.ni // px, g.nj // py
        od = OracleDycore(RunConfig(ni=ni, nj=nj, nk=g.nk), st)
        host = _HostRank(_HostGrid(ni, nj, h))
        halo = DecomposedHalo(host, px, py, rank, transport=DistTransport(rank), packer=TorchPacker(host.grid))
        t0 = time.perf_counter()
        for _ in range(steps):
            for names in od.phases():
                host.cur = {n: torch.from_numpy(st[n]).permute(2, 1, 0) for n in names}
                halo.update(names)
        q.put((rank, time.perf_counter() - t0, {n: st[n][h:-h, h:-h] for n in FIELDS}))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    import torch
    import torch.multiprocessing as mp

    from bench import cpu_tiles
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig()
    glob = initial_state(cfg)
    d = Dycore(cfg, glob)
    d.capture()
    for _ in range(steps):
        d.replay()
    torch.cuda.synchronize()
    gpu = d.download(FIELDS)
    h = cfg.halo

    px, py = cpu_tiles(os.cpu_count() or 1)
    world = px * py
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ni, nj = cfg.ni // px, cfg.nj // py
    blocks = []
    for r in range(world):  # each rank's block of the global state, halo included (wrapped)
        ri, rj = r % px, r // px
        blocks.append({n: np.ascontiguousarray(_block(a, ri, rj, ni, nj, h) if a.ndim == 3 else
                                               _block(a[..., None], ri, rj, ni, nj, h)[..., 0])
                       for n, a in glob.items()})
    del glob
    procs = [ctx.Process(target=_rank, args=(r, world, port, px, py, steps, blocks[r], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, t, out = q.get(timeout=3600)
        res[r] = (t, out)
    for p in procs:
        p.join(timeout=120)
    print(f"C2 192x192x80, {steps} timesteps (n_split=6, nq=8, del6, pt in log pressure): B200 CUDA-graph replay "
          f"vs the CPU oracle as {px}x{py} blocks on {world} host processes (gloo halos), "
          f"{max(t for t, _ in res.values()):.0f} s of CPU")
    worst = 0.0
    for n in FIELDS:
        top = cfg.nk + 1 if n in INTERFACE else cfg.nk
        a = gpu[n][h:-h, h:-h, :top]
        b = np.empty_like(a)
        for r, (_, out) in res.items():
            ri, rj = r % px, r // px
            b[ri * ni:(ri + 1) * ni, rj * nj:(rj + 1) * nj] = out[n][..., :top]
        same = np.array_equal(a, b)
        rel = float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
        worst = max(worst, rel)
        print(f"  {n:5s} bitwise={same}  max rel err {rel:.3e}  finite={bool(np.isfinite(a).all())}")
    print(f"worst max rel err {worst:.3e} (north_star bar 1e-9)")


if __name__ == "__main__":
    main()
