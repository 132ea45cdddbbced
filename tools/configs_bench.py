"""Timings of the BASELINE configs other than the bench workload, on one B200
(CUDA events, warm-up excluded, median of reps).  Writes one JSON line per
config to stdout.

  C1  48x48x16 acoustic substep (halo, c_grid, halo, d_sw, nh_d, halo,
      p_grad_d) on one GPU, doubly periodic — launch-bound;
  C3  cubed sphere C128 L80: six FULL_TILE tiles on one GPU with the
      cubed-sphere halo (rotation, corner fill) moved by device copies
      (parallel.LoopbackCluster) — the per-GPU work of the 6-GPU run;
  C4  768x768x80 doubly periodic full timestep on one GPU (the strong-scaling
      base; split 1x2 / 2x2 / 2x4 gives 768x384 / 384x384 / 384x192 blocks);
  C5  tracer_2d (nq = 8) + the vertical remapping (profile + map1_ppm of the
      8 tracers, pt and w) at 384x384x80.
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.cubesphere import CubeHalo
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.parallel import LoopbackCluster
from paper_2205_04148_b200.state import initial_state


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def c1():
    cfg = RunConfig(ni=48, nj=48, nk=16, n_split=1)
    d = Dycore(cfg, initial_state(cfg))

    def sub():
        d.halo.update(["u", "v", "w", "delp", "pt", "gz"])
        d.c_grid()
        d.halo.update(["uc", "vc"])
        d.d_sw()
        d.nh_d()
        d.halo.update(["pef", "gz"])
        d.p_grad_d()

    ms = timeit(sub, reps=20)
    g = torch.cuda.CUDAGraph()
    sub()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        sub()
    msg = timeit(g.replay, reps=20)
    return {"config": "C1 48x48x16 acoustic substep", "ms_eager": ms, "ms_graph": msg,
            "cells_per_s_graph": 48 * 48 * 16 / (msg * 1e-3)}


def c3(n=128, concurrent=True):
    cfg = RunConfig(ni=n, nj=n, nk=80)
    tiles = [Dycore(cfg, initial_state(RunConfig(ni=n, nj=n, nk=80, seed=2205 + t)), placement=(True,) * 4)
             for t in range(6)]
    cl = LoopbackCluster(tiles, halos=[CubeHalo(d, t, transport=None) for t, d in enumerate(tiles)],
                         concurrent=concurrent)
    ms = timeit(cl.step, reps=3, warm=1)
    cl.capture()
    msg = timeit(cl.replay, reps=5, warm=2)
    cells = 6 * n * n * 80
    return {"config": f"C3 cubed sphere C{n} L80, 6 tiles on 1 GPU (loopback halo{', tiles on concurrent streams' if concurrent else ''})", "ms_per_step_eager": ms,
            "ms_per_step": msg, "ms_per_tile_step": msg / 6, "cells_per_s": cells / (msg * 1e-3)}


def c4(n=768):
    cfg = RunConfig(ni=n, nj=n, nk=80)
    d = Dycore(cfg, initial_state(cfg))
    d.step()
    d.capture()
    ms = timeit(d.replay, reps=3, warm=2)
    return {"config": f"C4 {n}x{n}x80 full timestep on 1 GPU", "ms_per_step": ms, "cells_per_s": cfg.cells / (ms * 1e-3)}


def c5(n=384):
    cfg = RunConfig(ni=n, nj=n, nk=80)
    d = Dycore(cfg, initial_state(cfg))

    def tr():
        d.tracer_2d()
        d.remap()
        d.remap_map()

    ms = timeit(tr, reps=5)
    return {"config": f"C5 tracer_2d (nq=8) + remap (profile + map1_ppm, 10 fields) at {n}x{n}x80", "ms": ms,
            "cells_per_s": cfg.cells / (ms * 1e-3)}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c3", "c4", "c5"]
    for w in which:
        if w == "c3-serial":
            print(json.dumps(c3(concurrent=False)), flush=True)
            continue
        print(json.dumps(globals()[w]()), flush=True)
