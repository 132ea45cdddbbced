"""bench.py — FV3 dycore timestep throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): one full fp64 dycore timestep of
a doubly periodic 192x192x80 domain per GPU — n_split = 6 acoustic substeps
(c_grid = c_sw + riem_solver_c + p_grad_c, d_sw, nh_d, p_grad_d with their
halo updates), then tracer_2d (nq = 8), remap_tracers and remap_map.  The state
(~1.3 GB) exceeds the 126 MB L2, so no flush is needed between steps.

* ``value``  — grid cells per second over the whole job (N x cells / step
  time), device-resident state, CUDA-graph replay, CUDA events on the
  launching stream, max over ranks.
* ``e2e``    — the same metric through the public API with host buffers:
  each step copies the prognostic state (u, v, w, delp, pt, gz, q0..q7)
  from pinned host memory, runs the step and copies it back
  (``Dycore.step_host``: uploads and downloads on their own streams overlap
  the compute they do not feed, and successive steps pipeline).
* ``roofline`` — the dominant program launch (by device time) against the
  measured HBM copy bandwidth: algorithmic (first-touch compulsory) bytes per
  launch / its mean CUDA-event duration.
* ``cpu_baseline`` — the oracle restatement of the reference CPU path
  (``oracle/``, pinned bitwise against ``run_reference``) on the host cores.

N > 1: one process per GPU (torchrun), weak scaling: every rank owns a
192x192x80 block of a px x py doubly periodic domain (1x2, 2x2, 2x4) and
exchanges halos with its neighbours over NCCL.

``--impl reference`` times the reference CPU path (the oracle port; the
reference is Python and is not shipped to the GPU box) on all host cores on
rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP64_PEAK_OPS = 18.37e12  # measured fp64 op/s of one B200 (profiles/fp64_probe.txt: DFMA 63.2 op/clk/SM)
METRIC = "dycore step grid-cells/s (fp64 FV3 timestep, 192x192x80 per GPU)"
UNIT = "cells/s"


# ---------------------------------------------------------------------------
# CPU path: the oracle restatement of run_reference on host cores
# ---------------------------------------------------------------------------

class _HostGrid:
    """What DecomposedHalo / TorchPacker need from a Grid, for (K, J, I)
    views of the oracle's (I, J, K) state arrays (uniform halo, no pre-pad)."""

    def __init__(self, ni, nj, h):
        self.ni, self.nj, self.halo, self.i0 = ni, nj, h, h


class _HostRank:
    """What DecomposedHalo needs from a Dycore: grid, cur, device."""

    def __init__(self, grid):
        self.grid, self.cur, self.device, self.timer = grid, {}, "cpu", None


def _cpu_rank(rank, world, port, px, py, nk, steps, warmup, q):
    """One host process of the CPU arm: the oracle step on this rank's
    block of the 192x192 domain, the halos exchanged with the neighbour
    blocks over gloo at every halo point (DecomposedHalo + DistTransport)."""
    os.environ.update(OMP_NUM_THREADS="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.parallel import DecomposedHalo, DistTransport, TorchPacker
    from paper_2205_04148_b200.state import initial_state

    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = RunConfig(ni=192 // px, nj=192 // py, nk=nk)
        st = initial_state(cfg)  # the block's own synthetic state (as the GPU ranks of bench.py)
        od = OracleDycore(cfg, st)
        host = _HostRank(_HostGrid(cfg.ni, cfg.nj, cfg.halo))
        halo = DecomposedHalo(host, px, py, rank, transport=DistTransport(rank), packer=TorchPacker(host.grid))
        t0 = None
        for it in range(warmup + steps):
            if it == warmup:  # the timed steps start together
                dist.barrier()
                t0 = time.perf_counter()
            for names in od.phases():
                host.cur = {n: torch.from_numpy(st[n]).permute(2, 1, 0) for n in names}
                halo.update(names)
        dist.barrier()
        q.put((rank, time.perf_counter() - t0))
    finally:
        dist.destroy_process_group()


def cpu_tiles(cores: int, ni=192, nj=192, min_tile=32):
    """Split the domain into at most ``cores`` tiles of >= min_tile cells."""
    best = (1, 1)
    for px in range(1, ni // min_tile + 1):
        for py in range(1, nj // min_tile + 1):
            if px * py <= cores and ni % px == 0 and nj % py == 0 and px * py > best[0] * best[1]:
                best = (px, py)
    return best


def cpu_run(steps: int, nk=80, cores=None, warmup: int = 0):
    """``steps`` C2 timesteps of the whole 192 x 192 x nk doubly periodic
    domain on the host: the oracle (oracle/dycore.py, pinned bitwise to the
    reference's run_reference) on px x py blocks, one process per block,
    halos exchanged between them over gloo at every halo point of the step;
    returns (cells/s, processes, sample)."""
    import socket

    import torch.multiprocessing as mp

    cores = cores or os.cpu_count() or 1
    px, py = cpu_tiles(cores)
    nproc = px * py
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    t0 = time.perf_counter()
    procs = [ctx.Process(target=_cpu_rank, args=(r, nproc, port, px, py, nk, steps, warmup, q)) for r in range(nproc)]
    for p in procs:
        p.start()
    times = dict(q.get(timeout=1800) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    wall = time.perf_counter() - t0
    t = max(times.values())  # between barriers: the job's step time (process start-up excluded)
    cells = 192 * 192 * nk * steps
    sample = (f"{steps} full C2 timestep(s) (n_split=6, nq=8; after {warmup} untimed) of the 192x192x{nk} doubly periodic domain, "
              f"decomposed {px}x{py} into {192 // px}x{192 // py} blocks on {nproc} host processes (one core each), "
              f"halos exchanged over gloo at every halo point; {t:.1f} s between barriers, wall {wall:.1f} s")
    return cells / t, nproc, sample


def run_reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    # each step is one full C2 timestep of the 192x192x80 domain decomposed
    # over the host cores (blocks >= 32x32, gloo halo exchanges); about 7 s
    # per step on 16 cores, so the sample is bounded at 8 timed steps after
    # at most one untimed one (the run ends within a few minutes)
    v, cores, sample = cpu_run(min(K, 8), warmup=min(W, 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": 192 * 192 * 80 / v * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.config == "c2" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_of(args, world),
        "method": {"timing": "host wall clock between barriers, max over the host processes",
                   "engine": "the oracle (NumPy restatement of run_reference, pinned bitwise to it) on the host cores"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            out, _ = self.p.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            c = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(c[0]))
                mx = max(mx, float(c[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, c[3:]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

class LaunchTimer:
    """CUDA events around every libfv3b launch, on the launching stream."""

    def __init__(self):
        import torch

        self.torch = torch
        self.ev = []

    def start(self, node):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev.append([node, e, None])

    def stop(self, node):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[-1][2] = e

    def per_node(self):
        out = {}
        for n, a, b in self.ev:
            out.setdefault(n, []).append(a.elapsed_time(b) * 1e-3)
        return out


def workload_of(args, world: int) -> dict:
    """The line's ``config``: the workload of a bench config at ``world``
    ranks (shared by both arms, so their configs are the same dict)."""
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.parallel import grid_shape

    l2 = "state > 126 MB L2 per GPU (no flush)"
    if args.config == "c3":
        n, nk = args.c3_n, args.nk
        cfg = RunConfig(ni=n, nj=n, nk=nk)
        return {"workload": f"C3 cubed sphere C{n} L{nk}, 6 FULL_TILE tiles, edge rotation + corner fill (n_split=6, nq=8)",
                "name": "c3", "ni": n, "nj": n, "nk": nk, "n_split": cfg.n_split, "nq": cfg.nq,
                "decomposition": "6 tiles on 1 GPU" if world == 1 else "6 tiles on 6 GPUs", "l2": l2}
    px, py = grid_shape(world)
    if args.config == "c4":
        N = args.c4_n
        cfg = RunConfig(ni=N // px, nj=N // py, nk=args.nk)
        workload = f"C4 doubly periodic {N}x{N}x{args.nk} fp64 dycore timestep split {px}x{py} (n_split=6, nq=8)"
    else:
        cfg = RunConfig(ni=args.ni, nj=args.ni, nk=args.nk)
        workload = f"C2 doubly periodic {args.ni}x{args.ni}x{args.nk} fp64 dycore timestep per GPU (n_split=6, nq=8)"
    return {"workload": workload, "name": args.config, "ni": cfg.ni, "nj": cfg.nj, "nk": cfg.nk,
            "n_split": cfg.n_split, "nq": cfg.nq, "decomposition": f"{px}x{py}", "l2": l2}


class Setup:
    """What one rank runs for a bench config: ``runner`` (step / capture /
    replay: a Dycore, or a LoopbackCluster of cube tiles), its Dycores,
    the job's cells per step and the line's config fields."""

    def __init__(self, runner, dycores, cells_job, scaling, workload, decomposition, halo, graphs, sync=None):
        self.runner, self.dycores, self.cells_job = runner, dycores, cells_job
        self.scaling, self.workload, self.decomposition, self.halo = scaling, workload, decomposition, halo
        self.graphs, self.sync = graphs, sync


def setup_config(args, rank: int, world: int) -> Setup:
    """C2 (default): 192x192x80 per rank, px x py weak scaling.  C4: the
    768x768x80 domain split px x py (strong scaling: 768x384, 384x384,
    384x192 blocks at 2, 4, 8 ranks).  C3: the C128 L80 cubed sphere, one
    FULL_TILE tile per rank at 6 ranks, or all six tiles on one GPU
    (LoopbackCluster).  Every block starts from the synthetic state of its
    own shape (state.py): the same work per cell as the global field's
    block."""
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import (DecomposedHalo, HaloPlan, IpcPeers, LoopbackCluster, PeerHalo,
                                                grid_shape, new_flags)
    from paper_2205_04148_b200.state import initial_state

    if args.config == "c3":
        from paper_2205_04148_b200.cubesphere import CubeHalo, CubePeerHalo, topology

        n, nk = args.c3_n, args.nk
        cfg = RunConfig(ni=n, nj=n, nk=nk)
        workload = f"C3 cubed sphere C{n} L{nk}, 6 FULL_TILE tiles, edge rotation + corner fill (n_split=6, nq=8)"
        if world == 1:
            tiles = [Dycore(cfg, initial_state(RunConfig(ni=n, nj=n, nk=nk, seed=2205 + t)), placement=(True,) * 4)
                     for t in range(6)]
            cl = LoopbackCluster(tiles, halos=[CubeHalo(d, t, transport=None) for t, d in enumerate(tiles)],
                                 concurrent=True)  # (the six tiles' kernels share the GPU)
            return Setup(cl, tiles, 6 * cfg.cells, "strong", workload, "6 tiles on 1 GPU",
                         "cube rotation + corner fill, device copies (loopback)", True)
        if world != 6:
            raise SystemExit("--config c3 runs on 1 GPU (six tiles) or 6 ranks (one tile each)")
        d = Dycore(cfg, initial_state(RunConfig(ni=n, nj=n, nk=nk, seed=2205 + rank)), placement=(True,) * 4)
        sync = None
        if args.halo == "peer":
            nbrs = sorted({x.nb for x in topology()[rank].values()})
            ipc = IpcPeers(d, None, neighbours=nbrs, rank=rank, flags=new_flags(world, "cuda"))
            sync = ipc.flag_sync()
            d.halo = CubePeerHalo(d, rank, ipc.tiles(), sync=sync)
            halo = "cube rotation + corner fill by peer-memory stores (CUDA IPC) + device barriers"
        else:
            d.halo = CubeHalo(d, rank)
            halo = "cube rotation + corner fill over NCCL send/recv"
        return Setup(d, [d], 6 * cfg.cells, "strong", workload, "6 tiles on 6 GPUs", halo, args.halo == "peer", sync)

    px, py = grid_shape(world)
    if args.config == "c4":
        N = args.c4_n
        if N % px or N % py:
            raise SystemExit(f"--config c4: {N} does not split {px}x{py}")
        cfg = RunConfig(ni=N // px, nj=N // py, nk=args.nk)
        cells_job, scaling = N * N * args.nk, "strong"
        workload = f"C4 doubly periodic {N}x{N}x{args.nk} fp64 dycore timestep split {px}x{py} (n_split=6, nq=8)"
    else:
        cfg = RunConfig(ni=args.ni, nj=args.ni, nk=args.nk)
        cells_job, scaling = cfg.cells * world, "weak"
        workload = (f"C2 doubly periodic {args.ni}x{args.ni}x{args.nk} fp64 dycore timestep per GPU "
                    f"(n_split=6, nq=8)")
    d = Dycore(cfg, initial_state(cfg))
    sync = None
    if world > 1 and args.halo == "peer":
        # halos stored straight into the neighbours' buffers (CUDA IPC over
        # NVLink, fv3b_halo_peer_rects) behind device-side neighbour
        # barriers (fv3b_peer_barrier): no host sync, so whole steps replay
        # as CUDA graphs on every rank
        peers = IpcPeers(d, HaloPlan(cfg.ni, cfg.nj, cfg.halo, px, py, rank), flags=new_flags(world, "cuda"))
        sync = peers.flag_sync()
        d.halo = PeerHalo(d, px, py, rank, peers, sync=sync)
        halo = "peer-memory stores over CUDA IPC + device barriers"
    elif world > 1:
        # every rank owns one block of a (px ni) x (py nj) doubly periodic
        # domain; halos move over NCCL (grouped send/recv)
        d.halo = DecomposedHalo(d, px, py, rank)
        halo = "NCCL send/recv"
    else:
        halo = "periodic kernel"
    return Setup(d, [d], cells_job, scaling, workload, f"{px}x{py}", halo, world == 1 or args.halo == "peer", sync)


def run_ours(args, rank: int, world: int, local: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2205_04148_b200 import _lib
    from paper_2205_04148_b200.dycore import kernels_per_step
    from paper_2205_04148_b200 import perf_model

    torch.cuda.set_device(local)
    _lib.lib()  # no CPU fallback: fail loudly if the library is missing
    su = setup_config(args, rank, world)
    runner, dycores = su.runner, su.dycores
    d = dycores[0]
    cfg = d.cfg
    overlap = args.overlap == "on" or (args.overlap == "auto" and world > 1)
    for x in dycores:
        x.overlap = overlap and len(dycores) == 1
    torch.cuda.synchronize()
    # single rank, loopback clusters and peer halos: whole timesteps replayed
    # as CUDA graphs; NCCL halos: eager launches (exchanges outside capture)
    graphs = su.graphs
    run_step = runner.replay if graphs else runner.step

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (eager, then capture and replay)
    runner.step()
    if graphs:
        runner.capture()
    for _ in range(max(args.warmup, 3)):
        run_step()
    barrier()

    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        t0.record(stream)
        for _ in range(args.steps):
            run_step()
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1) / args.steps
    clocks = clk.summary()
    if su.sync is not None:
        su.sync.check()  # a timed-out neighbour barrier voids the run instead of reporting it

    # end to end: pinned host state in, step, host state out.  One Dycore:
    # Dycore.step_host (uploads and downloads on their own streams, the
    # tracers' uploads overlap the acoustic substeps, the dynamics fields'
    # downloads overlap tracer advection and remapping, successive steps
    # pipeline).  A cube cluster: every tile's upload, the lockstep step,
    # every tile's download, in stream order.
    from paper_2205_04148_b200.state import initial_state as _init
    h_in = [x.host_buffers() for x in dycores]
    h_out = [x.host_buffers() for x in dycores]
    for x, hb in zip(dycores, h_in):
        st0 = _init(x.cfg)
        for n, t in hb.items():
            t.copy_(torch.from_numpy(st0[n]))

    def e2e_step(hi, ho):
        if len(dycores) == 1:
            return dycores[0].step_host(hi[0], ho[0])
        for x, hb in zip(dycores, hi):
            x.load_host(hb)
        runner.step()
        for x, hb in zip(dycores, ho):
            x.store_host(hb)
        return torch.cuda.current_stream().record_event()

    e2e_step(h_in, h_out)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        done = e2e_step(h_in, h_out)
    stream.wait_event(done)  # the last step's downloads are inside the timed region
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    io_bytes = sum(t.numel() * t.element_size() for hb in h_in for t in hb.values())
    up_bytes = io_bytes
    if len(dycores) == 1:  # step_host: the refreshed fields' input halos stay on the host
        up_bytes, io_bytes = dycores[0].host_io_bytes(h_in[0])
    assert all(bool(torch.isfinite(t).all()) for hb in h_out for t in hb.values()), "non-finite state after e2e"
    # chained integration: every step's input is the previous step's output,
    # so a step's uploads wait for the previous downloads (no cross-step overlap)
    h_a, h_b = h_in, h_out
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        done = e2e_step(h_a, h_b)
        h_a, h_b = h_b, h_a
    stream.wait_event(done)
    e1.record(stream)
    barrier()
    e2e_chained_ms = e0.elapsed_time(e1) / args.steps

    # per-launch device times: the same K steps eagerly with events around
    # every libfv3b launch on the launching stream
    timer = LaunchTimer()
    for x in dycores:
        x.timer, x.launches = timer, 0
    barrier()
    for x in dycores:
        x.load(_init(x.cfg))
    for _ in range(args.steps):
        runner.step()
    barrier()
    eager_launches = sum(x.launches for x in dycores)
    per_node = timer.per_node()
    for x in dycores:
        x.timer = None

    def reduce_max(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = reduce_max(ms)
    e2e_ms = reduce_max(e2e_ms)
    e2e_chained_ms = reduce_max(e2e_chained_ms)
    if rank != 0:
        return

    cells = su.cells_job
    value = cells / (ms * 1e-3)
    node_total = {n: sum(v) for n, v in per_node.items()}
    # the Fig. 10 model-augmented report (perf_model): first-touch compulsory
    # bytes per launch / measured peak HBM bandwidth vs the CUDA-event times
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    nk_prog = {"c_grid": cfg.nk + 1, "nh_d": cfg.nk + 1, "p_grad_d": cfg.nk + 1, "remap_tracers": cfg.nk + 1}
    progs = [n for n in per_node if n != "halo"]
    doms = {n: (cfg.ni, cfg.nj, nk_prog.get(n, cfg.nk)) for n in progs}
    # the remapping: the profile launch covers the scalars and the winds, the
    # mapping runs as the scalars' and the winds' launches
    if "remap_map" in doms:
        doms["remap_map"] = (cfg.ni, cfg.nj, cfg.nk + 1, len(cfg.remap_linear()))
    if "remap_map_winds" in doms:  # u, v (and pt in log pressure)
        doms["remap_map_winds"] = (cfg.ni, cfg.nj, cfg.nk + 1, 2 + int(cfg.pt_logp))
    if "moist_pk" in doms:
        doms["moist_pk"] = (cfg.ni, cfg.nj, cfg.nk + 1, len(cfg.moist_names()))
    if "remap_tracers" in doms:
        doms["remap_tracers"] = (cfg.ni, cfg.nj, cfg.nk + 1, len(cfg.remapped()) + 2)
    report = perf_model.build_report({n: per_node[n] for n in progs}, doms, peak * 1e9)
    by = {e.kernel: e for e in report.entries}
    top = max(progs, key=lambda n: node_total[n])
    algo = by[top].unique_bytes
    mean_launch = statistics.mean(per_node[top])
    achieved = algo / mean_launch / 1e9
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(top)
    step_bytes = sum(by[n].unique_bytes * len(per_node[n]) for n in progs) / args.steps
    # the compute-side roof of the same kernel: fp64 thread operations per
    # launch (ncu DADD + DMUL + DFMA, profiles/fp64.json via
    # tools/traffic_from_ncu.py) / its mean launch time, against the fp64
    # issue peak measured on the box (tools/fp64_probe.cu, profiles/fp64_probe.txt)
    fp64 = None
    ff = ROOT / "profiles" / "fp64.json"
    if ff.exists() and json.loads(ff.read_text()).get(top):
        ops = json.loads(ff.read_text())[top]
        fp64_peak = FP64_PEAK_OPS * torch.cuda.get_device_properties(0).multi_processor_count / 148
        fp64 = {"kernel": top, "ops_per_launch": ops, "achieved": ops / mean_launch / 1e12,
                "peak": fp64_peak / 1e12, "unit": "Top/s", "frac": ops / mean_launch / fp64_peak,
                "source": "ncu op counts (profiles/fp64.json) / CUDA-event launch time; peak: "
                          "tools/fp64_probe.cu DFMA issue (profiles/fp64_probe.txt)"}
        # the program's own arithmetic (tools/opcount.py: each .stn operation
        # once per point, a division counted once), beside the executed count
        tab = json.loads((ROOT / "paper_2205_04148_b200" / "traffic_table.json").read_text())
        alg = tab.get(f"{top}@{doms[top][0]}x{doms[top][1]}x{doms[top][2]}", {}).get("algorithmic_ops")
        if alg:
            fp64.update({"algorithmic_ops_per_launch": alg["fp64_ops"], "algorithmic_divisions": alg.get("div", 0),
                         "algorithmic_frac": alg["fp64_ops"] / mean_launch / fp64_peak,
                         "executed_over_algorithmic": ops / alg["fp64_ops"]})
    # per program: the fraction of each roof (HBM: first-touch bytes; fp64
    # issue: ncu-executed DADD + DMUL + DFMA per launch, profiles/fp64.json)
    # and the binding one (the larger fraction)
    executed = json.loads(ff.read_text()) if ff.exists() else {}
    fp64_pk = FP64_PEAK_OPS * torch.cuda.get_device_properties(0).multi_processor_count / 148

    def binding_roof(kernel, t, hbm_frac):
        ops = executed.get(kernel)
        if not isinstance(ops, (int, float)) or t <= 0:
            return {}
        f = ops / t / fp64_pk
        return {"fp64_executed_frac": round(f, 4), "binding": "fp64 issue" if f > hbm_frac else "hbm",
                "binding_frac": round(max(f, hbm_frac), 4)}

    cpu = None
    if not args.no_cpu and world == 1 and args.config == "c2":
        v, cores, sample = cpu_run(1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": su.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded analytic state, state.py)",
        "config": workload_of(args, world),
        "method": {"halo": su.halo, "halo_overlap": overlap and len(dycores) == 1,
                   "timing": ("CUDA-graph replay of whole timesteps" if graphs else "eager launches, NCCL halo exchange") + ", CUDA events, max over ranks"},
        "e2e": {"value": cells / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": up_bytes, "d2h_bytes_per_step": io_bytes,
                "mode": "pipelined: the same host input every step, so step n+1's uploads overlap step n",
                "chained": {"value": cells / (e2e_chained_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_chained_ms,
                            "mode": "each step's input is the previous step's output (uploads wait for the downloads)"}},
        "gpu_launches": kernels_per_step(cfg) * args.steps * len(dycores),
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "algo_bytes_per_launch": algo,
                     "mean_launch_s": mean_launch, "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)",
                     "algo_bytes_source": by[top].source,
                     "movement_model_bytes_per_launch": perf_model.movement_bytes(top, doms[top]),
                     "step_algo_bytes": step_bytes, "step_frac": step_bytes / (ms * 1e-3) / 1e9 / peak},
        "fp64_roofline": fp64,
        "report": {e.kernel: {"invocations_per_step": e.invocations // args.steps,
                              "measured_us": round(e.measured_time * 1e6, 2),
                              "bound_us": round(e.bound_time * 1e6, 2),
                              "utilization": round(e.utilization, 4),
                              **binding_roof(e.kernel, e.measured_time, e.utilization),
                              "first_touch_bytes": e.unique_bytes,
                              "movement_model_bytes": perf_model.movement_bytes(e.kernel, doms[e.kernel])}
                   for e in report.entries},
        "hotspots": perf_model.hotspot_list(report, 3),
        "kernels_ms_per_step": {n: round(v * 1e3 / args.steps, 4) for n, v in
                                sorted(node_total.items(), key=lambda x: -x[1])},
        "eager_launches_per_step": eager_launches / args.steps,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c2", "c3", "c4"), default="c2",
                    help="c2: 192x192x80 per GPU (weak scaling, the BASELINE metric's workload); c3: the C128 L80 "
                         "cubed sphere (1 GPU: six tiles; 6 GPUs: a tile each); c4: 768x768x80 split over the GPUs")
    ap.add_argument("--c3-n", type=int, default=128)
    ap.add_argument("--c4-n", type=int, default=768)
    ap.add_argument("--ni", type=int, default=192)
    ap.add_argument("--nk", type=int, default=80)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--halo", choices=("nccl", "peer"), default="nccl",
                    help="N > 1 halo transport: NCCL send/recv, or peer-memory stores over CUDA IPC")
    ap.add_argument("--overlap", choices=("auto", "on", "off"), default="auto",
                    help="halo exchanges on their own stream, overlapped with compute (Dycore.step_overlapped); "
                         "auto: on for N > 1 (at N = 1 the periodic fill is a few us per update and the stream "
                         "fork / join costs more: 7.96 vs 7.93 ms, r2)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1 and os.environ.get("FV3B_SAME_GPU") == "1":
        # functional check of the N > 1 code paths on a one-GPU box: every
        # rank on cuda:0 (contexts time-slice; no timing meaning), gloo
        import torch.distributed as dist

        local = 0
        dist.init_process_group("gloo")
    elif world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        run_ours(args, rank, world, local)
        if world > 1:  # peers' IPC mappings stay valid until every rank is done
            import torch.distributed as dist

            dist.barrier()
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
