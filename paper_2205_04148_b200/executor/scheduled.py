"""Timing API of the reference's missing ``executor.scheduled`` module
(``SPEC.md:366-369`` TimingStats, ``:382-390`` run_scheduled, ``:402-410``
benchmark, ``:427`` CSV).

Per-kernel times are CUDA events recorded on the launching stream around
each launch (device time, not wall clock).  Kernels are keyed by node name
``<stencil>_<block>`` (``ir/graph.py:138-143``); a fused launch carries the
name of its first node.  Repeated invocations are aggregated.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass, field

import torch

from .run import Uploaded, execute, upload


@dataclass
class TimingStats:
    samples: list[float]  # seconds
    reps: int = 0

    @property
    def median(self) -> float:
        return statistics.median(self.samples) if self.samples else float("nan")

    @property
    def min(self) -> float:
        return min(self.samples) if self.samples else float("nan")


@dataclass
class BenchmarkResult:
    kernels: dict[str, TimingStats] = field(default_factory=dict)
    invocations: dict[str, int] = field(default_factory=dict)
    total: TimingStats = field(default_factory=lambda: TimingStats([]))


class _Collector:
    def __init__(self):
        self.events: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    def __call__(self, node, s, e):
        self.events.append((node, s, e))

    def per_node(self) -> dict[str, float]:
        out: dict[str, float] = {}
        for node, s, e in self.events:
            out[node] = out.get(node, 0.0) + s.elapsed_time(e) * 1e-3
        return out


def run_scheduled(program, inputs: dict, domain, workers: int = 1, placement=None):
    """Execute once with per-kernel timing: ``(outputs, {node: TimingStats})``.

    ``workers`` is the host worker count of the reference contract; on the
    device the parallel decomposition is the CUDA grid, so any value >= 1 is
    accepted (``workers < 1`` is an error, ``SPEC.md:386``).
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    up = upload(program, inputs, domain, placement)
    col = _Collector()
    execute(up, on_launch=col)
    torch.cuda.synchronize()
    stats = {n: TimingStats([t], 1) for n, t in col.per_node().items()}
    return up.download(), stats


def benchmark_uploaded(up: Uploaded, reps: int = 10, warmup: int = 1, flush_l2: bool = True) -> BenchmarkResult:
    """Time ``reps`` executions of device-resident state (warm-up excluded).
    Between reps a 256 MiB buffer is overwritten so every rep starts with a
    cold L2 (126 MB)."""
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda") if flush_l2 else None
    for _ in range(warmup):
        execute(up)
    res = BenchmarkResult()
    for _ in range(reps):
        if flush is not None:
            flush.fill_(0.0)
        # keep the GPU busy while the host enqueues the timed launches, so the
        # events bracket device execution only (not Python launch overhead)
        torch.cuda._sleep(1_000_000)
        col = _Collector()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        launched = execute(up, on_launch=col)
        t1.record()
        torch.cuda.synchronize()
        for node, t in col.per_node().items():
            res.kernels.setdefault(node, TimingStats([], 0)).samples.append(t)
            res.kernels[node].reps += 1
        res.invocations = {n: launched.count(n) for n in set(launched)}
        res.total.samples.append(t0.elapsed_time(t1) * 1e-3)
        res.total.reps += 1
    return res


def benchmark(program, inputs: dict, domain, reps: int = 10, placement=None) -> BenchmarkResult:
    """Median-of-reps device timing per kernel and in total (``SPEC.md:402-410``)."""
    if reps < 10:
        raise ValueError("reps must be >= 10 (SPEC.md:366-369)")
    up = upload(program, inputs, domain, placement)
    return benchmark_uploaded(up, reps=reps)


def timings_to_csv(result: BenchmarkResult) -> str:
    """CSV ``kernel,invocations,median_s,min_s`` (``SPEC.md:427``)."""
    lines = ["kernel,invocations,median_s,min_s"]
    for name in sorted(result.kernels):
        st = result.kernels[name]
        lines.append(f"{name},{result.invocations.get(name, 0)},{st.median:.9e},{st.min:.9e}")
    lines.append(f"total,1,{result.total.median:.9e},{result.total.min:.9e}")
    return "\n".join(lines) + "\n"
