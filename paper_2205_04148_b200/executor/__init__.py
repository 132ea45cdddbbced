"""The B200 engine behind the reference's execution API.

Reference slot: ``stencilkit.executor`` declares ``run_reference`` plus the
missing modules ``scheduled`` (``run_scheduled``, ``benchmark``,
``TimingStats``, ``BenchmarkResult``, ``timings_to_csv``) and ``bandwidth``
(``measure_bandwidth``) — ``pkg/src/stencilkit/executor/__init__.py:6-13``,
contracts ``SPEC.md:366-427``.  This package provides those names, backed by
hand-written sm_100a kernels:

* :func:`run_b200` has ``run_reference``'s contract
  (``executor/reference.py:307-339``);
* :func:`run_scheduled`, :func:`benchmark`, :func:`timings_to_csv`,
  :class:`TimingStats`, :class:`BenchmarkResult` follow ``SPEC.md:366-427``;
* :func:`measure_bandwidth` is the copy-stencil HBM probe (``SPEC.md:392-400``).
"""

from .bandwidth import measure_bandwidth
from .run import run_b200, upload
from .scheduled import BenchmarkResult, TimingStats, benchmark, run_scheduled, timings_to_csv

run_reference = run_b200  # drop-in alias for callers that import the reference name

__all__ = [
    "BenchmarkResult",
    "TimingStats",
    "benchmark",
    "measure_bandwidth",
    "run_b200",
    "run_reference",
    "run_scheduled",
    "timings_to_csv",
    "upload",
]
