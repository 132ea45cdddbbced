"""Is the column solver latency-bound?  Time riem_solver_c (one launch) at
1x, 2x and 4x the C2 column count: if 4x the columns take much less than 4x
the time, each SM has idle issue slots that more warps per column would fill."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_04148_b200.executor.scheduled import benchmark
from paper_2205_04148_b200.inputs import synthetic_inputs

for ni, nj in [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or ((192, 192), (384, 192), (384, 384)):
    dom = (ni, nj, 81)
    r = benchmark("riem_solver_c", synthetic_inputs("riem_solver_c", dom, 1), dom, reps=10)
    print(ni * nj, "columns:", {k: round(v.median * 1e6, 1) if hasattr(v, "median") else v for k, v in r.kernels.items()}, "us")
