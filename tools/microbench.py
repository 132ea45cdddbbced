"""Scratch per-kernel timing at config sizes (not the bench contract)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2205_04148_b200.executor.run import upload
from paper_2205_04148_b200.executor.scheduled import benchmark_uploaded
from paper_2205_04148_b200.inputs import synthetic_inputs
from paper_2205_04148_b200.traffic import compulsory_bytes

CASES = [("copy", (192, 192, 80)), ("fv_tp_2d", (192, 192, 80)), ("fv_tp_2d", (384, 384, 80)),
         ("tracer_2d", (384, 384, 80)), ("nh_d", (192, 192, 81)), ("riem_solver_c", (192, 192, 81))]
if len(sys.argv) > 1:
    CASES = [c for c in CASES if c[0] in sys.argv[1:]]
peak = 6541.8
for name, dom in CASES:
    inp = synthetic_inputs(name, dom, 1)
    up = upload(name, inp, dom, placement=(False,) * 4)
    res = benchmark_uploaded(up, reps=20, warmup=3)
    b = compulsory_bytes(name, dom)
    for node, st in res.kernels.items():
        gbs = b / st.median / 1e9
        print(json.dumps({"program": name, "domain": dom, "node": node, "median_us": round(st.median * 1e6, 2),
                          "min_us": round(st.min * 1e6, 2), "bytes": b, "GBps": round(gbs, 1),
                          "frac": round(gbs / peak, 3)}), flush=True)
