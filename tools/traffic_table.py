"""First-touch compulsory bytes of every dycore program at the
bench sizes, by brute force: the oracle interpreter with the FirstTouch
recorder (the reference AccessRecorder rule) on seeded inputs.  Writes
paper_2205_04148_b200/traffic_table.json, which bench.py uses for the
roofline's algorithmic bytes.

    python tools/traffic_table.py [ni]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import interp  # noqa: E402
from paper_2205_04148_b200.inputs import synthetic_inputs  # noqa: E402
from paper_2205_04148_b200.traffic import compulsory_bytes  # noqa: E402

ni = int(sys.argv[1]) if len(sys.argv) > 1 else 192
nk = 80
PROGS = [("c_grid", nk + 1), ("d_sw", nk), ("nh_d", nk + 1), ("p_grad_d", nk + 1), ("tracer_2d", nk),
         ("remap_tracers", nk + 1)]
out_path = ROOT / "paper_2205_04148_b200" / "traffic_table.json"
table = json.loads(out_path.read_text()) if out_path.exists() else {}
for name, k in PROGS:
    dom = (ni, ni, k)
    t = time.time()
    rec = interp.FirstTouch()
    interp.run_program(name, synthetic_inputs(name, dom, 1), dom, interp.PERIODIC, recorder=rec)
    b = rec.bytes()
    table[f"{name}@{ni}x{ni}x{k}"] = {"first_touch_bytes": b, "box_model_bytes": compulsory_bytes(name, dom),
                                       "cells": ni * ni * nk}
    print(name, dom, b, compulsory_bytes(name, dom), f"{time.time() - t:.1f}s", flush=True)
    out_path.write_text(json.dumps(table, indent=1, sort_keys=True) + "\n")
