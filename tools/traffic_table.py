"""Bytes per launch of every dycore program at the bench sizes:

* first-touch compulsory bytes by brute force: the oracle interpreter with
  the FirstTouch recorder (the reference AccessRecorder rule) on seeded
  inputs -- the roofline's algorithmic bytes;
* the reference's own per-node movement model (the paper's method):
  ``trace_movement(lower(program))`` (reference ir/movement.py:64-74), as
  all containers (each stencil node an unfused kernel: temporaries move
  through memory) and as the non-transient containers only.  Needs the
  reference (this container); the values are committed in the table.

Writes paper_2205_04148_b200/traffic_table.json, which bench.py reports.

    python tools/traffic_table.py [ni] [--movement-only]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from oracle import interp  # noqa: E402
from paper_2205_04148_b200.inputs import synthetic_inputs  # noqa: E402
from paper_2205_04148_b200.traffic import compulsory_bytes  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
ni = int(args[0]) if args else 192
nk = 80
PROGS = [("c_grid", nk + 1), ("d_sw", nk), ("nh_d", nk + 1), ("p_grad_d", nk + 1), ("tracer_2d", nk),
         ("remap_tracers", nk + 1)]
out_path = ROOT / "paper_2205_04148_b200" / "traffic_table.json"
table = json.loads(out_path.read_text()) if out_path.exists() else {}


def movement(name, dom):
    """(all containers, non-transient) bytes of the reference trace_movement."""
    import _ref
    from paper_2205_04148_b200.program import PROGRAM_DIR

    R = _ref.load()
    from stencilkit.ir.lower import lower
    from stencilkit.ir.movement import trace_movement

    g = lower(R.parse_program((PROGRAM_DIR / f"{name}.stn").read_text()), dom, R.RankPlacement(False, False, False, False))
    tm = trace_movement(g)
    total = sum(r + w for r, w in tm.values())
    persistent = sum(r + w for n, (r, w) in tm.items() if not g.arrays[n].transient)
    return total, persistent


for name, k in PROGS:
    dom = (ni, ni, k)
    key = f"{name}@{ni}x{ni}x{k}"
    t = time.time()
    row = table.get(key, {})
    if "--movement-only" not in sys.argv:
        rec = interp.FirstTouch()
        interp.run_program(name, synthetic_inputs(name, dom, 1), dom, interp.PERIODIC, recorder=rec)
        row.update({"first_touch_bytes": rec.bytes(), "box_model_bytes": compulsory_bytes(name, dom),
                    "cells": ni * ni * nk})
    total, persistent = movement(name, dom)
    row.update({"movement_model_bytes": total, "movement_model_nontransient_bytes": persistent})
    table[key] = row
    print(name, dom, row, f"{time.time() - t:.1f}s", flush=True)
    out_path.write_text(json.dumps(table, indent=1, sort_keys=True) + "\n")
