"""Generate the golden fixtures from the REFERENCE interpreter.

Runs in the build container only: imports ``stencilkit`` through
``tests/_ref.py`` and executes each shipped ``.stn`` program with the
reference ``run_reference`` (``executor/reference.py:307-339``) on seeded
synthetic inputs at small domains.  Inputs and outputs are saved as
``tests/golden/<program>__<case>.npz``; the oracle tests and the GPU parity
tests compare against them.

Usage: ``python tests/golden/make_golden.py``
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import _ref  # noqa: E402

from paper_2205_04148_b200.inputs import synthetic_inputs  # noqa: E402
from paper_2205_04148_b200.program import PROGRAM_DIR  # noqa: E402

# (program, case, domain, placement, seed)
CASES = [
    ("copy", "periodic", (12, 10, 3), (False, False, False, False), 7),
    ("fv_tp_2d", "periodic", (16, 14, 3), (False, False, False, False), 7),
    ("fv_tp_2d", "tile", (17, 15, 2), (True, True, True, True), 11),
    ("tracer_2d", "periodic", (14, 16, 2), (False, False, False, False), 7),
    ("riem_solver_c", "column", (5, 4, 17), (True, True, True, True), 7),
    ("remap_profile", "column", (5, 4, 17), (True, True, True, True), 7),
    ("remap_tracers", "column", (3, 2, 9), (True, True, True, True), 7),
    ("c_sw", "periodic", (14, 13, 2), (False, False, False, False), 7),
    ("c_sw", "tile", (13, 14, 2), (True, True, True, True), 8),
    ("c_grid", "tile", (13, 12, 5), (True, True, True, True), 7),
    ("d_sw", "periodic", (17, 16, 2), (False, False, False, False), 7),
    ("d_sw", "tile", (16, 17, 2), (True, True, True, True), 9),
    ("nh_d", "column", (5, 4, 17), (True, True, True, True), 7),
    ("p_grad_d", "periodic", (7, 6, 5), (False, False, False, False), 7),
]


def main(only: set[str] | None = None) -> None:
    ref = _ref.load()
    index = {}
    for prog_name, case, domain, placement, seed in CASES:
        if only and prog_name not in only:
            continue
        prog = ref.parse_program((PROGRAM_DIR / f"{prog_name}.stn").read_text())
        assert ref.validate(prog) == []
        inputs = synthetic_inputs(prog_name, domain, seed)
        out = ref.run_reference(prog, inputs, domain, placement=ref.RankPlacement(*placement))
        path = HERE / f"{prog_name}__{case}.npz"
        np.savez_compressed(path, **{f"in__{k}": v for k, v in inputs.items()},
                            **{f"out__{k}": v for k, v in out.items()})
        index[f"{prog_name}__{case}"] = {"program": prog_name, "domain": list(domain),
                                         "placement": list(placement), "seed": seed}
        print(path.name, f"{path.stat().st_size / 1024:.0f} KiB")
    idx_path = HERE / "index.json"
    old = json.loads(idx_path.read_text()) if idx_path.exists() else {}
    old.update(index)
    idx_path.write_text(json.dumps(old, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
