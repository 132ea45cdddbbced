"""Manifests of the SPEC known-answer programs, made
with the reference front end (tools/gen_programs.manifest: parse_program,
validate == [], compute_requirements, resolve_driver) so the oracle can run
them anywhere.  Build container only: python tests/golden/spec/make_spec.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "tools"))

PROGRAMS = {
    # SPEC.md:379 forward cumulative-sum solver
    "cumsum": """
field inp : float64 [I, J, K]
field a : float64 [I, J, K]

stencil cumsum:
    with computation(FORWARD), interval(0, 1):
        a = inp
    with computation(FORWARD), interval(1, None):
        a = a[0, 0, -1] + inp

driver:
    cumsum()
""",
    # SPEC.md:380 tridiagonal solver (Thomas algorithm as a FORWARD and a BACKWARD stencil)
    "tridiag": """
field sub : float64 [I, J, K]
field diag : float64 [I, J, K]
field sup : float64 [I, J, K]
field rhs : float64 [I, J, K]
field x : float64 [I, J, K]
field cp : float64 [I, J, K] temporary
field dp : float64 [I, J, K] temporary

stencil thomas_fwd:
    with computation(FORWARD), interval(0, 1):
        cp = sup / diag
        dp = rhs / diag
    with computation(FORWARD), interval(1, None):
        cp = sup / (diag - sub * cp[0, 0, -1])
        dp = (rhs - sub * dp[0, 0, -1]) / (diag - sub * cp[0, 0, -1])

stencil thomas_bwd:
    with computation(BACKWARD), interval(-1, None):
        x = dp
    with computation(BACKWARD), interval(0, -1):
        x = dp - cp * x[0, 0, 1]

driver:
    thomas_fwd()
    thomas_bwd()
""",
    # SPEC.md:390 / PAPER.md:532-537 Smagorinsky coefficient, ** form and its rewrite
    "smag_pow": """
const dt = 15.0
field divg : float64 [I, J, K]
field tens : float64 [I, J, K]
field smag : float64 [I, J, K]

stencil smagorinsky:
    with computation(PARALLEL), interval(...):
        smag = dt * (divg ** 2.0 + tens ** 2.0) ** 0.5

driver:
    smagorinsky()
""",
    "smag_rewrite": """
const dt = 15.0
field divg : float64 [I, J, K]
field tens : float64 [I, J, K]
field smag : float64 [I, J, K]

stencil smagorinsky:
    with computation(PARALLEL), interval(...):
        smag = dt * sqrt(divg * divg + tens * tens)

driver:
    smagorinsky()
""",
}


def main() -> None:
    import _ref
    from gen_programs import manifest

    ref = _ref.load()
    for name, text in PROGRAMS.items():
        (HERE / f"{name}.stn").write_text(text.lstrip())
        doc = manifest(name, text, ref)
        (HERE / f"{name}.json").write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
        print(name, doc["requirements"]["min_domain"])


if __name__ == "__main__":
    main()
