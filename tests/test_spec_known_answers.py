"""The SPEC's run_reference known answers on the
oracle, and on the live reference where it is importable.  The programs are
tests/golden/spec/*.stn; their manifests (reference front end) are committed
so these run without the reference.  Copy is in test_oracle.py
and, on the device, test_gpu_parity.py."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import _ref
from oracle import interp

SPEC = Path(__file__).resolve().parent / "golden" / "spec"
needs_ref = pytest.mark.skipif(not _ref.available(), reason="reference package not present")


def _doc(name):
    return json.loads((SPEC / f"{name}.json").read_text())


def _ref_run(name, inputs, domain):
    R = _ref.load()
    prog = R.parse_program((SPEC / f"{name}.stn").read_text())
    assert R.validate(prog) == []
    return R.run_reference(prog, inputs, domain, placement=R.RankPlacement(True, True, True, True))


def test_forward_cumulative_sum_known_answer():
    """`a = a[0,0,-1] + inp` over nk = 4 with inp = 1 -> a(k) = k + 1."""
    shapes = interp.input_shapes(_doc("cumsum"), (3, 2, 4))
    inp = np.ones(shapes["inp"])
    out = interp.run_program(_doc("cumsum"), {"inp": inp}, (3, 2, 4))
    assert np.array_equal(out["a"], np.broadcast_to(np.arange(1.0, 5.0), out["a"].shape))


def _tridiag_inputs(domain, seed=7):
    rng = np.random.default_rng(seed)
    shape = interp.input_shapes(_doc("tridiag"), domain)["diag"]
    sub, sup = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)
    diag = 2.5 + rng.uniform(0, 1, shape)  # diagonally dominant
    return {"sub": sub, "diag": diag, "sup": sup, "rhs": rng.uniform(-10, 10, shape)}


def test_tridiagonal_solver_vs_dense_lu():
    """The Thomas solver (FORWARD + BACKWARD stencils) against a dense LU
    solve of the same system per column on 8x8x8: max rel diff <= 1e-12
    (SPEC.md:380)."""
    domain = (8, 8, 8)
    ins = _tridiag_inputs(domain)
    x = interp.run_program(_doc("tridiag"), ins, domain)["x"]
    nk = domain[2]
    worst = 0.0
    for i in range(domain[0]):
        for j in range(domain[1]):
            A = np.diag(ins["diag"][i, j]) + np.diag(ins["sub"][i, j, 1:], -1) + np.diag(ins["sup"][i, j, :-1], 1)
            xd = np.linalg.solve(A, ins["rhs"][i, j])
            worst = max(worst, float(np.max(np.abs(x[i, j] - xd) / np.maximum(np.abs(xd), 1e-300))))
    assert nk == 8 and worst <= 1e-12, worst


def test_smagorinsky_power_rewrite_within_1e12():
    """dt * (divg**2 + tens**2)**0.5 (glibc pow, reference.py:45-53) vs the
    rewrite dt * sqrt(divg*divg + tens*tens) that d_sw.stn uses: <= 1e-12
    relative."""
    domain = (16, 16, 8)
    rng = np.random.default_rng(11)
    shape = interp.input_shapes(_doc("smag_pow"), domain)["divg"]
    ins = {"divg": rng.uniform(-1e-4, 1e-4, shape), "tens": rng.uniform(-1e-4, 1e-4, shape)}
    a = interp.run_program(_doc("smag_pow"), ins, domain)["smag"]
    b = interp.run_program(_doc("smag_rewrite"), ins, domain)["smag"]
    assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= 1e-12


@needs_ref
@pytest.mark.parametrize("name,domain", [("cumsum", (3, 2, 4)), ("tridiag", (8, 8, 8)), ("smag_pow", (6, 5, 3)),
                                         ("smag_rewrite", (6, 5, 3))])
def test_known_answer_programs_oracle_equals_reference(name, domain):
    doc = _doc(name)
    rng = np.random.default_rng(5)
    if name == "tridiag":
        ins = _tridiag_inputs(domain, 5)
    else:
        ins = {n: rng.uniform(0.1, 10, s) for n, s in interp.input_shapes(doc, domain).items()}
    got = interp.run_program(doc, ins, domain)
    ref = _ref_run(name, ins, domain)
    for n in ref:
        assert np.array_equal(got[n], ref[n]), n
