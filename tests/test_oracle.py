"""Pin the CPU oracle (oracle/interp.py) to the reference interpreter.

* against the golden fixtures produced by the reference ``run_reference``
  (tests/golden/make_golden.py) — always runs;
* against the live reference on every shipped program and on seeded random
  two-stencil chains (the pattern of ``pkg/tests/test_extents.py:187-221``)
  — only where the reference is importable (this container).
"""

from __future__ import annotations

import numpy as np
import pytest

import _ref
from helpers import assert_outputs_equal, golden_cases, load_golden
from oracle import interp


@pytest.mark.parametrize("key,meta", list(golden_cases()))
def test_oracle_matches_golden_bitwise(key, meta):
    inputs, ref_out = load_golden(key)
    got = interp.run_program(meta["program"], inputs, meta["domain"], interp.Placement(*meta["placement"]))
    assert_outputs_equal(got, ref_out)


@pytest.mark.parametrize("key,meta", list(golden_cases()))
def test_oracle_whole_block_shortcut_is_exact(key, meta):
    inputs, ref_out = load_golden(key)
    got = interp.run_program(meta["program"], inputs, meta["domain"], interp.Placement(*meta["placement"]),
                             whole_blocks=False)
    assert_outputs_equal(got, ref_out)


def test_oracle_shape_error_like_reference():
    key, meta = next(golden_cases("fv_tp_2d"))
    inputs, _ = load_golden(key)
    inputs["q"] = inputs["q"][1:]
    with pytest.raises(ValueError, match="has shape"):
        interp.run_program("fv_tp_2d", inputs, meta["domain"])


def test_oracle_missing_inputs_are_zero():
    out = interp.run_program("copy", {}, (4, 4, 2))
    assert np.all(out["out"] == 0.0) and out["out"].shape == (4, 4, 2)


def test_spec_known_answer_copy():
    rng = np.random.default_rng(3)
    inp = rng.uniform(0.1, 10, (8, 8, 8))
    out = interp.run_program("copy", {"inp": inp}, (8, 8, 8))
    assert np.array_equal(out["out"], inp)


needs_ref = pytest.mark.skipif(not _ref.available(), reason="reference package not present (GPU host)")


@needs_ref
@pytest.mark.parametrize("name", ["copy", "fv_tp_2d", "tracer_2d", "riem_solver_c", "remap_profile", "c_sw",
                                  "c_grid", "d_sw", "nh_d", "p_grad_d"])
def test_oracle_matches_live_reference(name):
    from paper_2205_04148_b200.inputs import synthetic_inputs
    from paper_2205_04148_b200.program import PROGRAM_DIR

    ref = _ref.load()
    prog = ref.parse_program((PROGRAM_DIR / f"{name}.stn").read_text())
    cases = [((15, 17, 3), (False,) * 4, 1), ((16, 16, 2), (True,) * 4, 2)]
    if name.startswith(("riem", "remap", "nh_d")):
        cases = [((4, 3, 12), (True,) * 4, 1), ((3, 3, 30), (False,) * 4, 2)]
    elif name in ("c_grid", "d_sw"):
        cases = [((17, 16, 5), (False,) * 4, 1), ((16, 17, 4), (True,) * 4, 2)]
    for domain, placement, seed in cases:
        inputs = synthetic_inputs(name, domain, seed)
        a = ref.run_reference(prog, inputs, domain, placement=ref.RankPlacement(*placement))
        b = interp.run_program(name, inputs, domain, interp.Placement(*placement))
        assert_outputs_equal(b, a)


def _random_chain_src(rng):
    offs1 = [tuple(int(x) for x in rng.integers(-3, 4, 3)) for _ in range(rng.integers(1, 4))]
    offs2 = [(int(rng.integers(-3, 4)), int(rng.integers(-3, 4)), 0) for _ in range(rng.integers(1, 4))]
    extra = tuple(int(x) for x in rng.integers(-3, 4, 3))
    ops = ["+", "-", "*", "/"]
    r1 = f" {ops[rng.integers(0, 4)]} ".join(f"inp[{a}, {b}, {c}]" for a, b, c in offs1)
    r2 = " + ".join(f"tmp[{a}, {b}, {c}]" for a, b, c in offs2)
    pol = ["PARALLEL", "FORWARD", "BACKWARD"][rng.integers(0, 3)]
    return (
        "field inp : float64 [I, J, K]\n"
        "field aux : float64 [I, J]\n"
        "field tmp : float64 [I, J, K] temporary\n"
        "field out : float64 [I, J, K]\n"
        "stencil s1:\n"
        f"    with computation({pol}), interval(...):\n"
        f"        tmp = {r1}\n"
        "stencil s2:\n"
        "    with computation(PARALLEL), interval(...):\n"
        f"        out = select({r2} > aux[{extra[0]}, {extra[1]}], sqrt(abs({r2})), min(aux, {r2}))\n"
        "driver:\n"
        "    s1()\n"
        "    s2()\n"
    )


@needs_ref
def test_oracle_matches_reference_on_random_chains():
    from paper_2205_04148_b200.program import canonicalize

    ref = _ref.load()
    rng = np.random.default_rng(2024)
    for case in range(60):
        src = _random_chain_src(rng)
        prog = ref.parse_program(src)
        req = ref.compute_requirements(prog)
        doc = {
            "program": canonicalize(prog),
            "requirements": {
                "extent": {n: [list(e.i), list(e.j), list(e.k)] for n, e in req.extent.items()},
                "extension": {n: {a: list(v) for a, v in d.items()} for n, d in req.extension.items()},
            },
            "trace": [(i.stencil, dict(i.kwargs)) for i in ref.resolve_driver(prog)],
        }
        domain = (16, 16, 5)
        shapes = interp.input_shapes(doc, domain)
        inputs = {n: rng.uniform(0.1, 10.0, s) for n, s in shapes.items()}
        a = ref.run_reference(prog, inputs, domain)
        b = interp.run_program(doc, inputs, domain)
        assert_outputs_equal(b, a)
