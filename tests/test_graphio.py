"""Graph persistence in the reference document format (graphio.py ↔
reference ir/serialize.py:154-306): documents the reference writes load
here and reach the same kernel plan and trace; documents written here are
byte-identical to the reference writer's for the same graph, load with the
reference's graph_from_json and execute with its run_reference_graph."""

from __future__ import annotations

import numpy as np
import pytest

import _ref
from oracle import interp
from paper_2205_04148_b200 import graphio
from paper_2205_04148_b200.inputs import synthetic_inputs
from paper_2205_04148_b200.program import PROGRAM_DIR, as_program

needs_ref = pytest.mark.skipif(not _ref.available(), reason="reference package not present")
PROGS = ["copy", "fv_tp_2d", "tracer_2d", "riem_solver_c", "remap_profile", "c_sw", "c_grid", "d_sw", "nh_d",
         "p_grad_d", "remap_tracers"]


def test_program_graph_roundtrip_is_stable():
    g = graphio.program_graph("c_grid", (16, 16, 9))
    text = graphio.graph_to_json(g)
    g2 = graphio.graph_from_json(text)
    assert graphio.graph_to_json(g2) == text
    p = as_program(g2)
    assert p.name == "c_grid" and p.trace == as_program("c_grid").trace


def test_bad_documents_are_rejected():
    with pytest.raises(graphio.SerializationError):
        graphio.graph_from_json('{"format": "other"}')
    with pytest.raises(graphio.SerializationError):
        graphio.graph_from_json('{"format": "stencilkit-graph", "version": 9}')


@needs_ref
@pytest.mark.parametrize("name", PROGS)
def test_reference_document_loads_and_rewrites_identically(name):
    R = _ref.load()
    from stencilkit.ir.lower import lower
    from stencilkit.ir.serialize import graph_to_json

    prog = R.parse_program((PROGRAM_DIR / f"{name}.stn").read_text())
    g = lower(prog, (16, 16, 9), R.RankPlacement(False, True, False, True))
    text = graph_to_json(g)
    ours = graphio.graph_from_json(text)
    assert graphio.graph_to_json(ours) == text
    p, q = as_program(ours), as_program(g)
    assert p.name == q.name == name and p.trace == q.trace
    assert ours.unrolled_trace() == g.unrolled_trace()


@needs_ref
@pytest.mark.parametrize("name,domain", [("fv_tp_2d", (12, 14, 3)), ("c_sw", (13, 12, 2)), ("riem_solver_c", (4, 3, 9)),
                                         ("p_grad_d", (7, 6, 5))])
def test_our_document_runs_on_the_reference(name, domain):
    """program_graph -> graph_to_json -> the reference graph_from_json ->
    run_reference_graph == the oracle on the program (bitwise)."""
    R = _ref.load()
    from stencilkit.executor.reference import run_reference_graph
    from stencilkit.ir.serialize import graph_from_json

    placement = (True, True, True, True)
    text = graphio.graph_to_json(graphio.program_graph(name, domain, placement))
    g = graph_from_json(text)
    ins = synthetic_inputs(name, domain, 3)
    got = run_reference_graph(g, ins)
    ref = interp.run_program(name, ins, domain, interp.Placement(*placement))
    for f in ref:
        assert np.array_equal(got[f], ref[f]), f
