"""Host-side logic without a GPU: manifests, fingerprint dispatch, driver
resolution, device layout arithmetic, and the C-ABI library surface."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import _ref
from paper_2205_04148_b200 import program as P
from paper_2205_04148_b200.device import Grid

ROOT = Path(__file__).resolve().parents[1]
needs_ref = pytest.mark.skipif(not _ref.available(), reason="reference package not present")


def test_all_manifests_load():
    progs = P.known_programs()
    names = {p.name for p in progs.values()}
    assert {"copy", "fv_tp_2d", "tracer_2d"} <= names
    for p in progs.values():
        assert p.trace, p.name
        assert all(len(ext) == 3 for ext in (f.extent for f in p.fields.values()))


def test_stn_regenerates_identically():
    """The committed .stn files are exactly what the templates emit."""
    from paper_2205_04148_b200.programs import templates

    for name, text_now in templates.programs().items():
        text = (P.PROGRAM_DIR / f"{name}.stn").read_text()
        assert text.split("\n", 1)[1] == text_now, name


@needs_ref
def test_reference_ast_dispatches_by_fingerprint():
    ref = _ref.load()
    for name in P.known_programs_names():
        prog = ref.parse_program((P.PROGRAM_DIR / f"{name}.stn").read_text())
        got = P.as_program(prog)
        assert got.name == name
        assert got.trace == [(i.stencil, dict(i.kwargs)) for i in ref.resolve_driver(prog)]


@needs_ref
def test_unknown_program_is_rejected():
    ref = _ref.load()
    prog = ref.parse_program(
        "field a : float64 [I, J, K]\nfield b : float64 [I, J, K]\n"
        "stencil s:\n    with computation(PARALLEL), interval(...):\n        b = a * 2.0\n"
        "driver:\n    s()\n")
    with pytest.raises(KeyError, match="no B200 kernel plan"):
        P.as_program(prog)


@needs_ref
def test_driver_resolution_matches_reference():
    ref = _ref.load()
    src = (
        "const n_split = 3\nconst do_corners = 1\n"
        "field a : float64 [I, J, K]\nfield b : float64 [I, J, K]\n"
        "stencil sa uses (w):\n    with computation(PARALLEL), interval(...):\n        a = w * b\n"
        "stencil sb:\n    with computation(PARALLEL), interval(...):\n        b = a + 1.0\n"
        "driver:\n    x = 5\n    y = x + 1\n    if do_corners:\n        sa(w = y)\n    else:\n        sb()\n"
        "    for t in range(n_split) unroll:\n        sb()\n        sa(w = t * 2.0)\n")
    prog = ref.parse_program(src)
    assert P.resolve_trace(P.canonicalize(prog)) == [(i.stencil, dict(i.kwargs)) for i in ref.resolve_driver(prog)]


def test_grid_layout_matches_reference_allocate_layout_rule():
    # scheduling.py:377-407: pre_pad = (a - h_lo % a) % a, rows padded to a
    g = Grid(192, 192, 80, halo=4)
    assert g.pre_pad == 4 and g.i0 == 8 and g.pitch == 208 and g.rows == 200 and g.levels == 81
    g3 = Grid(48, 48, 16, halo=3)
    assert g3.pre_pad == 5 and g3.i0 == 8 and g3.pitch % 8 == 0 and g3.pitch >= 5 + 48 + 6
    assert (g3.i0 * 8) % 64 == 0


def test_grid_host_roundtrip_cpu():
    g = Grid(10, 7, 3, halo=4)
    t = g.new3(device="cpu")
    host = np.arange(16 * 13 * 3, dtype=np.float64).reshape(16, 13, 3)  # halos (3,3),(3,3)
    g.put(t, host, ("I", "J", "K"), (3, 3, 0))
    back = g.get(t, ("I", "J", "K"), (3, 3, 0), host.shape)
    assert np.array_equal(back, host)
    assert t[0, 4, 8].item() == host[3, 3, 0]  # interior origin


def _header_symbols():
    text = (ROOT / "include" / "fv3b.h").read_text()
    return sorted(set(re.findall(r"\b(fv3b_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2205_04148_b200 import _lib

    if not _lib.LIB_PATH.exists():
        from paper_2205_04148_b200.build import build

        build()
    h = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = _header_symbols()
    assert "fv3b_fv_tp_2d" in syms and "fv3b_last_error" in syms
    for s in syms:
        assert hasattr(h, s), f"{s} declared in include/fv3b.h but not exported"
    assert _lib.lib().fv3b_abi_version() == _lib.ABI_VERSION


@pytest.mark.skipif(not _ref.available(), reason="reference not importable")
@pytest.mark.parametrize("name", ["copy", "fv_tp_2d", "tracer_2d", "c_sw", "c_grid", "d_sw", "nh_d", "p_grad_d",
                                  "riem_solver_c", "remap_profile", "remap_tracers"])
def test_lowered_graph_intake_matches_program(name):
    """run_scheduled(graph, ...) contract: a DataflowGraph
    from the reference ``lower`` maps to the same kernel plan and the same
    resolved invocation trace as the StencilProgram it was lowered from."""
    from paper_2205_04148_b200.program import PROGRAM_DIR, as_program

    R = _ref.load()
    from stencilkit.ir.lower import lower

    prog = R.parse_program((PROGRAM_DIR / f"{name}.stn").read_text())
    g = lower(prog, (16, 16, 9), R.RankPlacement(False, False, False, False))
    pa, pg = as_program(prog), as_program(g)
    assert pg.name == pa.name == name
    assert pg.trace == pa.trace
