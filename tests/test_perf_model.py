"""Performance model / report (perf_model.py), first-touch
bytes and field I/O (fieldio.py, buffers.py:83-116) on CPU."""

from __future__ import annotations

import json

import numpy as np
import pytest

import _ref
from oracle import interp
from paper_2205_04148_b200 import perf_model
from paper_2205_04148_b200.fieldio import load_field, reference_layout, save_field
from paper_2205_04148_b200.inputs import synthetic_inputs
from paper_2205_04148_b200.traffic import compulsory_bytes


def test_model_kernel_copy_known_answer():
    # SPEC.md: copy stencil (8,8,4) float64, B = 10 GB/s -> 4096 B, 409.6 ns
    kb = perf_model.model_kernel("copy", (8, 8, 4), 10e9)
    assert kb.unique_bytes == 4096
    assert kb.bound_time == pytest.approx(409.6e-9)


def test_report_ranking_hotspots_and_csv():
    doms = {"copy": (64, 64, 8), "fv_tp_2d": (64, 64, 8)}
    b_copy = perf_model.model_kernel("copy", doms["copy"], 1e12).bound_time
    b_tp = perf_model.model_kernel("fv_tp_2d", doms["fv_tp_2d"], 1e12).bound_time
    timings = {"copy": [b_copy] * 3, "fv_tp_2d": [2 * b_tp] * 3}  # 100% and 50% utilization
    rep = perf_model.build_report(timings, doms, 1e12)
    assert sorted(rep.ranking) == sorted(doms)
    by = {e.kernel: e for e in rep.entries}
    assert by["copy"].utilization == pytest.approx(1.0) and by["fv_tp_2d"].utilization == pytest.approx(0.5)
    assert perf_model.hotspot_list(rep, 1) == ["fv_tp_2d"]
    csv = perf_model.report_to_csv(rep, reps=3)
    assert csv.startswith("kernel,invocations,measured_s,bound_s,utilization,flags\n")
    assert len(csv.strip().splitlines()) == 3


@pytest.mark.parametrize("name,domain", [("copy", (12, 10, 4)), ("fv_tp_2d", (16, 14, 3)), ("d_sw", (16, 14, 3)),
                                         ("riem_solver_c", (6, 5, 9)), ("tracer_2d", (14, 12, 2)),
                                         ("c_grid", (16, 14, 5))])
def test_first_touch_recorder_vs_box_model(name, domain):
    """The box model (whole allocated halo boxes) bounds the brute-force
    first-touch bytes from above; equal for the copy stencil."""
    rec = interp.FirstTouch()
    interp.run_program(name, synthetic_inputs(name, domain, 1), domain, interp.PERIODIC, recorder=rec,
                       whole_blocks=False)
    box = compulsory_bytes(name, domain)
    assert rec.bytes() <= box
    if name == "copy":
        assert rec.bytes() == box


def test_first_touch_whole_block_path_records_the_same():
    for name, dom in (("fv_tp_2d", (16, 14, 3)), ("riem_solver_c", (6, 5, 9))):
        a, b = interp.FirstTouch(), interp.FirstTouch()
        inp = synthetic_inputs(name, dom, 2)
        interp.run_program(name, inp, dom, interp.PERIODIC, recorder=a, whole_blocks=False)
        interp.run_program(name, inp, dom, interp.PERIODIC, recorder=b, whole_blocks=True)
        assert a.bytes() == b.bytes()


def test_traffic_table_is_first_touch_and_close_to_box_model():
    tab = perf_model._TABLE
    doc = json.loads(tab.read_text())
    assert "d_sw@192x192x80" in doc
    for key, v in doc.items():
        assert v["first_touch_bytes"] <= v["box_model_bytes"] <= 1.01 * v["first_touch_bytes"], key


def test_field_io_roundtrip_and_text(tmp_path):
    a = np.random.default_rng(1).uniform(size=(12, 10, 5))
    save_field("delp", a, tmp_path / "delp.bin", halo_lo=(3, 3, 0))
    name, layout, b = load_field(tmp_path / "delp.bin")
    assert name == "delp" and np.array_equal(a, b)
    assert layout == reference_layout(("I", "J", "K"), (12, 10, 5), (3, 3, 0))
    save_field("delp", a, tmp_path / "delp.txt", text=True)
    lines = (tmp_path / "delp.txt").read_text().splitlines()
    assert lines[0].startswith("# field delp dtype float64 shape [12, 10, 5]") and len(lines) == 1 + a.size


@pytest.mark.skipif(not _ref.available(), reason="reference not importable")
def test_field_io_interoperates_with_reference(tmp_path):
    """Files written here load with the reference load_field (and its Layout)."""
    _ref.load()
    from stencilkit.executor.buffers import load_field as ref_load

    a = np.random.default_rng(2).uniform(size=(14, 12, 6))
    save_field("pt", a, tmp_path / "pt.bin", halo_lo=(3, 3, 0))
    name, layout, b = ref_load(tmp_path / "pt.bin")
    assert name == "pt" and np.array_equal(a, b)
    assert layout.to_json() == reference_layout(("I", "J", "K"), (14, 12, 6), (3, 3, 0))


def test_algorithmic_op_counts():
    """tools/opcount.py: the copy stencil has no arithmetic; the committed
    C2 counts are what the counter gives; d_sw's executed fp64 count (ncu,
    profiles/fp64.json) exceeds its algorithmic count (tile-halo recompute,
    reciprocal refinement) but by less than 2x."""
    import json
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root / "tools"))
    import opcount

    assert opcount.program_ops("copy", (8, 8, 4))["fp64_ops"] == 0
    tab = json.loads((root / "paper_2205_04148_b200" / "traffic_table.json").read_text())
    for name, k in opcount.PROGS:
        key = f"{name}@192x192x{k}"
        assert tab[key]["algorithmic_ops"] == opcount.program_ops(name, (192, 192, k)), name
    executed = json.loads((root / "profiles" / "fp64.json").read_text())["d_sw"]
    alg = tab["d_sw@192x192x80"]["algorithmic_ops"]["fp64_ops"]
    assert alg < executed < 2 * alg
