"""The C-ABI error channel (include/fv3b.h): every entry point rejects bad
arguments with a negative status and a message naming it in
fv3b_last_error(), before touching the device (so this runs on CPU), like
run_reference's exceptions (reference.py:164-167)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2205_04148_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "fv3b.h"
UNIFORM = r"int (fv3b_[a-z0-9_]+)\(const fv3b_field\* f, int nf, const double\* s, int ns,\s*const fv3b_domain\* d, void\* stream\);"
ENTRIES = sorted(set(re.findall(UNIFORM, HEADER.read_text())))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_2205_04148_b200.build import build

        build()
    return _lib.lib()


def test_entries_parsed():
    assert "fv3b_d_sw" in ENTRIES and "fv3b_remap_map" in ENTRIES and len(ENTRIES) >= 15


@pytest.mark.parametrize("name", ENTRIES)
def test_bad_arguments_give_status_and_message(lib, name):
    fn = _lib.entry(name)
    dom = _lib.Domain()
    dom.ni, dom.nj, dom.nk = 8, 8, 4
    fields = (_lib.Field * 1)()  # one zeroed descriptor (null data): never a valid call
    scal = (ctypes.c_double * 1)(0.0)
    rc = fn(fields, 1, scal, 0, ctypes.byref(dom), None)
    assert rc < 0, f"{name} accepted a bad call"
    msg = lib.fv3b_last_error().decode()
    assert msg, f"{name}: empty error message"


def test_null_pointers_are_rejected(lib):
    for name in ENTRIES:
        rc = _lib.entry(name)(None, 0, None, 0, None, None)
        assert rc < 0, name


def test_wrong_rank_is_a_layout_error(lib):
    """fv3b_copy with a 2-D descriptor where a 3-D field is required."""
    import numpy as np

    buf = np.zeros(16 * 16 * 6)
    f = _lib.Field()
    f.data = buf.ctypes.data
    f.stride[:] = [1, 16, 256]
    f.shape[:] = [16, 16, 6]
    f.halo_lo[:] = [0, 0, 0]
    f.rank = 2
    fields = (_lib.Field * 2)(f, f)
    dom = _lib.Domain()
    dom.ni, dom.nj, dom.nk = 8, 8, 4
    rc = _lib.entry("fv3b_copy")(fields, 2, None, 0, ctypes.byref(dom), None)
    assert rc == -2, rc  # FV3B_ELAYOUT
    assert "rank" in lib.fv3b_last_error().decode()


def test_tuning_knobs_roundtrip(lib):
    """fv3b_tune_set / fv3b_tune_get (host-only state, no device)."""
    assert _lib.tune_get("kchunk") == 0
    with _lib.tuning(kchunk=3, kchunk_csw=5):
        assert _lib.tune_get("kchunk") == 3 and _lib.tune_get("kchunk_csw") == 5
    assert _lib.tune_get("kchunk") == 0 and _lib.tune_get("kchunk_csw") == 0
    assert lib.fv3b_tune_set(99, 1) < 0 and "unknown knob" in lib.fv3b_last_error().decode()
    assert lib.fv3b_tune_set(0, -1) < 0
    assert lib.fv3b_tune_get(99) == -1
    assert set(_lib.TUNE.values()) == set(range(len(_lib.TUNE)))


def test_tuning_table_roundtrip(tmp_path, monkeypatch, lib):
    """tuning.record / apply: knobs of the matching (device, shape) entry only."""
    from paper_2205_04148_b200 import tuning

    monkeypatch.setattr(tuning, "PATH", tmp_path / "tuning.json")
    tuning.record("GPU X", (192, 192, 80), {"knobs": {"kchunk_csw": 20}})
    assert tuning.lookup("GPU X", (192, 192, 80)) == {"kchunk_csw": 20}
    assert tuning.apply("GPU Y", (192, 192, 80)) == {}
    try:
        assert tuning.apply("GPU X", (192, 192, 80)) == {"kchunk_csw": 20}
        assert _lib.tune_get("kchunk_csw") == 20
    finally:
        _lib.tune_set("kchunk_csw", 0)
