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


def _host_field(arr, halo=0):
    """A host array as an ABI field (validation only: nothing is launched)."""
    f = _lib.Field()
    f.data = arr.ctypes.data
    nk, nj, ni = arr.shape
    f.stride[:] = [1, ni, ni * nj]
    f.shape[:] = [ni, nj, nk]
    f.halo_lo[:] = [halo, halo, 0]
    f.rank = 3
    return f


def test_buffer_fields_are_checked(lib):
    """ABI v5: message buffers, index lists and flag words travel as rank-1
    buffer fields; a rank other than 1, a null address or too small a
    capacity is rejected before any launch (so this runs on CPU)."""
    import numpy as np

    dom = _lib.Domain()
    dom.ni, dom.nj, dom.nk = 8, 8, 4
    field = np.zeros((5, 16, 16))
    small = np.zeros(4)
    f = _host_field(field, halo=4)
    stream = None

    def call(name, fields, scalars):
        farr = (_lib.Field * len(fields))(*fields)
        sarr = (ctypes.c_double * max(1, len(scalars)))(*scalars)
        return _lib.entry(name)(farr, len(fields), sarr, len(scalars), ctypes.byref(dom), stream)

    # a strip of 4 x 1 cells over 5 levels needs 20 doubles
    rc = call("fv3b_halo_pack", [f, _lib.buffer_field(small.ctypes.data, small.size)], [0, 0, 4, 1])
    assert rc < 0 and "needs" in lib.fv3b_last_error().decode()
    rc = call("fv3b_halo_pack", [f, _host_field(field)], [0, 0, 4, 1])  # a rank-3 field as the buffer
    assert rc < 0 and "rank-1" in lib.fv3b_last_error().decode()
    # one rectangle of 2 x 2 at offset 0, one field of 5 levels: 20 doubles
    rc = call("fv3b_halo_pack_rects", [f, _lib.buffer_field(small.ctypes.data, small.size)], [1, 0, 0, 2, 2, 0])
    assert rc < 0 and "needs" in lib.fv3b_last_error().decode()
    # gather: 3 entries over 5 levels need 15 doubles and 6 int32
    rc = call("fv3b_halo_gather", [f, _lib.buffer_field(small.ctypes.data, small.size),
                                   _lib.buffer_field(small.ctypes.data, 8)], [3])
    assert rc < 0 and "needs" in lib.fv3b_last_error().decode()
    # the barrier's words: a null address
    rc = call("fv3b_peer_barrier", [_lib.buffer_field(0, 1), _lib.buffer_field(small.ctypes.data, 1)], [1, 0])
    assert rc < 0 and "non-null" in lib.fv3b_last_error().decode()
