"""ctypes binding of ``libfv3b.so`` (declared in ``include/fv3b.h``).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the engine fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("FV3B_LIB", Path(__file__).resolve().parent / "libfv3b.so"))

ABI_VERSION = 5


class Field(ctypes.Structure):
    """``fv3b_field``."""

    _fields_ = [
        ("data", ctypes.c_void_p),
        ("stride", ctypes.c_int64 * 3),
        ("shape", ctypes.c_int32 * 3),
        ("halo_lo", ctypes.c_int32 * 3),
        ("rank", ctypes.c_int32),
    ]


class Domain(ctypes.Structure):
    """``fv3b_domain`` (== ``RankPlacement`` + sizes)."""

    _fields_ = [
        ("ni", ctypes.c_int32),
        ("nj", ctypes.c_int32),
        ("nk", ctypes.c_int32),
        ("own_i_start", ctypes.c_uint8),
        ("own_i_end", ctypes.c_uint8),
        ("own_j_start", ctypes.c_uint8),
        ("own_j_end", ctypes.c_uint8),
    ]


class Fv3bError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed with status {code}: {msg}")
        self.code = code


_ENTRY_SIG = [ctypes.POINTER(Field), ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
              ctypes.POINTER(Domain), ctypes.c_void_p]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 engine has no CPU fallback)"
            )
        h = ctypes.CDLL(str(LIB_PATH))
        h.fv3b_abi_version.restype = ctypes.c_int
        h.fv3b_last_error.restype = ctypes.c_char_p
        if h.fv3b_abi_version() != ABI_VERSION:
            raise ImportError(f"libfv3b ABI {h.fv3b_abi_version()} != expected {ABI_VERSION}")
        _lib = h
    return _lib


def entry(name: str):
    fn = getattr(lib(), name)
    fn.restype = ctypes.c_int
    fn.argtypes = _ENTRY_SIG
    return fn


def buffer_field(addr: int, n: int) -> Field:
    """A device buffer as an ABI buffer field (include/fv3b.h): rank 1, data
    = its address, shape[0] = its capacity in elements of its type."""
    f = Field()
    f.data = addr
    f.stride[:] = [1, 0, 0]
    f.shape[:] = [n, 1, 1]
    f.halo_lo[:] = [0, 0, 0]
    f.rank = 1
    return f


def tensor_buffer(t) -> Field:
    """``buffer_field`` of a contiguous device tensor (capacity: its numel)."""
    assert t.is_contiguous()
    return buffer_field(t.data_ptr(), t.numel())


def call(name: str, fields: list[Field], scalars: list[float], domain: Domain, stream: int) -> None:
    call_prepared(name, prepare(fields, scalars), domain, stream)


def prepare(fields: list[Field], scalars: list[float]) -> tuple:
    """The ctypes argument arrays of a call, reusable while the buffers live."""
    farr = (Field * len(fields))(*fields)
    sarr = (ctypes.c_double * max(1, len(scalars)))(*scalars)
    return farr, len(fields), sarr, len(scalars)


def call_prepared(name: str, args: tuple, domain: Domain, stream: int) -> None:
    farr, nf, sarr, ns = args
    rc = entry(name)(farr, nf, sarr, ns, ctypes.byref(domain), ctypes.c_void_p(stream))
    if rc != 0:
        raise Fv3bError(name, rc, lib().fv3b_last_error().decode())


def memcpy2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream: int) -> None:
    """``fv3b_memcpy2d``: ``height`` rows of ``width`` bytes, pitches in bytes."""
    fn = lib().fv3b_memcpy2d
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                   ctypes.c_int64, ctypes.c_void_p]
    rc = fn(dst, dpitch, src, spitch, width, height, stream)
    if rc != 0:
        raise Fv3bError("fv3b_memcpy2d", rc, lib().fv3b_last_error().decode())


def enable_peer_access(peer: int) -> None:
    """``fv3b_enable_peer_access`` for the current device."""
    fn = lib().fv3b_enable_peer_access
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int]
    rc = fn(peer)
    if rc != 0:
        raise Fv3bError("fv3b_enable_peer_access", rc, lib().fv3b_last_error().decode())


# launch-configuration knobs (include/fv3b.h FV3B_TUNE_*)
TUNE = {
    "kchunk": 0,
    "kchunk_dsw_transport": 1,
    "kchunk_dsw_momentum": 2,
    "kchunk_csw": 3,
    "kchunk_tracer": 4,
    "kchunk_fv_tp_2d": 5,
    "riem_cols": 6,
}


def tune_set(knob: str, value: int) -> None:
    """``fv3b_tune_set``: process-wide override of a launch-configuration
    knob (0 restores the automatic choice)."""
    fn = lib().fv3b_tune_set
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int, ctypes.c_int]
    rc = fn(TUNE[knob], int(value))
    if rc != 0:
        raise Fv3bError("fv3b_tune_set", rc, lib().fv3b_last_error().decode())


def tune_get(knob: str) -> int:
    fn = lib().fv3b_tune_get
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int]
    return fn(TUNE[knob])


class tuning:
    """Context manager: ``with tuning(kchunk=3): ...`` sets knobs and
    restores their previous values on exit."""

    def __init__(self, **knobs: int):
        self.knobs = knobs
        self.saved: dict[str, int] = {}

    def __enter__(self):
        for k, v in self.knobs.items():
            self.saved[k] = tune_get(k)
            tune_set(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            tune_set(k, v)
        return False
