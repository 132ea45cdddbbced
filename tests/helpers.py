"""Shared test helpers: golden fixtures, tolerance checks."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden_cases(program: str | None = None):
    idx = json.loads((GOLDEN / "index.json").read_text())
    for key, meta in sorted(idx.items()):
        if program is None or meta["program"] == program:
            yield key, meta


def load_golden(key: str):
    z = np.load(GOLDEN / f"{key}.npz")
    inputs = {k[4:]: z[k] for k in z.files if k.startswith("in__")}
    outputs = {k[5:]: z[k] for k in z.files if k.startswith("out__")}
    return inputs, outputs


def max_rel_err(a: np.ndarray, b: np.ndarray) -> float:
    """Element-wise relative error with denominator max(|ref|, 1e-300)
    (SURVEY 8c tolerance definition)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def assert_outputs_equal(got: dict, ref: dict, rtol: float = 0.0, names=None):
    names = names or ref.keys()
    for n in names:
        assert got[n].shape == ref[n].shape, f"{n}: shape {got[n].shape} vs {ref[n].shape}"
        if rtol == 0.0:
            if not np.array_equal(got[n], ref[n], equal_nan=True):
                bad = np.argwhere(got[n] != ref[n])
                raise AssertionError(f"{n}: {len(bad)} cells differ (first {bad[:3].tolist()}), "
                                     f"max rel err {max_rel_err(got[n], ref[n]):.3e}")
        else:
            err = max_rel_err(got[n], ref[n])
            assert err <= rtol, f"{n}: max rel err {err:.3e} > {rtol:.1e}"
