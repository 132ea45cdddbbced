"""The post-remap pressure / heat-capacity diagnostics' oracle
(oracle/thermo.py) and its deterministic exp (oracle/detmath.det_exp): exp
within 1 ulp of the correctly rounded libm result over the whole normal
range, the diagnostics' defining properties, and the host-side scalars of
the product (RunConfig.moist_scalars) equal to the oracle's."""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import thermo
from oracle.detmath import det_exp, det_log
from paper_2205_04148_b200.config import RunConfig


@pytest.mark.parametrize("lo,hi", [(-708.0, 708.0), (-2.0, 2.0), (-0.35, 0.35), (1.0, 4.0), (-1e-9, 1e-9)])
def test_det_exp_within_one_ulp(lo, hi):
    x = np.random.default_rng(7).uniform(lo, hi, 50000)
    got = det_exp(x)
    want = np.array([math.exp(v) for v in x])
    assert (np.abs(got - want) <= np.spacing(want)).all()


def test_det_exp_edges():
    assert det_exp(0.0) == 1.0
    assert det_exp(1e-300) == 1.0
    x = np.array([np.inf, -np.inf, np.nan, 710.0, -750.0])
    got = det_exp(x)
    with np.errstate(over="ignore"):
        want = np.exp(x)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    np.testing.assert_array_equal(got[~np.isnan(got)], want[~np.isnan(got)])
    # exp(log(x)) round trip near 1 ulp
    v = np.random.default_rng(3).uniform(1.0, 1e5, 1000)
    assert np.allclose(det_exp(det_log(v)), v, rtol=4e-16 * 8)


def test_moist_scalars_match_oracle():
    cfg = RunConfig()
    assert cfg.moist_scalars() == thermo.constants(cfg.consts)


@pytest.mark.parametrize("nw", [0, 1, 3, 6])
def test_moist_pk_properties(nw):
    cfg = RunConfig()
    nk = 40
    rng = np.random.default_rng(nw)
    delp = (1e5 - 300.0) / nk * (1 + 0.5 * rng.uniform(-1, 1, (5, 4, nk)))
    qs = [1e-3 * rng.uniform(0, 1, delp.shape) for _ in range(nw)]
    sc = cfg.moist_scalars()
    out = thermo.moist_pk(delp, qs, nk, sc)
    pe, pk, pkz = out["pe"], out["pk"], out["pkz"]
    assert np.array_equal(pe[..., 0], np.full(pe.shape[:-1], 300.0))
    assert np.allclose(pe[..., -1], 300.0 + delp.sum(-1), rtol=1e-14)
    assert np.allclose(pk, pe ** sc[1], rtol=4e-15)
    assert ((pkz >= pk[..., :-1]) & (pkz <= pk[..., 1:])).all()  # a layer mean of p^kappa
    dry = thermo.moist_pk(delp, [], nk, sc)["cvm"]
    assert np.array_equal(dry, np.full(dry.shape, sc[2]))  # no water: cv of dry air
    if nw:
        assert not np.array_equal(out["cvm"], dry)
