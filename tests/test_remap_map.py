"""CPU checks of the remap-mapping oracle (oracle/remap_map.py): the
vectorised restatement against the scalar map1_ppm transliteration, and the
properties of the method (conservation, constants, identity coordinate)."""

import numpy as np
import pytest

from oracle import remap_map as rm
from paper_2205_04148_b200.config import RunConfig


def _profile(q, delp, nk):
    """Edge values / curvature with the remap_profile conventions (a simple
    consistent profile for the mapping checks: edges from neighbour means)."""
    a2 = np.empty_like(q)
    a3 = np.empty_like(q)
    a2[..., 1:nk] = 0.5 * (q[..., : nk - 1] + q[..., 1:nk])
    a2[..., 0] = q[..., 0]
    a3[..., : nk - 1] = a2[..., 1:nk]
    a3[..., nk - 1] = q[..., nk - 1]
    a4 = 3.0 * (2.0 * q - (a2 + a3))
    return a2, a3, a4


def _columns(n, nk, seed):
    rng = np.random.default_rng(seed)
    delp = (1.0e5 - 300.0) / nk * (1.0 + 0.3 * rng.uniform(-1, 1, (n, nk)))
    q = rng.uniform(0.5, 2.0, (n, nk))
    return delp, q


@pytest.mark.parametrize("nk", [3, 8, 30])
def test_vectorised_matches_scalar_bitwise(nk):
    delp, q = _columns(64, nk, 3)
    ak, bk = RunConfig(nk=nk).target_coordinate()
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    a2, a3, a4 = _profile(q, delp, nk)
    got = rm.map_columns(pe1, pe2, q, a2, a3, a4, nk)
    for c in range(delp.shape[0]):
        want = rm.map_column(pe1[c], pe2[c], q[c], a2[c], a3[c], a4[c], nk)
        assert np.array_equal(got[c], want), c


def test_column_integral_conserved():
    nk = 40
    delp, q = _columns(128, nk, 5)
    ak, bk = RunConfig(nk=nk).target_coordinate()
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    a2, a3, a4 = _profile(q, delp, nk)
    q2 = rm.map_columns(pe1, pe2, q, a2, a3, a4, nk)
    before = (q * (pe1[:, 1:] - pe1[:, :-1])).sum(axis=1)
    after = (q2 * (pe2[:, 1:] - pe2[:, :-1])).sum(axis=1)
    assert np.allclose(after, before, rtol=1e-12, atol=0)


def test_constant_is_preserved_and_identity_coordinate():
    nk = 16
    delp, _ = _columns(32, nk, 7)
    ak, bk = RunConfig(nk=nk).target_coordinate()
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    c = np.full((32, nk), 1.25)
    q2 = rm.map_columns(pe1, pe2, c, c, c, np.zeros_like(c), nk)
    assert np.allclose(q2, 1.25, rtol=1e-13)
    # mapping onto the source interfaces returns the layer means
    _, q = _columns(32, nk, 8)
    a2, a3, a4 = _profile(q, delp, nk)
    q3 = rm.map_columns(pe1, pe1, q, a2, a3, a4, nk)
    assert np.allclose(q3, q, rtol=1e-12)


def test_log_pressure_mapping_conserves_and_preserves_constants():
    """The log-pressure mapping (FV3 pt, kord_tm < 0): map1_ppm on the log
    interfaces conserves the column integral of q d(log p) and maps a
    constant profile exactly; log_thickness is the difference of the log
    interfaces."""
    from paper_2205_04148_b200.config import RunConfig

    nk = 24
    delp, q = _columns(64, nk, 5)
    ak, bk = RunConfig(nk=nk).target_coordinate()
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    l1, l2 = rm.log_edges(pe1, pe2)
    assert np.array_equal(rm.log_thickness(delp, ak, nk), l1[..., 1:] - l1[..., :-1])
    assert np.array_equal(l1[..., 0], l2[..., 0]) and np.array_equal(l1[..., -1], l2[..., -1])
    a2, a3, a4 = _profile(q, delp, nk)
    q2 = rm.map_columns(l1, l2, q, a2, a3, a4, nk)
    before = (q * (l1[..., 1:] - l1[..., :-1])).sum(axis=-1)
    after = (q2 * (l2[..., 1:] - l2[..., :-1])).sum(axis=-1)
    assert np.allclose(after, before, rtol=1e-12)
    c = np.full_like(q, 3.25)
    assert np.allclose(rm.map_columns(l1, l2, c, c, c, np.zeros_like(c), nk), 3.25, rtol=1e-14)
