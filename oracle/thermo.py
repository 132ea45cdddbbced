"""CPU restatement of the pressure and heat-capacity diagnostics of the
remapped state: the pe / pk / moist_cv part of FV3's Lagrangian-to-Eulerian
step (``fv_mapz`` after ``map1_ppm``).

TEST INFRASTRUCTURE ONLY: used by tests/, the oracle step driver
(oracle/dycore.py) and the CPU legs of bench.py, as the checker of
``fv3b_moist_pk``.

Parity unpinned: the reference ships no remapping, so this
restatement defines the operation and the device kernel reproduces it
bitwise (det_log / det_exp of oracle/detmath.py, the same IEEE operations in
the same order).  Definitions (FV3, hydrostatic pkz):

    pe[0] = ptop, pe[k+1] = pe[k] + delp[k]
    peln = log(pe), pk = exp(akap * peln)
    pkz[k] = (pk[k+1] - pk[k]) / (akap * (peln[k+1] - peln[k]))
    cvm = (1 - (qv + ql + qs)) * cv_air + qv * cv_vap + ql * c_liq + qs * c_ice

with ql = liquid + rain and qs = ice + snow + graupel (FV3's six water
species, tracers q0..q5 in that order; absent species count as 0).
"""

from __future__ import annotations

import numpy as np

from .detmath import det_exp, det_log

SPECIES = 6


def constants(consts: dict) -> list[float]:
    """[ptop, akap, cv_air, cv_vap, c_liq, c_ice] from RunConfig.consts
    (the scalars of fv3b_moist_pk, computed once on the host)."""
    rdgas, cp_air, rvgas = consts["rdgas"], consts["cp_air"], consts["rvgas"]
    return [consts["ptop"], rdgas / cp_air, cp_air - rdgas, 3.0 * rvgas, consts["c_liq"], consts["c_ice"]]


def moist_pk(delp: np.ndarray, qs: list, nk: int, scalars: list[float]) -> dict[str, np.ndarray]:
    """delp (..., >= nk), qs: the moist tracers (0..6 arrays like delp).
    Returns pe, peln, pk (..., nk+1) and pkz, cvm (..., nk)."""
    ptop, akap, cv_air, cv_vap, c_liq, c_ice = scalars
    shape = delp.shape[:-1] + (nk + 1,)
    pe = np.empty(shape)
    pe[..., 0] = ptop
    for k in range(nk):
        pe[..., k + 1] = pe[..., k] + delp[..., k]
    peln = det_log(pe)
    pk = det_exp(akap * peln)
    pkz = (pk[..., 1:] - pk[..., :-1]) / (akap * (peln[..., 1:] - peln[..., :-1]))
    zero = np.zeros(delp.shape[:-1] + (nk,))
    q = [x[..., :nk] for x in qs] + [zero] * (SPECIES - len(qs))
    qv, ql, qsol = q[0], q[1] + q[2], q[3] + q[4] + q[5]
    qd = ql + qsol
    cvm = (1.0 - (qv + qd)) * cv_air + qv * cv_vap + ql * c_liq + qsol * c_ice
    return {"pe": pe, "peln": peln, "pk": pk, "pkz": pkz, "cvm": cvm}


def apply(state: dict, names: list[str], nk: int, h: int, scalars: list[float]) -> None:
    """In place on the interior columns of reference-convention arrays: the
    diagnostics of ``state['delp']`` and the moist tracers ``names``."""
    sl = (slice(h, -h or None), slice(h, -h or None))
    out = moist_pk(state["delp"][sl], [state[n][sl] for n in names], nk, scalars)
    for n in ("pe", "peln", "pk"):
        state[n][sl][..., : nk + 1] = out[n]
    for n in ("pkz", "cvm"):
        state[n][sl][..., :nk] = out[n]
