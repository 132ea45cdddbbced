"""CPU restatement of the vertical remapping step that follows
remap_profile: the piecewise-parabolic profile of every Lagrangian layer is
integrated over the target (Eulerian) layers -- FV3's ``map_single`` /
``map1_ppm`` (Lin 2004; the "Lagrangian contributions" of PAPER.md:87-89,
:639).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
CPU legs of bench.py, as the checker of ``fv3b_remap_map``.

Parity unpinned: the reference ships no remapping (it needs
data-dependent vertical indexing, which its DSL cannot express), so this
restatement *defines* the algorithm and the device kernel reproduces it
bitwise (same IEEE operations in the same order per column).  Its own
correctness is checked against a scalar transliteration (``map_column``)
and by the properties of the method: the column integral of q*dp is
conserved, and a profile with a4_2 = a4_3 = q, a4_4 = 0 maps a constant
exactly.

Conventions: k = 0 is the model top; pe1 are the Lagrangian interface
pressures (pe1[0] = ptop, pe1[k+1] = pe1[k] + delp[k]), pe2 the target
interfaces pe2[k] = ak[k] + bk[k] * ps with ps = pe1[nk] and both end
interfaces copied from pe1 (as FV3 does).  a2, a3, a4 are remap_profile's
a4_2 (left edge), a4_3 (right edge), a4_4 (curvature).
"""

from __future__ import annotations

import numpy as np

from .detmath import det_log

R3 = 1.0 / 3.0
R23 = 2.0 / 3.0


def pe_edges(delp: np.ndarray, ak: np.ndarray, bk: np.ndarray, nk: int) -> tuple[np.ndarray, np.ndarray]:
    """pe1, pe2 of shape (..., nk+1) for layer thicknesses delp (..., >= nk)."""
    shape = delp.shape[:-1] + (nk + 1,)
    pe1 = np.empty(shape)
    pe1[..., 0] = ak[0]
    for k in range(nk):
        pe1[..., k + 1] = pe1[..., k] + delp[..., k]
    ps = pe1[..., nk]
    pe2 = np.empty(shape)
    pe2[..., 0] = pe1[..., 0]
    for k in range(1, nk):
        pe2[..., k] = ak[k] + bk[k] * ps
    pe2[..., nk] = ps
    return pe1, pe2


def map_columns(pe1, pe2, q, a2, a3, a4, nk: int) -> np.ndarray:
    """Vectorised over columns (leading axes flattened); returns q2 (..., nk)."""
    lead = pe1.shape[:-1]
    P1 = pe1.reshape(-1, nk + 1)
    P2 = pe2.reshape(-1, nk + 1)
    Q, A2, A3, A4 = (x[..., :nk].reshape(-1, nk) for x in (q, a2, a3, a4))
    n = P1.shape[0]
    cols = np.arange(n)
    dp1 = P1[:, 1:] - P1[:, :-1]
    q2 = np.empty((n, nk))
    k0 = np.zeros(n, dtype=np.int64)
    for k2 in range(nk):
        top, bot = P2[:, k2], P2[:, k2 + 1]
        # first k1 >= k0 with pe2(k2) <= pe1(k1+1)
        k1 = k0.copy()
        adv = (top > P1[cols, k1 + 1]) & (k1 < nk - 1)
        while adv.any():
            k1[adv] += 1
            adv = (top > P1[cols, k1 + 1]) & (k1 < nk - 1)
        d = dp1[cols, k1]
        pl = (top - P1[cols, k1]) / d
        b2, b3, b4 = A2[cols, k1], A3[cols, k1], A4[cols, k1]
        inside = bot <= P1[cols, k1 + 1]
        # the whole target layer inside source layer k1
        pr = (bot - P1[cols, k1]) / d
        q_in = b2 + 0.5 * (b4 + b3 - b2) * (pr + pl) - b4 * R3 * (pr * (pr + pl) + pl * pl)
        # fractional: the rest of layer k1, whole layers, then part of the last one
        qsum = (P1[cols, k1 + 1] - top) * (b2 + 0.5 * (b4 + b3 - b2) * (1.0 + pl) - b4 * (R3 * (1.0 + pl * (1.0 + pl))))
        m = k1 + 1
        kend = k1.copy()
        act = ~inside & (m < nk)
        while act.any():
            mm = np.where(act, m, 0)
            whole = act & (bot > P1[cols, np.minimum(mm + 1, nk)])
            part = act & ~whole
            qsum = np.where(whole, qsum + dp1[cols, mm] * Q[cols, mm], qsum)
            dp = bot - P1[cols, mm]
            esl = dp / dp1[cols, mm]
            qp = qsum + dp * (A2[cols, mm] + 0.5 * esl * (A3[cols, mm] - A2[cols, mm] + A4[cols, mm] * (1.0 - R23 * esl)))
            qsum = np.where(part, qp, qsum)
            kend = np.where(part, mm, kend)
            m = np.where(whole, m + 1, m)
            act = whole & (m < nk)
        q2[:, k2] = np.where(inside, q_in, qsum / (bot - top))
        k0 = np.where(inside, k1, kend)
    return q2.reshape(lead + (nk,))


def map_column(pe1, pe2, q, a2, a3, a4, nk: int) -> np.ndarray:
    """Scalar transliteration of map1_ppm for one column (checker of
    map_columns; same operations, Python floats)."""
    dp1 = [pe1[k + 1] - pe1[k] for k in range(nk)]
    q2 = np.empty(nk)
    k0 = 0
    for k2 in range(nk):
        top, bot = pe2[k2], pe2[k2 + 1]
        k1 = k0
        while top > pe1[k1 + 1] and k1 < nk - 1:
            k1 += 1
        pl = (top - pe1[k1]) / dp1[k1]
        if bot <= pe1[k1 + 1]:
            pr = (bot - pe1[k1]) / dp1[k1]
            q2[k2] = a2[k1] + 0.5 * (a4[k1] + a3[k1] - a2[k1]) * (pr + pl) - a4[k1] * R3 * (pr * (pr + pl) + pl * pl)
            k0 = k1
            continue
        qsum = (pe1[k1 + 1] - top) * (a2[k1] + 0.5 * (a4[k1] + a3[k1] - a2[k1]) * (1.0 + pl) -
                                      a4[k1] * (R3 * (1.0 + pl * (1.0 + pl))))
        kend = k1
        for m in range(k1 + 1, nk):
            if bot > pe1[m + 1]:
                qsum = qsum + dp1[m] * q[m]
            else:
                dp = bot - pe1[m]
                esl = dp / dp1[m]
                qsum = qsum + dp * (a2[m] + 0.5 * esl * (a3[m] - a2[m] + a4[m] * (1.0 - R23 * esl)))
                kend = m
                break
        q2[k2] = qsum / (bot - top)
        k0 = kend
    return q2


def face_thickness(delp: np.ndarray, nk: int, h: int) -> tuple[np.ndarray, np.ndarray]:
    """Layer thickness at the D-grid wind points (u(i, j) between cells
    (i, j-1) and (i, j), v(i, j) between (i-1, j) and (i, j)), interior
    columns, as fv3b_face_thickness: du = 0.5 * (delp[0,-1,0] + delp)."""
    du = np.zeros_like(delp)
    dv = np.zeros_like(delp)
    I, J = delp.shape[0] - 2 * h, delp.shape[1] - 2 * h
    c = delp[h:h + I, h:h + J, :nk]
    du[h:h + I, h:h + J, :nk] = 0.5 * (delp[h:h + I, h - 1:h - 1 + J, :nk] + c)
    dv[h:h + I, h:h + J, :nk] = 0.5 * (delp[h - 1:h - 1 + I, h:h + J, :nk] + c)
    return du, dv


def log_edges(pe1: np.ndarray, pe2: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """The interfaces in the log-pressure mapping coordinate (FV3 maps pt in
    log(p) when kord_tm < 0: ``peln`` and ``log(pe2)`` in fv_mapz), through
    the deterministic det_log (the device's)."""
    return det_log(pe1), det_log(pe2)


def log_thickness(delp: np.ndarray, ak, nk: int) -> np.ndarray:
    """dlnp[k] = log(pe1[k+1]) - log(pe1[k]) (..., nk): the layer thickness
    remap_profile takes for a field remapped in log pressure
    (fv3b_log_thickness)."""
    pe1, _ = pe_edges(delp, ak, np.zeros(nk + 1), nk)
    ln1 = det_log(pe1)
    return ln1[..., 1:] - ln1[..., :-1]


def remap_map(state: dict, names: list[str], ak, bk, nk: int, h: int, delp_key: str = "delp",
              log: bool = False) -> None:
    """In place on the interior columns of reference-convention arrays:
    every field q in ``names`` <- its profile (q_a2, q_a3, q_a4) mapped onto
    the target layers of the thickness ``state[delp_key]``; then that
    thickness <- pe2 differences.  ``log``: the mapping coordinate is
    log(p) (the profiles were formed at log_thickness) and the thickness is
    left as it is."""
    sl = (slice(h, -h or None), slice(h, -h or None))
    delp = state[delp_key][sl]
    pe1, pe2 = pe_edges(delp, ak, bk, nk)
    x1, x2 = log_edges(pe1, pe2) if log else (pe1, pe2)
    for n in names:
        q = state[n][sl]
        q2 = map_columns(x1, x2, q, state[f"{n}_a2"][sl], state[f"{n}_a3"][sl], state[f"{n}_a4"][sl], nk)
        q[..., :nk] = q2
    if not log:  # (a log-pressure mapping only reads the thickness)
        delp[..., :nk] = pe2[..., 1:] - pe2[..., :-1]
