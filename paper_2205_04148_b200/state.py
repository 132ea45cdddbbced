"""Deterministic initial state of the doubly periodic f-plane dycore
(SURVEY 8d "Full-step inputs"): smooth analytic winds plus seeded noise,
hydrostatic thickness and geopotential, uniform 10 km metrics.

Arrays are in the reference convention (axes I, J, K; C order) with a
uniform halo ``cfg.halo`` on I and J and ``nk + 1`` levels on K, already
halo-filled periodically.  Both the CPU oracle step and the B200 step start
from exactly these bits.
"""

from __future__ import annotations

import numpy as np

from .config import DIAG_3D, METRICS_2D, STATE_3D, RunConfig

DX = 1.0e4


def periodic_fill(a: np.ndarray, h: int) -> None:
    """Periodic halo of width h on axes 0 (I) and 1 (J), in place."""
    if h == 0:
        return
    ni, nj = a.shape[0] - 2 * h, a.shape[1] - 2 * h
    a[:h] = a[ni : ni + h]
    a[ni + h :] = a[h : 2 * h]
    a[:, :h] = a[:, nj : nj + h]
    a[:, nj + h :] = a[:, h : 2 * h]


def initial_state(cfg: RunConfig) -> dict[str, np.ndarray]:
    h, ni, nj, nk = cfg.halo, cfg.ni, cfg.nj, cfg.nk
    rng = np.random.default_rng(cfg.seed)
    I, J = ni + 2 * h, nj + 2 * h
    L = nk + 1
    st: dict[str, np.ndarray] = {}
    # metrics (uniform, exact reciprocals)
    for n, v in {"dx": DX, "dy": DX, "dxc": DX, "dyc": DX, "area": DX * DX, "f0": 1.0e-4, "fc": 1.0e-4,
                 "del6_u": 1.0, "del6_v": 1.0}.items():  # del6_u = sin_sg dx / dyc, del6_v = sin_sg dy / dxc
        st[n] = np.full((I, J), v)
    for n, v in {"rdx": 1.0 / DX, "rdy": 1.0 / DX, "rdxc": 1.0 / DX, "rdyc": 1.0 / DX, "rdxa": 1.0 / DX,
                 "rdya": 1.0 / DX, "rarea": 1.0 / (DX * DX), "rarea_c": 1.0 / (DX * DX), "ws": 0.0}.items():
        st[n] = np.full((I, J), v)
    x = 2 * np.pi * (np.arange(I) - h) / ni
    y = 2 * np.pi * (np.arange(J) - h) / nj
    X, Y = np.meshgrid(x, y, indexing="ij")
    kk = np.arange(L)
    z = np.zeros((I, J, L))
    # layer thickness: ptop..1e5 Pa split evenly, with a smooth horizontal
    # pressure perturbation (drives the gradient terms) + 1e-4 noise
    dp0 = (1.0e5 - cfg.consts["ptop"]) / nk
    pert = 1.0 + 2.0e-3 * np.sin(X)[..., None] * np.cos(Y)[..., None]
    st["delp"] = dp0 * pert * (1.0 + 1.0e-4 * rng.uniform(-1, 1, (I, J, L))) + z
    st["pt"] = (300.0 - 40.0 * kk / nk) * (1.0 + 1.0e-4 * rng.uniform(-1, 1, (I, J, L))) + z
    st["u"] = 10.0 * np.sin(Y)[..., None] * (1.0 + 1.0e-3 * rng.uniform(-1, 1, (I, J, L)))
    st["v"] = 10.0 * np.cos(X)[..., None] * (1.0 + 1.0e-3 * rng.uniform(-1, 1, (I, J, L)))
    st["w"] = 1.0e-3 * rng.uniform(-1, 1, (I, J, L))
    # hydrostatic interface geopotential from the surface (flat, gz = 0) up
    dm, pt = st["delp"], st["pt"]
    pem = cfg.consts["ptop"] + np.concatenate([np.zeros((I, J, 1)), np.cumsum(dm[..., :nk], axis=-1)], axis=-1)
    gz = np.zeros((I, J, L))
    for k in range(nk - 1, -1, -1):
        pm = dm[..., k] / np.log(pem[..., k + 1] / pem[..., k])
        gz[..., k] = gz[..., k + 1] + cfg.consts["rdgas"] * pt[..., k] * dm[..., k] / pm
    st["gz"] = gz
    st["pef"] = pem.copy()
    for n in ("uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy", "dp1", *DIAG_3D):
        st[n] = np.zeros((I, J, L))
    for t in range(cfg.nq):
        st[f"q{t}"] = 1.0e-3 * (1.5 + np.sin(X + t)[..., None] * np.cos(Y - t)[..., None]) * \
            (1.0 + 1.0e-3 * rng.uniform(-1, 1, (I, J, L)))
    # the unused top slot of layer fields (level nk) repeats the last layer
    for n in ("delp", "pt", "u", "v", "w") + tuple(f"q{t}" for t in range(cfg.nq)):
        st[n][..., nk] = st[n][..., nk - 1]
    for a in st.values():
        periodic_fill(a, h)
    assert set(STATE_3D) | set(METRICS_2D) <= set(st)
    return st
