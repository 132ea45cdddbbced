"""Deterministic synthetic inputs for the shipped programs.

One ``numpy.random.default_rng(seed)`` stream, one draw per non-temporary
field in declaration order (as ``pkg/tests/test_extents.py:28-34``).  Ranges
are chosen per field role so both branches of every upwind ``select`` fire
and every flux-form denominator stays well away from zero:

* Courant numbers ``crx cry cx cy``: U(-0.8, 0.8)
* area / mass fluxes ``xfx yfx mfx mfy``: U(-0.25, 0.25) (cell area ~1)
* cell areas ``area``: U(0.9, 1.1), ``rarea = 1/area``
* layer thickness ``dp1 delp``: U(5, 10)
* everything else: U(0.1, 10) (``SPEC.md:652``)
"""

from __future__ import annotations

import numpy as np

from .program import as_program

_RANGES = {
    "crx": (-0.8, 0.8), "cry": (-0.8, 0.8), "cx": (-0.8, 0.8), "cy": (-0.8, 0.8),
    "xfx": (-0.25, 0.25), "yfx": (-0.25, 0.25), "mfx": (-0.25, 0.25), "mfy": (-0.25, 0.25),
    "area": (0.9, 1.1), "dp1": (5.0, 10.0),
    # vertical-column state (Pa, K, m/s)
    "dm": (900.0, 1300.0), "delp": (900.0, 1300.0), "delpc": (900.0, 1300.0),
    "pt": (270.0, 300.0), "ptc": (270.0, 300.0),
    "w": (-1.0, 1.0), "wc": (-1.0, 1.0), "ws": (-0.1, 0.1),
}

# Programs on a physical grid (they declare metric terms): ~10 km cells,
# f-plane Coriolis, winds of tens of m/s.
_PHYSICAL = {
    "u": (-15.0, 15.0), "v": (-15.0, 15.0), "uc": (-15.0, 15.0), "vc": (-15.0, 15.0),
    "dx": (9.5e3, 1.05e4), "dy": (9.5e3, 1.05e4), "dxc": (9.5e3, 1.05e4), "dyc": (9.5e3, 1.05e4),
    "rdxa": (0.95e-4, 1.05e-4), "rdya": (0.95e-4, 1.05e-4),
    "rdx": (0.95e-4, 1.05e-4), "rdy": (0.95e-4, 1.05e-4), "rdxc": (0.95e-4, 1.05e-4), "rdyc": (0.95e-4, 1.05e-4),
    "area": (0.9e8, 1.1e8), "rarea": (0.9e-8, 1.1e-8), "rarea_c": (0.9e-8, 1.1e-8),
    "fc": (0.9e-4, 1.1e-4), "f0": (0.9e-4, 1.1e-4),
    "del6_u": (0.9, 1.1), "del6_v": (0.9, 1.1),
    "cx": (-1.0, 1.0), "cy": (-1.0, 1.0), "xfa": (-1.0, 1.0), "yfa": (-1.0, 1.0),
    "mfx": (-1.0, 1.0), "mfy": (-1.0, 1.0),
}

PTOP = 300.0
RDGAS = 287.05


def field_range(name: str, physical: bool = False) -> tuple[float, float]:
    if physical and name in _PHYSICAL:
        return _PHYSICAL[name]
    return _RANGES.get(name, (0.1, 10.0))


def synthetic_inputs(program, domain, seed: int = 7) -> dict[str, np.ndarray]:
    prog = as_program(program)
    rng = np.random.default_rng(seed)
    physical = any(m in prog.fields for m in ("dx", "dy", "rdx", "rdy"))
    out = {}
    for name, info in prog.fields.items():
        if info.temporary:
            continue
        shape = info.shape(tuple(domain))
        if name.startswith("r") and name[1:] in out and prog.fields[name[1:]].dims == info.dims:
            # reciprocal metric (rarea = 1/area, rdx = 1/dx, ...) on its own window
            base = prog.fields[name[1:]]
            offs = [base.halo(a)[0] - info.halo(a)[0] for a in info.dims]
            if all(o >= 0 for o in offs):
                sl = tuple(slice(o, o + n) for o, n in zip(offs, shape))
                if all(s.stop <= m for s, m in zip(sl, out[name[1:]].shape)):
                    out[name] = 1.0 / out[name[1:]][sl]
                    continue
        lo, hi = field_range(name, physical)
        out[name] = rng.uniform(lo, hi, shape)
    if "pef" in out and "gz" in out and not any(n in out for n in ("dm", "delp", "delpc")):
        # interface pressure and geopotential of a random hydrostatic column
        dm = rng.uniform(900.0, 1300.0, out["pef"].shape)
        pt = rng.uniform(270.0, 300.0, out["pef"].shape)
        out["pef"] = PTOP + np.concatenate([np.zeros(dm.shape[:-1] + (1,)), np.cumsum(dm[..., :-1], axis=-1)], axis=-1)
        out["gz"] = hydrostatic_gz(dm, pt, rng)
    for gz in ("gz", "gzc"):
        if gz in out:
            dm = next((out[n] for n in ("dm", "delpc", "delp") if n in out), None)
            pt = next((out[n] for n in ("pt", "ptc") if n in out), None)
            if dm is not None and pt is not None and dm.shape == out[gz].shape:
                out[gz] = hydrostatic_gz(dm, pt, rng)
    return out


def hydrostatic_gz(dm: np.ndarray, pt: np.ndarray, rng, hs_range=(0.0, 2000.0)) -> np.ndarray:
    """Interface geopotential (last axis = nk+1 interfaces; the last layer
    slot of dm/pt is unused) integrated upward from a random surface value,
    with the log-mean layer pressure, plus 1e-3 relative noise."""
    n = dm.shape[-1] - 1
    pem = PTOP + np.concatenate([np.zeros(dm.shape[:-1] + (1,)), np.cumsum(dm[..., :n], axis=-1)], axis=-1)
    gz = np.empty_like(dm)
    gz[..., n] = rng.uniform(*hs_range, dm.shape[:-1])
    for k in range(n - 1, -1, -1):
        pm = dm[..., k] / np.log(pem[..., k + 1] / pem[..., k])
        dz = RDGAS * pt[..., k] * dm[..., k] / pm
        gz[..., k] = gz[..., k + 1] + dz * (1.0 + 1e-3 * rng.uniform(-1.0, 1.0, dz.shape))
    return gz
