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
    "area": (0.9, 1.1), "dp1": (5.0, 10.0), "delp": (5.0, 10.0),
}


def field_range(name: str) -> tuple[float, float]:
    return _RANGES.get(name, (0.1, 10.0))


def synthetic_inputs(program, domain, seed: int = 7) -> dict[str, np.ndarray]:
    prog = as_program(program)
    rng = np.random.default_rng(seed)
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
        lo, hi = field_range(name)
        out[name] = rng.uniform(lo, hi, shape)
    return out
