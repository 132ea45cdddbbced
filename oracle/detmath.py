"""Deterministic ``log`` for the documented oracle extension.

TEST INFRASTRUCTURE (imported by ``oracle/interp.py`` and ``tests/_ref.py``).

The reference DSL has no ``log`` (``frontend/ast.py:28``); the extension adds
one.  Its semantics are fixed here as an explicit IEEE-754 algorithm so that
every engine that evaluates it with the same operations in the same order
(NumPy on the host, CUDA with ``-fmad=false`` on the device) produces the
same bits: the range reduction and minimax polynomial of fdlibm's
``__ieee754_log`` (Sun Microsystems, 1993), error < 1 ulp, restated with
only ``frexp``, ``+ - * /``.  ``csrc/detmath.cuh`` is the device copy.
"""

from __future__ import annotations

import numpy as np

LN2_HI = float.fromhex("0x1.62e42fee00000p-1")
LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
LG1 = float.fromhex("0x1.5555555555593p-1")
LG2 = float.fromhex("0x1.999999997fa04p-2")
LG3 = float.fromhex("0x1.2492494229359p-2")
LG4 = float.fromhex("0x1.c71c51d8e78afp-3")
LG5 = float.fromhex("0x1.7466496cb03dep-3")
LG6 = float.fromhex("0x1.39a09d078c69fp-3")
LG7 = float.fromhex("0x1.2f112df3e5244p-3")
SQRT_HALF = float.fromhex("0x1.6a09e667f3bcdp-1")


def det_log(x):
    """log(x) for finite x > 0; NaN/-inf/inf follow ``numpy.log``."""
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(all="ignore"):
        return _det_log(x)


def _det_log(x):
    m, e = np.frexp(x)                      # x = m * 2**e, m in [0.5, 1)
    low = m < SQRT_HALF
    m = np.where(low, m * 2.0, m)           # m in [sqrt(1/2), sqrt(2))
    dk = (e - low.astype(np.int64)).astype(np.float64)
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    w = z * z
    t1 = w * (LG2 + w * (LG4 + w * LG6))
    t2 = z * (LG1 + w * (LG3 + w * (LG5 + w * LG7)))
    r = t2 + t1
    hfsq = 0.5 * f * f
    out = dk * LN2_HI - ((hfsq - (s * (hfsq + r) + dk * LN2_LO)) - f)
    special = ~(np.isfinite(x) & (x > 0.0))
    if np.any(special):
        out = np.where(special, np.log(x), out)
    return out if out.ndim else float(out)
