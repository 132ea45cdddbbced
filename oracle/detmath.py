"""Deterministic ``log`` (the documented oracle extension) and ``exp`` (the
post-remap pressure diagnostics, oracle/thermo.py).

TEST INFRASTRUCTURE (imported by ``oracle/interp.py`` and ``tests/_ref.py``).

The reference DSL has no ``log`` (``frontend/ast.py:28``); the extension adds
one.  Its semantics are fixed here as an explicit IEEE-754 algorithm so that
every engine that evaluates it with the same operations in the same order
(NumPy on the host, CUDA with ``-fmad=false`` on the device) produces the
same bits: the range reduction and minimax polynomial of fdlibm's
``__ieee754_log`` (Sun Microsystems, 1993), error < 1 ulp, restated with
only ``frexp``, ``+ - * /``; ``det_exp`` likewise restates fdlibm's
``__ieee754_exp`` (argument reduction by k*ln2 in two parts, the degree-5
Remez polynomial for the reduced argument, exact scaling by 2**k).
``csrc/detmath.cuh`` is the device copy.
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


INVLN2 = float.fromhex("0x1.71547652b82fep+0")
P1 = float.fromhex("0x1.555555555553ep-3")
P2 = float.fromhex("-0x1.6c16c16bebd93p-9")
P3 = float.fromhex("0x1.1566aaf25de2cp-14")
P4 = float.fromhex("-0x1.bbd41c5d26bf1p-20")
P5 = float.fromhex("0x1.6376972bea4d0p-25")
EXP_MAX = 708.0  # |x| above this: the scaling could leave the normal range


def det_exp(x):
    """exp(x) for finite |x| <= 708 (fdlibm __ieee754_exp); anything else
    follows ``numpy.exp``."""
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(all="ignore"):
        return _det_exp(x)


def _det_exp(x):
    hx = (x.view(np.int64) >> 32).astype(np.int64) & 0x7FFFFFFF
    neg = x < 0.0
    # |x| in (0.5 ln2, 1.5 ln2): k = +-1 with the two-part ln2
    near = (hx > 0x3FD62E42) & (hx < 0x3FF0A2B2)
    far = hx >= 0x3FF0A2B2
    kf = (INVLN2 * x + np.where(neg, -0.5, 0.5)).astype(np.int64)
    k = np.where(near, np.where(neg, -1, 1), np.where(far, kf, 0))
    t = k.astype(np.float64)
    hi_near = np.where(neg, x + LN2_HI, x - LN2_HI)
    lo_near = np.where(neg, -LN2_LO, LN2_LO)
    hi = np.where(near, hi_near, x - t * LN2_HI)
    lo = np.where(near, lo_near, t * LN2_LO)
    red = np.where(near | far, hi - lo, x)
    t2 = red * red
    c = red - t2 * (P1 + t2 * (P2 + t2 * (P3 + t2 * (P4 + t2 * P5))))
    y0 = 1.0 - ((red * c) / (c - 2.0) - red)            # k == 0
    y1 = 1.0 - ((lo - (red * c) / (2.0 - c)) - hi)      # k != 0
    out = np.where(k == 0, y0, np.ldexp(y1, k.astype(np.int32)))
    tiny = hx < 0x3E300000                              # |x| < 2**-28
    out = np.where(tiny, 1.0 + x, out)
    special = ~(np.isfinite(x) & (np.abs(x) <= EXP_MAX))
    if np.any(special):
        out = np.where(special, np.exp(x), out)
    return out if out.ndim else float(out)
