// Deterministic log and exp (device copies of oracle/detmath.py): fdlibm
// __ieee754_log / __ieee754_exp range reductions + minimax polynomials,
// evaluated with the same IEEE operations in the same order as the NumPy
// restatement, so host oracle and device agree bitwise (library built with
// -fmad=false).
#pragma once

#include <math.h>

namespace fv3b {

__device__ __forceinline__ double det_log(double x) {
  if (!(x > 0.0) || isinf(x)) return log(x);  // NaN / 0 / negative / inf follow libm
  int e;
  double m = frexp(x, &e);  // m in [0.5, 1)
  if (m < 0x1.6a09e667f3bcdp-1) {
    m = m * 2.0;
    e -= 1;
  }
  const double dk = (double)e;
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double w = z * z;
  const double t1 = w * (0x1.999999997fa04p-2 + w * (0x1.c71c51d8e78afp-3 + w * 0x1.39a09d078c69fp-3));
  const double t2 = z * (0x1.5555555555593p-1 + w * (0x1.2492494229359p-2 + w * (0x1.7466496cb03dep-3 + w * 0x1.2f112df3e5244p-3)));
  const double r = t2 + t1;
  const double hfsq = 0.5 * f * f;
  return dk * 0x1.62e42fee00000p-1 - ((hfsq - (s * (hfsq + r) + dk * 0x1.a39ef35793c76p-33)) - f);
}

// exp(x) for finite |x| <= 708; anything else follows libm
__device__ __forceinline__ double det_exp(double x) {
  if (!(fabs(x) <= 708.0)) return exp(x);  // NaN / inf / out of the normal range
  const int hx = __double2hiint(x) & 0x7fffffff;
  if (hx < 0x3e300000) return 1.0 + x;  // |x| < 2**-28
  const bool neg = x < 0.0;
  int k = 0;
  double hi = 0.0, lo = 0.0, r = x;
  if (hx > 0x3fd62e42) {   // |x| > 0.5 ln2
    if (hx < 0x3ff0a2b2) {  // |x| < 1.5 ln2
      hi = neg ? x + 0x1.62e42fee00000p-1 : x - 0x1.62e42fee00000p-1;
      lo = neg ? -0x1.a39ef35793c76p-33 : 0x1.a39ef35793c76p-33;
      k = neg ? -1 : 1;
    } else {
      k = (int)(0x1.71547652b82fep+0 * x + (neg ? -0.5 : 0.5));
      const double t = (double)k;
      hi = x - t * 0x1.62e42fee00000p-1;
      lo = t * 0x1.a39ef35793c76p-33;
    }
    r = hi - lo;
  }
  const double t = r * r;
  const double c = r - t * (0x1.555555555553ep-3 + t * (-0x1.6c16c16bebd93p-9 + t * (0x1.1566aaf25de2cp-14 +
                                                       t * (-0x1.bbd41c5d26bf1p-20 + t * 0x1.6376972bea4d0p-25))));
  if (k == 0) return 1.0 - ((r * c) / (c - 2.0) - r);
  const double y = 1.0 - ((lo - (r * c) / (2.0 - c)) - hi);
  return ldexp(y, k);
}

}  // namespace fv3b
