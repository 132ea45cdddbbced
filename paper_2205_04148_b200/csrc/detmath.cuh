// Deterministic log (device copy of oracle/detmath.py): fdlibm
// __ieee754_log range reduction + minimax polynomial, evaluated with the
// same IEEE operations in the same order as the NumPy restatement, so host
// oracle and device agree bitwise (library built with -fmad=false).
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

}  // namespace fv3b
