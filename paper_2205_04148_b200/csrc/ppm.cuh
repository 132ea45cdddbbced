// Register sliding-window PPM face values (templates.ppm_flux; FV3
// xppm/yppm with the hord=5 smoothness switch).
//
// For NF consecutive faces f = 0..NF-1 along a line (face f lies between
// cells f-1 and f) the statement chain of the .stn source is evaluated with
// each edge value `al` and each per-cell quantity (bl, br, b0, sm) computed
// once and reused by both neighbouring faces:
//
//   al = ppm_p1 * (Q[-1] + Q) + ppm_p2 * (Q[-2] + Q[1])
//   bl = al - Q ; br = al[1] - Q ; b0 = bl + br
//   sm = select(abs(3.0 * b0) < abs(bl - br), 1.0, 0.0)
//   F  = select(C > 0.0, Q[-1] + select(sm[-1] + sm > 0.0, (1.0 - C) * (br[-1] - C * b0[-1]), 0.0),
//                        Q    + select(sm[-1] + sm > 0.0, (1.0 + C) * (bl + C * b0), 0.0))
//
// `q` points at cell 0 (q[d * s] is cell d, needs d in [-3, NF+2)), `c` at
// the Courant number of face 0 (c[f * cs]).  With NC > 0 the cell values
// 0 .. NC-1 of the window are also returned in `qc` (the inner-update
// numerators reuse them instead of reloading shared memory).
#pragma once

namespace fv3b {

template <int NF, int NC = 0>
__device__ __forceinline__ void ppm_line(const double* q, int s, const double* c, int cs, double p1, double p2,
                                         double* out, double* qc = nullptr) {
  static_assert(NC <= NF + 2, "centre values lie in the window");
  double qv[NF + 5];  // cells -3 .. NF+1
#pragma unroll
  for (int d = 0; d < NF + 5; ++d) qv[d] = q[(d - 3) * s];
  if constexpr (NC > 0) {
#pragma unroll
    for (int u = 0; u < NC; ++u) qc[u] = qv[u + 3];
  }
  double al[NF + 2];  // cells -1 .. NF
#pragma unroll
  for (int m = 0; m < NF + 2; ++m) {
    // cell m-1: p1*(q(m-2) + q(m-1)) + p2*(q(m-3) + q(m))
    al[m] = p1 * (qv[m + 1] + qv[m + 2]) + p2 * (qv[m] + qv[m + 3]);
  }
  double bl[NF + 1], br[NF + 1], b0[NF + 1];
  bool sm[NF + 1];  // cells -1 .. NF-1
#pragma unroll
  for (int m = 0; m < NF + 1; ++m) {
    const double qc = qv[m + 2];  // cell m-1
    bl[m] = al[m] - qc;
    br[m] = al[m + 1] - qc;
    b0[m] = bl[m] + br[m];
    sm[m] = fabs(3.0 * b0[m]) < fabs(bl[m] - br[m]);
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    // Only the selected upwind candidate is evaluated (select() has no side
    // effects, so dropping the other branch changes nothing), with operand
    // selects instead of two evaluations: for cc > 0 the candidate is
    // (1 - cc) * (br[f] - cc * b0[f]) = (1 + m) * (br[f] + m * b0[f]) with
    // m = -cc, exactly (x - y == x + (-y) and (-cc) * b == -(cc * b) in IEEE).
    const double cc = c[f * cs];
    const bool smooth = sm[f] || sm[f + 1];  // cells f-1, f
    const bool pos = cc > 0.0;
    const double m = pos ? -cc : cc;
    const double t = (1.0 + m) * ((pos ? br[f] : bl[f + 1]) + m * (pos ? b0[f] : b0[f + 1]));
    const double base = pos ? qv[f + 2] : qv[f + 3];
    out[f] = base + (smooth ? t : 0.0);
  }
}

}  // namespace fv3b
