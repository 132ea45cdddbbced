// K1 fv_tp_2d and K7 tracer_2d: FV3 2-D finite-volume transport
// (programs/fv_tp_2d.stn, programs/tracer_2d.stn; templates.fv_tp_2d).
//
// One CTA owns a TI x TJ tile of one level and keeps every intermediate of
// the .stn statement chain in shared memory:
//
//   fy2 = yppm(q, cry)                      faces j in [0, TJ]  , i in [-3, TI+3)
//   qi  = (q*area + fy2*yfx - fy2[j+1]*yfx[j+1]) / (area + yfx - yfx[j+1])
//   fx2 = xppm(q, crx)                      faces i in [0, TI]  , j in [-3, TJ+3)
//   qj  = (q*area + fx2*xfx - fx2[i+1]*xfx[i+1]) / (area + xfx - xfx[i+1])
//   fx  = 0.5*(xppm(qi, crx) + fx2) * (xfx | mfx)
//   fy  = 0.5*(yppm(qj, cry) + fy2) * (yfx | mfy)
//   q'  = q + (fx - fx[i+1] + fy - fy[j+1]) * rarea                  (fv_tp_2d)
//   q'  = (q*dp1 + (...)*rarea) / (dp1 + (mfx - mfx[i+1] + mfy - mfy[j+1])*rarea)  (tracer)
//
// Temporaries are recomputed over the tile halo exactly as the reference
// computes them over their extension (extents.py:128-164), so every value
// that reaches an output is produced by the same IEEE operations.  The
// tracer variant loops over the tracers inside the CTA so the shared
// Courant numbers and fluxes are read from HBM once per tile.
#include "common.cuh"

namespace fv3b {

constexpr int NQMAX = 16;

// PPM face value on the low face of cell `q[0]` along stride `s`
// (templates.ppm_flux; FV3 xppm/yppm, hord=5 smoothness switch).
__device__ __forceinline__ double ppm_face(const double* q, int s, double c, double p1, double p2) {
  const double qm3 = q[-3 * s], qm2 = q[-2 * s], qm1 = q[-s], q0 = q[0], qp1 = q[s], qp2 = q[2 * s];
  const double al_m = p1 * (qm2 + qm1) + p2 * (qm3 + q0);   // al at cell i-1
  const double al_0 = p1 * (qm1 + q0) + p2 * (qm2 + qp1);   // al at cell i
  const double al_p = p1 * (q0 + qp1) + p2 * (qm1 + qp2);   // al at cell i+1
  const double bl_m = al_m - qm1, br_m = al_0 - qm1, b0_m = bl_m + br_m;
  const double bl_0 = al_0 - q0, br_0 = al_p - q0, b0_0 = bl_0 + br_0;
  const bool smooth = (fabs(3.0 * b0_m) < fabs(bl_m - br_m)) || (fabs(3.0 * b0_0) < fabs(bl_0 - br_0));
  if (c > 0.0) return qm1 + (smooth ? (1.0 - c) * (br_m - c * b0_m) : 0.0);
  return q0 + (smooth ? (1.0 + c) * (bl_0 + c * b0_0) : 0.0);
}

struct TpArgs {
  View crx, cry, xfx, yfx, area, rarea;
  View mfx, mfy, dp1;  // tracer variant only
  double* qin[NQMAX];
  double* qout[NQMAX];
  int64_t sj, sk;  // shared 3-D strides
  int nq, ni, nj, nk;
  double p1, p2;
};

template <int TI, int TJ>
struct TpSmem {
  // element counts of each tile array
  static constexpr int QW = TI + 6, QH = TJ + 6;
  static constexpr int n_q = QW * QH;
  static constexpr int n_cx = (TI + 1) * QH;   // crx, xfx, fx2
  static constexpr int n_cy = QW * (TJ + 1);   // cry, yfx, fy2
  static constexpr int n_qi = QW * TJ;
  static constexpr int n_qj = TI * QH;
  static constexpr int n_fx = (TI + 1) * TJ;
  static constexpr int n_fy = TI * (TJ + 1);
  static constexpr int total = n_q + 3 * n_cx + 3 * n_cy + n_qi + n_qj + n_fx + n_fy + n_fx + n_fy + TI * TJ;
  static constexpr size_t bytes = sizeof(double) * total;
};

template <int TI, int TJ, bool MASS>
__global__ void __launch_bounds__(256) tp_kernel(TpArgs a) {
  using S = TpSmem<TI, TJ>;
  extern __shared__ double smem[];
  const int NT = blockDim.x, tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ, k = blockIdx.z;
  double* p = smem;
  const STile sq{p, -3, -3, S::QW};           p += S::n_q;
  const STile scrx{p, 0, -3, TI + 1};        p += S::n_cx;
  const STile sxfx{p, 0, -3, TI + 1};        p += S::n_cx;
  const STile sfx2{p, 0, -3, TI + 1};        p += S::n_cx;
  const STile scry{p, -3, 0, S::QW};         p += S::n_cy;
  const STile syfx{p, -3, 0, S::QW};         p += S::n_cy;
  const STile sfy2{p, -3, 0, S::QW};         p += S::n_cy;
  const STile sqi{p, -3, 0, S::QW};          p += S::n_qi;
  const STile sqj{p, 0, -3, TI};             p += S::n_qj;
  const STile sfx{p, 0, 0, TI + 1};          p += S::n_fx;
  const STile sfy{p, 0, 0, TI};              p += S::n_fy;
  const STile swx{p, 0, 0, TI + 1};          p += S::n_fx;   // flux weight xfx | mfx on faces
  const STile swy{p, 0, 0, TI};              p += S::n_fy;   // flux weight yfx | mfy on faces
  const STile sdp2{p, 0, 0, TI};

  const int ni = a.ni, nj = a.nj;
  auto inside = [&](int li, int lj, int hi_lo, int hi_hi, int hj_lo, int hj_hi) {
    const int gi = gi0 + li, gj = gj0 + lj;
    return gi >= -hi_lo && gi < ni + hi_hi && gj >= -hj_lo && gj < nj + hj_hi;
  };

  // --- shared inputs: Courant numbers and area fluxes ---------------------
  for (int e = tid; e < S::n_cx; e += NT) {
    const int li = e % (TI + 1), lj = e / (TI + 1) - 3;
    const bool ok = inside(li, lj, 0, 1, 3, 3);
    scrx(li, lj) = ok ? a.crx(gi0 + li, gj0 + lj, k) : 0.0;
    sxfx(li, lj) = ok ? a.xfx(gi0 + li, gj0 + lj, k) : 0.0;
  }
  for (int e = tid; e < S::n_cy; e += NT) {
    const int li = e % S::QW - 3, lj = e / S::QW;
    const bool ok = inside(li, lj, 3, 3, 0, 1);
    scry(li, lj) = ok ? a.cry(gi0 + li, gj0 + lj, k) : 0.0;
    syfx(li, lj) = ok ? a.yfx(gi0 + li, gj0 + lj, k) : 0.0;
  }
  for (int e = tid; e < S::n_fx; e += NT) {
    const int li = e % (TI + 1), lj = e / (TI + 1);
    const bool ok = inside(li, lj, 0, 1, 0, 0);
    swx(li, lj) = ok ? (MASS ? a.mfx(gi0 + li, gj0 + lj, k) : sxfx(li, lj)) : 0.0;
  }
  for (int e = tid; e < S::n_fy; e += NT) {
    const int li = e % TI, lj = e / TI;
    const bool ok = inside(li, lj, 0, 0, 0, 1);
    swy(li, lj) = ok ? (MASS ? a.mfy(gi0 + li, gj0 + lj, k) : syfx(li, lj)) : 0.0;
  }
  __syncthreads();
  if (MASS) {
    // dp2 = dp1 + (mfx - mfx[1,0,0] + mfy - mfy[0,1,0]) * rarea   (tracer_dp)
    for (int e = tid; e < TI * TJ; e += NT) {
      const int li = e % TI, lj = e / TI;
      if (!inside(li, lj, 0, 0, 0, 0)) continue;
      const int gi = gi0 + li, gj = gj0 + lj;
      sdp2(li, lj) = a.dp1(gi, gj, k) + (swx(li, lj) - swx(li + 1, lj) + swy(li, lj) - swy(li, lj + 1)) * a.rarea(gi, gj, 0);
    }
  }

  const double p1 = a.p1, p2 = a.p2;
  for (int t = 0; t < a.nq; ++t) {
    const View q{a.qin[t], a.sj, a.sk};
    const View qo{a.qout[t], a.sj, a.sk};
    for (int e = tid; e < S::n_q; e += NT) {
      const int li = e % S::QW - 3, lj = e / S::QW - 3;
      sq(li, lj) = inside(li, lj, 3, 3, 3, 3) ? q(gi0 + li, gj0 + lj, k) : 0.0;
    }
    __syncthreads();
    // fy2 = yppm(q, cry) on faces j in [0, TJ], i in [-3, TI+3)
    for (int e = tid; e < S::n_cy; e += NT) {
      const int li = e % S::QW - 3, lj = e / S::QW;
      sfy2(li, lj) = ppm_face(&sq(li, lj), S::QW, scry(li, lj), p1, p2);
    }
    // fx2 = xppm(q, crx) on faces i in [0, TI], j in [-3, TJ+3)
    for (int e = tid; e < S::n_cx; e += NT) {
      const int li = e % (TI + 1), lj = e / (TI + 1) - 3;
      sfx2(li, lj) = ppm_face(&sq(li, lj), 1, scrx(li, lj), p1, p2);
    }
    __syncthreads();
    // qi over i in [-3, TI+3), j in [0, TJ); qj over i in [0, TI), j in [-3, TJ+3)
    for (int e = tid; e < S::n_qi; e += NT) {
      const int li = e % S::QW - 3, lj = e / S::QW;
      const double ar = inside(li, lj, 3, 3, 0, 0) ? a.area(gi0 + li, gj0 + lj, 0) : 0.0;
      sqi(li, lj) = (sq(li, lj) * ar + sfy2(li, lj) * syfx(li, lj) - sfy2(li, lj + 1) * syfx(li, lj + 1)) /
                    (ar + syfx(li, lj) - syfx(li, lj + 1));
    }
    for (int e = tid; e < S::n_qj; e += NT) {
      const int li = e % TI, lj = e / TI - 3;
      const double ar = inside(li, lj, 0, 0, 3, 3) ? a.area(gi0 + li, gj0 + lj, 0) : 0.0;
      sqj(li, lj) = (sq(li, lj) * ar + sfx2(li, lj) * sxfx(li, lj) - sfx2(li + 1, lj) * sxfx(li + 1, lj)) /
                    (ar + sxfx(li, lj) - sxfx(li + 1, lj));
    }
    __syncthreads();
    // fx = 0.5*(xppm(qi) + fx2) * w ;  fy = 0.5*(yppm(qj) + fy2) * w
    for (int e = tid; e < S::n_fx; e += NT) {
      const int li = e % (TI + 1), lj = e / (TI + 1);
      const double fx1 = ppm_face(&sqi(li, lj), 1, scrx(li, lj), p1, p2);
      sfx(li, lj) = 0.5 * (fx1 + sfx2(li, lj)) * swx(li, lj);
    }
    for (int e = tid; e < S::n_fy; e += NT) {
      const int li = e % TI, lj = e / TI;
      const double fy1 = ppm_face(&sqj(li, lj), TI, scry(li, lj), p1, p2);
      sfy(li, lj) = 0.5 * (fy1 + sfy2(li, lj)) * swy(li, lj);
    }
    __syncthreads();
    for (int e = tid; e < TI * TJ; e += NT) {
      const int li = e % TI, lj = e / TI;
      if (!inside(li, lj, 0, 0, 0, 0)) continue;
      const int gi = gi0 + li, gj = gj0 + lj;
      const double div = (sfx(li, lj) - sfx(li + 1, lj) + sfy(li, lj) - sfy(li, lj + 1)) * a.rarea(gi, gj, 0);
      if (MASS)
        qo(gi, gj, k) = (sq(li, lj) * a.dp1(gi, gj, k) + div) / sdp2(li, lj);
      else
        qo(gi, gj, k) = sq(li, lj) + div;
    }
    __syncthreads();
  }
}

template <bool MASS>
static int launch_tp(const TpArgs& a, cudaStream_t st) {
  constexpr int TI = 32, TJ = 16;
  using S = TpSmem<TI, TJ>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tp_kernel<TI, TJ, MASS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
    attr = true;
  }
  dim3 grid(cdiv(a.ni, TI), cdiv(a.nj, TJ), a.nk);
  tp_kernel<TI, TJ, MASS><<<grid, 256, S::bytes, st>>>(a);
  return check_launch(MASS ? "tracer_2d" : "fv_tp_2d");
}

}  // namespace fv3b

using namespace fv3b;

extern "C" int fv3b_fv_tp_2d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                             void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 8 || ns != 2)
    return fail(FV3B_EINVAL, "fv3b_fv_tp_2d: expects 8 fields, 2 scalars (got %d, %d)", nf, ns);
  TpArgs a{};
  View q, qo;
  const Halo hq = {3, 3, 3, 3, 0, 0}, hx = {0, 1, 3, 3, 0, 0}, hy = {3, 3, 0, 1, 0, 0}, h0 = {0, 0, 0, 0, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, hq, "q", &q));
  FV3B_TRY(view_of(f[1], 3, *d, hx, "crx", &a.crx));
  FV3B_TRY(view_of(f[2], 3, *d, hy, "cry", &a.cry));
  FV3B_TRY(view_of(f[3], 3, *d, hx, "xfx", &a.xfx));
  FV3B_TRY(view_of(f[4], 3, *d, hy, "yfx", &a.yfx));
  FV3B_TRY(view_of(f[5], 2, *d, hq, "area", &a.area));
  FV3B_TRY(view_of(f[6], 2, *d, h0, "rarea", &a.rarea));
  FV3B_TRY(view_of(f[7], 3, *d, h0, "q_out", &qo));
  const View v3[6] = {q, a.crx, a.cry, a.xfx, a.yfx, qo};
  FV3B_TRY(same_strides(v3, 6, "fv3b_fv_tp_2d"));
  if (f[7].data == f[0].data) return fail(FV3B_EINVAL, "fv3b_fv_tp_2d: q_out must not alias q");
  a.qin[0] = q.o;
  a.qout[0] = qo.o;
  a.sj = q.sj;
  a.sk = q.sk;
  a.nq = 1;
  a.ni = d->ni; a.nj = d->nj; a.nk = d->nk;
  a.p1 = s[0];
  a.p2 = s[1];
  if (a.ni <= 0 || a.nj <= 0 || a.nk <= 0) return FV3B_OK;
  return launch_tp<false>(a, (cudaStream_t)stream);
}

extern "C" int fv3b_tracer_2d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                              void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || ns != 2 || nf < 11 || (nf - 9) % 2 != 0 || (nf - 9) / 2 > NQMAX)
    return fail(FV3B_EINVAL, "fv3b_tracer_2d: expects 9 + 2*nq fields (nq <= %d), 2 scalars", NQMAX);
  const int nq = (nf - 9) / 2;
  TpArgs a{};
  const Halo hq = {3, 3, 3, 3, 0, 0}, hx = {0, 1, 3, 3, 0, 0}, hy = {3, 3, 0, 1, 0, 0}, h0 = {0, 0, 0, 0, 0, 0};
  const Halo hmx = {0, 1, 0, 0, 0, 0}, hmy = {0, 0, 0, 1, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, hx, "cx", &a.crx));
  FV3B_TRY(view_of(f[1], 3, *d, hy, "cy", &a.cry));
  FV3B_TRY(view_of(f[2], 3, *d, hx, "xfx", &a.xfx));
  FV3B_TRY(view_of(f[3], 3, *d, hy, "yfx", &a.yfx));
  FV3B_TRY(view_of(f[4], 3, *d, hmx, "mfx", &a.mfx));
  FV3B_TRY(view_of(f[5], 3, *d, hmy, "mfy", &a.mfy));
  FV3B_TRY(view_of(f[6], 3, *d, h0, "dp1", &a.dp1));
  FV3B_TRY(view_of(f[7], 2, *d, hq, "area", &a.area));
  FV3B_TRY(view_of(f[8], 2, *d, h0, "rarea", &a.rarea));
  View v3[7 + 2 * NQMAX];
  v3[0] = a.crx; v3[1] = a.cry; v3[2] = a.xfx; v3[3] = a.yfx; v3[4] = a.mfx; v3[5] = a.mfy; v3[6] = a.dp1;
  for (int t = 0; t < nq; ++t) {
    char nm[32];
    snprintf(nm, sizeof nm, "q%d", t);
    FV3B_TRY(view_of(f[9 + t], 3, *d, hq, nm, &v3[7 + t]));
    snprintf(nm, sizeof nm, "q%d_out", t);
    FV3B_TRY(view_of(f[9 + nq + t], 3, *d, h0, nm, &v3[7 + nq + t]));
    if (f[9 + t].data == f[9 + nq + t].data) return fail(FV3B_EINVAL, "fv3b_tracer_2d: q%d_out aliases q%d", t, t);
    a.qin[t] = v3[7 + t].o;
    a.qout[t] = v3[7 + nq + t].o;
  }
  FV3B_TRY(same_strides(v3, 7 + 2 * nq, "fv3b_tracer_2d"));
  a.sj = a.crx.sj;
  a.sk = a.crx.sk;
  a.nq = nq;
  a.ni = d->ni; a.nj = d->nj; a.nk = d->nk;
  a.p1 = s[0];
  a.p2 = s[1];
  if (a.ni <= 0 || a.nj <= 0 || a.nk <= 0) return FV3B_OK;
  return launch_tp<true>(a, (cudaStream_t)stream);
}
