// K3b d_sw momentum group (programs/d_sw.stn: d_sw_courant, d_sw_ke,
// d_sw_vort, d_sw_damp and the u / v statements of d_sw_update) as one
// level-marching, TMA-pipelined kernel (the transport kernel's machinery,
// dsw_transport.cu).  Per level:
//
//   S0  courant (crx, xfx, cry, yfx) and the absolute vorticity wk over the
//       tile halo, from the staged uc / vc / u / v tiles and the metrics;
//   S1  phase A of fv_tp_2d(wk) (yppm -> fy2, qi ; xppm -> fx2, qj), the
//       kinetic-energy upwind values ub*uu (xppm of u with cub) and vb*vv
//       (yppm of v with cvb) at cell corners, and the Smagorinsky-scaled
//       divergence damping ddv at corners;
//   S2  phase B of fv_tp_2d(wk) -> fxv, fyv (smem; fyv in place of the
//       phase-A y fluxes) and ked = 0.5 * (ub*uu + vb*vv);
//   S3  (during the next level's S0, before its stage wait) the u / v
//       updates, every thread a share of the tile's cells.
//
// The vorticity flux carries its del6 damping (templates.delnflux on wk with
// dampv, nord = 2): order 1 of the Laplacian chain (d2_v1, each cell forming
// its four order-0 face fluxes from dampv * wk) runs in S1, order 2 (d2_v2)
// in S2, and the u / v updates add the last order's face fluxes to fxv /
// fyv.
//
// Every statement keeps the .stn operand order and association (ked is
// 0.5 * (ub*uu + vb*vv) with both products rounded as in the interpreter),
// so results are bitwise the reference's.
#include "common.cuh"
#include "dsw.cuh"
#include "fastdiv.cuh"
#include "ppm.cuh"
#include "tma.cuh"

namespace fv3b {

namespace {

constexpr int SEG = 4;
#ifndef FV3B_MO_NT
#define FV3B_MO_NT 352
#endif
template <int TJ> constexpr int nt_of() { return TJ >= 16 ? FV3B_MO_NT : 256; }
template <int TJ> constexpr int cps_of() { return TJ >= 16 ? 1 : 2; }

__host__ __device__ constexpr int a16(int n) { return (n + 15) / 16 * 16; }

// numpy minimum / maximum (NaN-propagating, reference.py:247-257)
__device__ __forceinline__ double np_min(double a, double b) {
  if (isnan(a) || isnan(b)) return a + b;
  return b < a ? b : a;
}
__device__ __forceinline__ double np_max(double a, double b) {
  if (isnan(a) || isnan(b)) return a + b;
  return b > a ? b : a;
}

template <int TI, int TJ>
struct MoLayout {
  static constexpr int QW = TI + 10, QH = TJ + 6;  // q-box: i in [-4, TI+6), j in [-3, TJ+3)
  static constexpr int XW = TI + 2, XH = TJ + 6;   // x faces: i in [0, TI+2), j in [-3, TJ+3)
  static constexpr int YW = TI + 8, YH = TJ + 1;   // y faces: i in [-4, TI+4), j in [0, TJ+1)
  static constexpr int JW = TI + 2;                // qj row width
  static constexpr int CW = TI + 2, CH = TJ + 1;   // corners: i in [0, TI+2), j in [0, TJ+1)
  static constexpr int D1W = TI + 3, D1H = TJ + 3; // d2_v1: [-2, TI+1) x [-2, TJ+1)
  static constexpr int D2W = TI + 1, D2H = TJ + 1; // d2_v2: [-1, TI) x [-1, TJ)
  static constexpr int n_q = a16(QW * QH), n_q1 = a16(QW * (QH + 1));
  static constexpr int n_x = a16(XW * XH), n_y = a16(YW * YH);
  static constexpr int n_mx = a16(XW * TJ), n_my = a16(TI * YH);
  static constexpr int n_qi = a16(QW * TJ), n_qj = a16(JW * QH);
  static constexpr int n_cn = a16(CW * CH);
  static constexpr int n_stage = n_q1 + 3 * n_q;        // u (+1 row), v, uc, vc
  static constexpr int o_stage = 0;
  static constexpr int o_met = 2 * n_stage;              // dx (+1 row), then 11 q-box metrics
  static constexpr int o_crx = o_met + n_q1 + 11 * n_q;
  static constexpr int o_xfx = o_crx + n_x;
  static constexpr int o_cry = o_xfx + n_x;
  static constexpr int o_yfx = o_cry + n_y;
  static constexpr int o_wk = o_yfx + n_y;
  static constexpr int o_ked = o_wk + n_q;               // ub*uu, then ked
  static constexpr int o_vv = o_ked + n_cn;              // vb*vv
  static constexpr int o_ddv = o_vv + n_cn;
  static constexpr int o_qi = o_ddv + n_cn;
  static constexpr int o_qj = o_qi + n_qi;
  static constexpr int o_fx2 = o_qj + n_qj;
  static constexpr int o_fy2 = o_fx2 + n_mx;
  static constexpr int o_fx = o_fy2 + n_my;
  static constexpr int o_d1 = o_fx + n_mx;
  static constexpr int o_d2 = o_d1 + a16(D1W * D1H);
  static constexpr int total = o_d2 + a16(D2W * D2H);
  static constexpr size_t bytes = total * sizeof(double) + 64;
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static_assert(TJ % SEG == 0 && TI % SEG == 0 && QW % 4 == 2 && XW % 4 == 2 && JW % 4 == 2, "tile shape");
  static constexpr uint32_t tx_stage = (QW * (QH + 1) + 3 * QW * QH) * 8;
  static constexpr uint32_t tx_met = (QW * (QH + 1) + 11 * QW * QH) * 8;
};

template <int TI, int TJ>
__global__ void __launch_bounds__(nt_of<TJ>(), cps_of<TJ>()) dsw_momentum_kernel(const __grid_constant__ DswMoArgs a) {
  using L = MoLayout<TI, TJ>;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::total);
  const int tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ;
  const int k0 = blockIdx.z * a.kchunk;
  const int k1 = min(a.nk, k0 + a.kchunk);
  const int xq = a.i0 + gi0 - 4, yq = a.j0 + gj0 - 3;
  const double p1 = a.p1, p2 = a.p2, dt = a.dt;

  auto issue = [&](int k) {
    const int b = (k - k0) & 1;
    double* st = smem + L::o_stage + b * L::n_stage;
    mbar_expect_tx(&bar[b], L::tx_stage);
    tma_load3(st, &a.u, xq, yq, k, &bar[b]);
    tma_load3(st + L::n_q1, &a.v, xq, yq, k, &bar[b]);
    tma_load3(st + L::n_q1 + L::n_q, &a.uc, xq, yq, k, &bar[b]);
    tma_load3(st + L::n_q1 + 2 * L::n_q, &a.vc, xq, yq, k, &bar[b]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && k1 > k0) {
    mbar_expect_tx(&bar[2], L::tx_met);
    tma_load3(smem + L::o_met, &a.met[0], xq, yq, 0, &bar[2]);
#pragma unroll
    for (int f = 1; f < 12; ++f) tma_load3(smem + L::o_met + L::n_q1 + (f - 1) * L::n_q, &a.met[f], xq, yq, 0, &bar[2]);
    issue(k0);
  }
  const double* sdx = smem + L::o_met;
  const double* sdy = sdx + L::n_q1;
  const double* srdxa = sdy + L::n_q;
  const double* srdya = srdxa + L::n_q;
  const double* sarea = srdya + L::n_q;
  const double* sf0 = sarea + L::n_q;
  const double* srarea = sf0 + L::n_q;
  const double* srdx = srarea + L::n_q;
  const double* srdy = srdx + L::n_q;
  const double* sdxc = srdy + L::n_q;
  const double* sdyc = sdxc + L::n_q;
  const double* srac = sdyc + L::n_q;
  double* scrx = smem + L::o_crx;
  double* sxfx = smem + L::o_xfx;
  double* scry = smem + L::o_cry;
  double* syfx = smem + L::o_yfx;
  double* swk = smem + L::o_wk;    // q-box geometry
  double* sked = smem + L::o_ked;  // corners: ub*uu, then ked
  double* svv = smem + L::o_vv;    // corners: vb*vv
  double* sddv = smem + L::o_ddv;  // corners
  double* sqi = smem + L::o_qi;
  double* sqj = smem + L::o_qj;
  double* sfx2 = smem + L::o_fx2;
  double* sfy2 = smem + L::o_fy2;
  double* sfx = smem + L::o_fx;
  double* sd1 = smem + L::o_d1;
  double* sd2 = smem + L::o_d2;
  auto D1 = [&](int i, int j) { return sd1 + (j + 2) * L::D1W + (i + 2); };
  auto D2 = [&](int i, int j) { return sd2 + (j + 1) * L::D2W + (i + 1); };
  // del6 metrics straight from L1 / L2 (tile-local (i, j); 2-D, J stride sj)
  const double* gd6u = a.del6_u + gi0 + (int64_t)gj0 * a.sj;
  const double* gd6v = a.del6_v + gi0 + (int64_t)gj0 * a.sj;
  // del6 order 1 / 2 loads of a ragged edge tile are clamped into the
  // allocation (the cells beyond it are outside every owned cell's stencil)
  const int64_t mlo = a.mlo - (gi0 + (int64_t)gj0 * a.sj), mhi = a.mhi - (gi0 + (int64_t)gj0 * a.sj) - a.sj;
  const double dampv = a.dampv;
  auto QB = [&](auto* p, int i, int j) { return p + (j + 3) * L::QW + (i + 4); };
  auto CX = [&](auto* p, int i, int j) { return p + (j + 3) * L::XW + i; };
  auto CY = [&](auto* p, int i, int j) { return p + j * L::YW + (i + 4); };
  auto CN = [&](auto* p, int i, int j) { return p + j * L::CW + i; };
  if (k1 > k0) mbar_wait(&bar[2], 0);

  constexpr int NSEG = TI / SEG;
  constexpr int NX2 = TJ * NSEG, NY2 = TI * (TJ / SEG);
  static_assert(NX2 + NY2 <= nt_of<TJ>(), "one item per thread in phase B");
  const bool yth = tid >= NX2 && tid < NX2 + NY2;
  const int ci2 = yth ? (tid - NX2) % TI : 0;
  const int jb2 = yth ? ((tid - NX2) / TI) * SEG : 0;
  double fy[SEG + 1];
  int pend_k = -1;
  const int64_t sj = a.sj, sk = a.sk;

  // u / v updates of the previous level, every thread a share of the tile's
  // cells (the weighted y fluxes wait in sfy2, which the next phase A rewrites)
  const double* sfyv = sfy2;
  auto write_pending = [&]() {
    if (pend_k < 0) return;
    const double* st = smem + L::o_stage + ((pend_k - k0) & 1) * L::n_stage;
    const double* U = st;
    const double* V = st + L::n_q1;
    for (int e = tid; e < TI * TJ; e += blockDim.x) {
      const int i = e % TI, j = e / TI, gi = gi0 + i, gj = gj0 + j;
      if (gi < a.ni && gj < a.nj) {
        const int64_t off = gi + gj * sj + (int64_t)pend_k * sk;
        const double rdx = *QB(srdx, i, j), rdy = *QB(srdy, i, j);
        const int64_t m = i + j * sj;
        // fyv / fxv + their del6 increments dfy_v2 / dfx_v2
        const double fyv = sfyv[j * TI + i] + __ldg(gd6u + m) * (*D2(i, j) - *D2(i, j - 1));
        const double fxv = sfx[j * L::XW + i] + __ldg(gd6v + m) * (*D2(i, j) - *D2(i - 1, j));
        a.uo[off] = (*QB(U, i, j) * *QB(sdx, i, j) + *CN(sked, i, j) - *CN(sked, i + 1, j) + fyv) * rdx +
                    (*CN(sddv, i + 1, j) - *CN(sddv, i, j)) * rdx;
        a.vo[off] = (*QB(V, i, j) * *QB(sdy, i, j) + *CN(sked, i, j) - *CN(sked, i, j + 1) - fxv) * rdy +
                    (*CN(sddv, i, j + 1) - *CN(sddv, i, j)) * rdy;
      }
    }
  };

  for (int k = k0; k < k1; ++k) {
    const double* st = smem + L::o_stage + ((k - k0) & 1) * L::n_stage;
    const double* U = st;
    const double* V = st + L::n_q1;
    const double* UC = st + L::n_q1 + L::n_q;
    const double* VC = st + L::n_q1 + 2 * L::n_q;

    // ---- S0: previous level's u/v; courant; vorticity ---------------------
    write_pending();
    mbar_wait(&bar[(k - k0) & 1], ((k - k0) >> 1) & 1);
    for (int e = tid; e < L::XW * L::XH; e += blockDim.x) {
      const int i = e % L::XW, j = e / L::XW - 3;
      const double uc = *QB(UC, i, j);
      *CX(sxfx, i, j) = dt * uc * *QB(sdy, i, j);
      *CX(scrx, i, j) = uc > 0.0 ? dt * uc * *QB(srdxa, i - 1, j) : dt * uc * *QB(srdxa, i, j);
    }
    for (int e = tid; e < L::YW * L::YH; e += blockDim.x) {
      const int i = e % L::YW - 4, j = e / L::YW;
      const double vc = *QB(VC, i, j);
      *CY(syfx, i, j) = dt * vc * *QB(sdx, i, j);
      *CY(scry, i, j) = vc > 0.0 ? dt * vc * *QB(srdya, i, j - 1) : dt * vc * *QB(srdya, i, j);
    }
    // wk = f0 + rarea * (u*dx - u[0,1,0]*dx[0,1] + v[1,0,0]*dy[1,0] - v*dy) over [-3, TI+3) x [-3, TJ+3)
    for (int e = tid; e < (TI + 6) * (TJ + 6); e += blockDim.x) {
      const int i = e % (TI + 6) - 3, j = e / (TI + 6) - 3;
      *QB(swk, i, j) = *QB(sf0, i, j) + *QB(srarea, i, j) * (*QB(U, i, j) * *QB(sdx, i, j) -
                                                            *QB(U, i, j + 1) * *QB(sdx, i, j + 1) +
                                                            *QB(V, i + 1, j) * *QB(sdy, i + 1, j) -
                                                            *QB(V, i, j) * *QB(sdy, i, j));
    }
    __syncthreads();

    // ---- S1: phase A of fv_tp_2d(wk); ke upwind values; divergence damping --
    if (tid == 0 && k + 1 < k1) {
      fence_async_smem();
      issue(k + 1);
    }
    {
      constexpr int NCY = TI + 6, NSY = TJ / SEG;
      constexpr int NRX = TJ + 6, NSX = TI / SEG;
      constexpr int NY = NCY * NSY, NX = NRX * NSX;
      constexpr int NU = (TJ + 1) * NSEG;   // ub*uu rows j in [0, TJ+1), faces [0, TI+1)
      constexpr int NV = (TI + 1) * (TJ / SEG);  // vb*vv columns i in [0, TI+1), faces [0, TJ+1)
      constexpr int ND = (TI + 1) * (TJ + 1);    // ddv corners
      constexpr int N1 = L::D1W * L::D1H;        // d2_v1 cells
      for (int item = tid; item < NY + NX + NU + NV + ND + N1; item += blockDim.x) {
        if (item >= NY + NX + NU + NV + ND) {
          // d2_v0 = dampv * wk ; dfx_v0 = del6_v * (d2_v0[-1,0] - d2_v0) ; d2_v1 = div(dfx_v0, dfy_v0) * rarea
          const int e = item - (NY + NX + NU + NV + ND);
          const int i = e % L::D1W - 2, j = e / L::D1W - 2;
          const int64_t m = min(max(i + j * sj, mlo), mhi);
          const double v0 = __ldg(gd6v + m), v1 = __ldg(gd6v + m + 1), u0 = __ldg(gd6u + m), u1 = __ldg(gd6u + m + sj);
          const double c = dampv * *QB(swk, i, j), wq = dampv * *QB(swk, i - 1, j), eq = dampv * *QB(swk, i + 1, j);
          const double sq = dampv * *QB(swk, i, j - 1), nq = dampv * *QB(swk, i, j + 1);
          const double fx0 = v0 * (wq - c), fx1 = v1 * (c - eq), fy0 = u0 * (sq - c), fy1 = u1 * (c - nq);
          *D1(i, j) = (fx0 - fx1 + fy0 - fy1) * *QB(srarea, i, j);
          continue;
        }
        if (item < NY) {
          const int ci = item % NCY - 3, jb = (item / NCY) * SEG;
          double f[SEG + 1];
          ppm_line<SEG + 1>(QB(swk, ci, jb), L::QW, CY(scry, ci, jb), L::YW, p1, p2, f);
          // branch-free fast-path quotients, one exact fallback per item (fastdiv.cuh)
          double num[SEG], den[SEG], v[SEG];
          bool ok = true;
#pragma unroll
          for (int u = 0; u < SEG; ++u) {
            const int j = jb + u;
            const double ar = *QB(sarea, ci, j);
            const double y0 = *CY(syfx, ci, j), y1 = *CY(syfx, ci, j + 1);
            num[u] = *QB(swk, ci, j) * ar + f[u] * y0 - f[u + 1] * y1;
            den[u] = ar + y0 - y1;
            v[u] = div_fast(num[u], den[u], ok);
          }
          if (!ok)
#pragma unroll
            for (int u = 0; u < SEG; ++u) v[u] = num[u] / den[u];
#pragma unroll
          for (int u = 0; u < SEG; ++u) sqi[(jb + u) * L::QW + ci + 4] = v[u];
          if (ci >= 0 && ci < TI) {
#pragma unroll
            for (int u = 0; u < SEG; ++u) sfy2[(jb + u) * TI + ci] = f[u];
            if (jb + SEG == TJ) sfy2[TJ * TI + ci] = f[SEG];
          }
        } else if (item < NY + NX) {
          const int it = item - NY;
          const int rj = it % NRX - 3, ib = (it / NRX) * SEG;
          double f[SEG + 1];
          ppm_line<SEG + 1>(QB(swk, ib, rj), 1, CX(scrx, ib, rj), 1, p1, p2, f);
          double num[SEG], den[SEG], v[SEG];
          bool ok = true;
#pragma unroll
          for (int u = 0; u < SEG; ++u) {
            const int i = ib + u;
            const double ar = *QB(sarea, i, rj);
            const double x0 = *CX(sxfx, i, rj), x1 = *CX(sxfx, i + 1, rj);
            num[u] = *QB(swk, i, rj) * ar + f[u] * x0 - f[u + 1] * x1;
            den[u] = ar + x0 - x1;
            v[u] = div_fast(num[u], den[u], ok);
          }
          if (!ok)
#pragma unroll
            for (int u = 0; u < SEG; ++u) v[u] = num[u] / den[u];
#pragma unroll
          for (int u = 0; u < SEG; ++u) sqj[(rj + 3) * L::JW + ib + u] = v[u];
          if (rj >= 0 && rj < TJ) {
#pragma unroll
            for (int u = 0; u < SEG; ++u) sfx2[rj * L::XW + ib + u] = f[u];
            if (ib + SEG == TI) sfx2[rj * L::XW + TI] = f[SEG];
          }
        } else if (item < NY + NX + NU) {
          // ub = 0.5*dt*(uc[0,-1,0] + uc) ; cub = select(ub > 0, ub*rdx[-1,0], ub*rdx) ; uu = xppm(u, cub)
          const int it = item - NY - NX;
          const int j = it % (TJ + 1), ib = (it / (TJ + 1)) * SEG;
          double ub[SEG + 1], cub[SEG + 1], f[SEG + 1];
#pragma unroll
          for (int u = 0; u < SEG + 1; ++u) {
            const int i = ib + u;
            ub[u] = 0.5 * dt * (*QB(UC, i, j - 1) + *QB(UC, i, j));
            cub[u] = ub[u] > 0.0 ? ub[u] * *QB(srdx, i - 1, j) : ub[u] * *QB(srdx, i, j);
          }
          ppm_line<SEG + 1>(QB(U, ib, j), 1, cub, 1, p1, p2, f);
          const int nf = (ib + SEG == TI) ? SEG + 1 : SEG;
#pragma unroll
          for (int u = 0; u < SEG + 1; ++u)
            if (u < nf) *CN(sked, ib + u, j) = ub[u] * f[u];
        } else if (item < NY + NX + NU + NV) {
          // vb = 0.5*dt*(vc[-1,0,0] + vc) ; cvb = select(vb > 0, vb*rdy[0,-1], vb*rdy) ; vv = yppm(v, cvb)
          const int it = item - NY - NX - NU;
          const int i = it % (TI + 1), jb = (it / (TI + 1)) * SEG;
          double vb[SEG + 1], cvb[SEG + 1], f[SEG + 1];
#pragma unroll
          for (int u = 0; u < SEG + 1; ++u) {
            const int j = jb + u;
            vb[u] = 0.5 * dt * (*QB(VC, i - 1, j) + *QB(VC, i, j));
            cvb[u] = vb[u] > 0.0 ? vb[u] * *QB(srdy, i, j - 1) : vb[u] * *QB(srdy, i, j);
          }
          ppm_line<SEG + 1>(QB(V, i, jb), L::QW, cvb, 1, p1, p2, f);
          const int nf = (jb + SEG == TJ) ? SEG + 1 : SEG;
#pragma unroll
          for (int u = 0; u < SEG + 1; ++u)
            if (u < nf) *CN(svv, i, jb + u) = vb[u] * f[u];
        } else {
          // divg / tens / smag / dmp / ddv at corner (i, j)
          const int it = item - NY - NX - NU - NV;
          const int i = it % (TI + 1), j = it / (TI + 1);
          const double rac = *QB(srac, i, j);
          const double ue = *QB(U, i, j) * *QB(sdyc, i, j), uw = *QB(U, i - 1, j) * *QB(sdyc, i - 1, j);
          const double vn = *QB(V, i, j) * *QB(sdxc, i, j), vs = *QB(V, i, j - 1) * *QB(sdxc, i, j - 1);
          const double divg = rac * (ue - uw + vn - vs);
          const double tens = rac * (ue - uw - vn + vs);
          const double smag = dt * sqrt(divg * divg + tens * tens);
          const double dmp = a.da_min * np_max(a.d2_bg, np_min(0.2, a.dddmp * smag));
          *CN(sddv, i, j) = dmp * divg;
        }
      }
    }
    __syncthreads();

    // ---- S2: phase B of fv_tp_2d(wk) (weights xfx / yfx); ked -------------
    if (tid < NX2) {
      const int rj = tid % TJ, ib = (tid / TJ) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(sqi + rj * L::QW + ib + 4, 1, CX(scrx, ib, rj), 1, p1, p2, f);
      const int nf = (ib + SEG == TI) ? SEG + 1 : SEG;
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        if (u < nf) {
          const int i = ib + u;
          sfx[rj * L::XW + i] = 0.5 * (f[u] + sfx2[rj * L::XW + i]) * *CX(sxfx, i, rj);
        }
      }
    } else if (yth) {
      ppm_line<SEG + 1>(sqj + (jb2 + 3) * L::JW + ci2, L::JW, CY(scry, ci2, jb2), L::YW, p1, p2, fy);
      // the weighted fluxes of this thread's own faces jb2 .. jb2+SEG-1 (face
      // jb2+SEG belongs to the next segment's thread), in place of fy2
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        const int j = jb2 + u;
        sfy2[j * TI + ci2] = 0.5 * (fy[u] + sfy2[j * TI + ci2]) * *CY(syfx, ci2, j);
      }
    } else {
      // ked = 0.5 * (ub*uu + vb*vv) over corners [0, TI+1) x [0, TJ+1)
      for (int e = tid - NX2 - NY2; e < (TI + 1) * (TJ + 1); e += blockDim.x - NX2 - NY2) {
        const int i = e % (TI + 1), j = e / (TI + 1);
        *CN(sked, i, j) = 0.5 * (*CN(sked, i, j) + *CN(svv, i, j));
      }
    }
    pend_k = k;
    // d2_v2 = div(dfx_v1, dfy_v1) * rarea, dfx_v1 = del6_v * (d2_v1 - d2_v1[-1,0])
    for (int e = tid; e < L::D2W * L::D2H; e += blockDim.x) {
      const int i = e % L::D2W - 1, j = e / L::D2W - 1;
      const int64_t m = min(max(i + j * sj, mlo), mhi);
      const double v0 = __ldg(gd6v + m), v1 = __ldg(gd6v + m + 1), u0 = __ldg(gd6u + m), u1 = __ldg(gd6u + m + sj);
      const double c = *D1(i, j);
      const double fx0 = v0 * (c - *D1(i - 1, j)), fx1 = v1 * (*D1(i + 1, j) - c);
      const double fy0 = u0 * (c - *D1(i, j - 1)), fy1 = u1 * (*D1(i, j + 1) - c);
      *D2(i, j) = (fx0 - fx1 + fy0 - fy1) * *QB(srarea, i, j);
    }
    __syncthreads();
  }
  write_pending();
}

}  // namespace

constexpr int MO_TI = 32, MO_TJ = 16;

int launch_dsw_momentum(const DswMoArgs& a0, cudaStream_t st) {
  using L = MoLayout<MO_TI, MO_TJ>;
  FV3B_TRY(ensure_smem((const void*)dsw_momentum_kernel<MO_TI, MO_TJ>, L::bytes, "d_sw momentum smem attribute"));
  DswMoArgs a = a0;
  const int tiles = cdiv(a.ni, MO_TI) * cdiv(a.nj, MO_TJ);
  a.kchunk = level_chunk(FV3B_TUNE_KCHUNK_DSW_MOMENTUM, tiles, a.nk, cps_of<MO_TJ>());
  dim3 grid(cdiv(a.ni, MO_TI), cdiv(a.nj, MO_TJ), cdiv(a.nk, a.kchunk));
  dsw_momentum_kernel<MO_TI, MO_TJ><<<grid, nt_of<MO_TJ>(), L::bytes, st>>>(a);
  return check_launch("d_sw momentum");
}

int dsw_momentum_maps(DswMoArgs& a, const Geo& g, const fv3b_field& u, const fv3b_field& v, const fv3b_field& uc,
                      const fv3b_field& vc, const fv3b_field* met12) {
  using L = MoLayout<MO_TI, MO_TJ>;
  FV3B_TRY(tensor_map(u.data, g.pitch, g.rows, g.levels, L::QW, L::QH + 1, &a.u));
  FV3B_TRY(tensor_map(v.data, g.pitch, g.rows, g.levels, L::QW, L::QH, &a.v));
  FV3B_TRY(tensor_map(uc.data, g.pitch, g.rows, g.levels, L::QW, L::QH, &a.uc));
  FV3B_TRY(tensor_map(vc.data, g.pitch, g.rows, g.levels, L::QW, L::QH, &a.vc));
  FV3B_TRY(tensor_map(met12[0].data, g.pitch, g.rows, 1, L::QW, L::QH + 1, &a.met[0]));
  for (int f = 1; f < 12; ++f) FV3B_TRY(tensor_map(met12[f].data, g.pitch, g.rows, 1, L::QW, L::QH, &a.met[f]));
  return FV3B_OK;
}

}  // namespace fv3b
