// K1 fv_tp_2d and K7 tracer_2d: FV3 2-D finite-volume transport
// (programs/fv_tp_2d.stn, programs/tracer_2d.stn; templates.fv_tp_2d).
//
// Statement chain per level (faces: fx on west faces, fy on south faces):
//   fy2 = yppm(q, cry)
//   qi  = (q*area + fy2*yfx - fy2[j+1]*yfx[j+1]) / (area + yfx - yfx[j+1])
//   fx2 = xppm(q, crx)
//   qj  = (q*area + fx2*xfx - fx2[i+1]*xfx[i+1]) / (area + xfx - xfx[i+1])
//   fx  = 0.5*(xppm(qi, crx) + fx2) * (xfx | mfx)
//   fy  = 0.5*(yppm(qj, cry) + fy2) * (yfx | mfy)
//   q'  = q + (fx - fx[i+1] + fy - fy[j+1]) * rarea                          fv_tp_2d
//   q'  = (q*dp1 + (...)*rarea) / (dp1 + (mfx-mfx[i+1]+mfy-mfy[j+1])*rarea)   tracer
//
// Kernel structure (one CTA = TI x TJ columns x a chunk of levels):
//  * every level's input tiles (q with a 3-cell halo, Courant numbers and
//    fluxes on the faces the chain touches) arrive by TMA into a
//    double-buffered shared-memory stage; the load of level k+1 (or the next
//    tracer) is issued before level k is computed, so HBM streams while the
//    FP64 pipes work;
//  * y-direction passes are column-per-thread, x-direction passes
//    row-segment-per-thread, each a register sliding window (ppm.cuh);
//  * temporaries are recomputed over the tile halo exactly where the
//    reference extends them (extents.py:128-164), so outputs are bitwise the
//    interpreter's.
// tracer_2d (tracer2_kernel) walks (level, group of TG tracers) steps so the
// shared Courant numbers / fluxes / dp1 are fetched once per level for all
// tracers and every barrier interval carries TG tracers' work.
#include "common.cuh"
#include "fastdiv.cuh"
#include "ppm.cuh"
#include "tma.cuh"

namespace fv3b {

constexpr int NQMAX = 16;
constexpr int SEG = 4;  // cells per sliding-window segment
// threads per CTA / CTAs per SM by tile height (>= phase-A items): 32x16
// tiles one CTA of 11 warps, 32x8 tiles two CTAs of 8 warps
template <int TJ> constexpr int nt_of() { return TJ >= 16 ? 352 : 256; }
// two CTAs per SM cap tp_kernel<32,16> at 93 registers, and ptxas spills
// 24 B (L1-resident); one CTA per SM removes the spill but measured slower
// (C2 fv_tp_2d 82 vs 74 us, 384x384x80 306 vs 265 us)
#ifndef FV3B_TP_CPS
#define FV3B_TP_CPS 2
#endif
template <int TJ> constexpr int cps_of() { return FV3B_TP_CPS; }

struct TpArgs {
  CUtensorMap q[NQMAX];
  CUtensorMap crx, xfx, cry, yfx, mfx, mfy, dp1, area;
  double* qout[NQMAX];
  const double* rarea;  // interior origin of rarea (2-D)
  int64_t sj, sk;       // 3-D strides (elements)
  int i0, j0;           // allocated column / row of the interior origin
  int nq, ni, nj, nk, kchunk;
  double p1, p2;
};

__host__ __device__ constexpr int align16(int n) { return (n + 15) / 16 * 16; }

template <int TI, int TJ, bool MASS>
struct TpLayout {
  // Row widths of tiles read by row-segment threads are = 2 (mod 4) doubles so
  // the threads of a warp (consecutive rows) hit distinct bank pairs.
  static constexpr int QW = TI + 10, QH = TJ + 6;  // q, area: i in [-4, TI+6), j in [-3, TJ+3)
  static constexpr int XW = TI + 2, XH = TJ + 6;   // crx, xfx: i in [0, TI+2), j in [-3, TJ+3)
  static constexpr int YW = TI + 8, YH = TJ + 1;   // cry, yfx: i in [-4, TI+4), j in [0, TJ+1)
  static constexpr int JW = TI + 2;                // qj row width
  static constexpr int n_q = align16(QW * QH);
  static constexpr int n_x = align16(XW * XH);
  static constexpr int n_y = align16(YW * YH);
  static constexpr int n_mx = align16(XW * TJ);    // mfx: i in [0, TI+2), j in [0, TJ)
  static constexpr int n_my = align16(TI * YH);    // mfy: i in [0, TI), j in [0, TJ+1)
  static constexpr int n_dp = align16(TI * TJ);    // dp1
  static constexpr int n_shared = 2 * n_x + 2 * n_y + (MASS ? n_mx + n_my + n_dp : 0);
  // intermediates
  static constexpr int n_qi = align16(QW * TJ);    // i in [-4, TI+4), j in [0, TJ)
  static constexpr int n_qj = align16(JW * QH);    // i in [0, TI), j in [-3, TJ+3)
  static constexpr int n_fx = align16(XW * TJ);    // faces i in [0, TI+1)
  static constexpr int n_fy = align16(TI * YH);    // faces j in [0, TJ+1)
  // offsets (doubles)
  static constexpr int o_q = 0;                      // 2 q stages
  static constexpr int o_sh = o_q + 2 * n_q;         // 2 shared stages
  static constexpr int o_area = o_sh + 2 * n_shared;
  static constexpr int o_qi = o_area + n_q;
  static constexpr int o_qj = o_qi + n_qi;
  static constexpr int o_fx2 = o_qj + n_qj;
  static constexpr int o_fy2 = o_fx2 + n_fx;
  static constexpr int o_fx = o_fy2 + n_fy;
  static constexpr int o_dp2 = o_fx + n_fx;
  static constexpr int total = o_dp2 + (MASS ? n_dp : 0);
  static constexpr size_t bytes = total * sizeof(double) + 64;  // + mbarriers
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static_assert(TJ % SEG == 0 && TI % SEG == 0 && QW % 4 == 2 && XW % 4 == 2 && JW % 4 == 2, "tile shape");
  // TMA transaction bytes
  static constexpr uint32_t tx_q = QW * QH * 8;
  static constexpr uint32_t tx_shared = (2 * XW * XH + 2 * YW * YH + (MASS ? XW * TJ + TI * YH + TI * TJ : 0)) * 8;
  static constexpr uint32_t tx_area = QW * QH * 8;
};

template <int TI, int TJ>
__global__ void __launch_bounds__(nt_of<TJ>(), (cps_of<TJ>())) tp_kernel(const __grid_constant__ TpArgs a) {
  constexpr bool MASS = false;  // tracer_2d: tracer2_kernel
  using L = TpLayout<TI, TJ, MASS>;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::total);  // [0],[1] step stages, [2] area
  const int tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ;
  const int k0 = blockIdx.z * a.kchunk;
  const int k1 = min(a.nk, k0 + a.kchunk);
  const int nsteps = (k1 - k0) * a.nq;
  const int xq = a.i0 + gi0 - 4, yq = a.j0 + gj0 - 3;  // box origins (allocated coords)
  const int xx = a.i0 + gi0, yy = a.j0 + gj0;
  const double p1 = a.p1, p2 = a.p2;

  auto issue = [&](int step) {  // single thread
    const int k = k0 + step / a.nq, t = step % a.nq;
    const int b = step & 1;
    double* sq = smem + L::o_q + b * L::n_q;
    uint32_t tx = L::tx_q;
    if (t == 0) tx += L::tx_shared;
    mbar_expect_tx(&bar[b], tx);
    tma_load3(sq, &a.q[t], xq, yq, k, &bar[b]);
    if (t == 0) {
      double* sh = smem + L::o_sh + ((k - k0) & 1) * L::n_shared;
      tma_load3(sh, &a.crx, xx, yq, k, &bar[b]);
      tma_load3(sh + L::n_x, &a.xfx, xx, yq, k, &bar[b]);
      tma_load3(sh + 2 * L::n_x, &a.cry, xq, yy, k, &bar[b]);
      tma_load3(sh + 2 * L::n_x + L::n_y, &a.yfx, xq, yy, k, &bar[b]);
    }
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && nsteps > 0) {
    mbar_expect_tx(&bar[2], L::tx_area);
    tma_load3(smem + L::o_area, &a.area, xq, yq, 0, &bar[2]);
    issue(0);
  }
  const double* sarea = smem + L::o_area;  // row width QW, origin (-4, -3)
  double* sqi = smem + L::o_qi;            // QW, origin (-4, 0)
  double* sqj = smem + L::o_qj;            // JW, origin (0, -3)
  double* sfx2 = smem + L::o_fx2;          // XW, origin (0, 0)
  double* sfy2 = smem + L::o_fy2;          // TI, origin (0, 0)
  double* sfx = smem + L::o_fx;            // XW, origin (0, 0)
  if (nsteps > 0) mbar_wait(&bar[2], 0);

  constexpr int NSEG = TI / SEG;
  static_assert((TI + 6) * (TJ / SEG) + (TJ + 6) * (TI / SEG) <= nt_of<TJ>(), "one phase-A item per thread");
  constexpr int NX2 = TJ * NSEG, NY2 = TI * (TJ / SEG);
  static_assert(NX2 + NY2 <= nt_of<TJ>(), "one item per thread in phase 2");
  // Phase-2 y threads own a fixed column segment for the whole CTA: they
  // keep rarea, and the previous step's fy / q / dp in registers and write
  // that step's result while the next step's phase 1 runs (2 barriers/level).
  const bool yth = tid >= NX2 && tid < NX2 + NY2;
  const int ci2 = yth ? (tid - NX2) % TI : 0;
  const int jb2 = yth ? ((tid - NX2) / TI) * SEG : 0;
  const int gi2 = gi0 + ci2;
  // phase-A worker slot: the y threads (which also write the pending cell
  // updates in phase A) take items only after every other thread has one
  const int wslot = tid < NX2 ? tid : (yth ? nt_of<TJ>() - NY2 + (tid - NX2) : tid - NY2);
  double ra[SEG];
#pragma unroll
  for (int u = 0; u < SEG; ++u) {
    const int gj = gj0 + jb2 + u;
    ra[u] = (yth && gi2 < a.ni && gj < a.nj) ? a.rarea[gi2 + (int64_t)gj * a.sj] : 0.0;
  }
  double fy[SEG + 1], qc[SEG];
  int pend_k = -1, pend_t = 0;  // step whose output is pending

  auto write_pending = [&]() {
    if (!yth || pend_k < 0) return;
    double* qo = a.qout[pend_t];
#pragma unroll
    for (int u = 0; u < SEG; ++u) {
      const int j = jb2 + u, gj = gj0 + j;
      if (gi2 < a.ni && gj < a.nj) {
        const int64_t off = gi2 + (int64_t)gj * a.sj + (int64_t)pend_k * a.sk;
        const double div = (sfx[j * L::XW + ci2] - sfx[j * L::XW + ci2 + 1] + fy[u] - fy[u + 1]) * ra[u];
        qo[off] = qc[u] + div;
      }
    }
  };

  int k = k0, t = 0;  // level / tracer of `step`, advanced incrementally
  for (int step = 0; step < nsteps; ++step, (++t == a.nq ? (t = 0, ++k) : 0)) {
    const int b = step & 1;
    if (tid == 0 && step + 1 < nsteps) {
      fence_async_smem();
      issue(step + 1);
    }
    mbar_wait(&bar[b], (step >> 1) & 1);
    const double* sq = smem + L::o_q + b * L::n_q;                             // QW, origin (-4, -3)
    const double* sh = smem + L::o_sh + ((k - k0) & 1) * L::n_shared;
    const double* scrx = sh;                                                   // XW, origin (0, -3)
    const double* sxfx = sh + L::n_x;                                          // XW, origin (0, -3)
    const double* scry = sh + 2 * L::n_x;                                      // YW, origin (-4, 0)
    const double* syfx = sh + 2 * L::n_x + L::n_y;                             // YW, origin (-4, 0)
    auto Q = [&](int i, int j) { return sq + (j + 3) * L::QW + (i + 4); };
    auto CX = [&](const double* p, int i, int j) { return p + (j + 3) * L::XW + i; };
    auto CY = [&](const double* p, int i, int j) { return p + j * L::YW + (i + 4); };

    // ---- phase A: previous step's output; yppm(q)/xppm(q) ---------------
    write_pending();
    // Y items: consecutive threads own consecutive columns; X items:
    // consecutive threads own consecutive rows (bank-conflict-free, see QW).
    {
      constexpr int NCY = TI + 6, NSY = TJ / SEG;  // columns i in [-3, TI+3)
      constexpr int NRX = TJ + 6, NSX = TI / SEG;  // rows j in [-3, TJ+3)
      constexpr int NY = NCY * NSY, NX = NRX * NSX;
      for (int item = wslot; item < NY + NX; item += blockDim.x) {
        if (item < NY) {
          const int ci = item % NCY - 3, jb = (item / NCY) * SEG;
          double f[SEG + 1];
          ppm_line<SEG + 1>(Q(ci, jb), L::QW, CY(scry, ci, jb), L::YW, p1, p2, f);
          // branch-free fast-path quotients, one exact fallback per item (fastdiv.cuh)
          double num[SEG], den[SEG], v[SEG];
          bool ok = true;
#pragma unroll
          for (int u = 0; u < SEG; ++u) {
            const int j = jb + u;
            const double ar = sarea[(j + 3) * L::QW + ci + 4];
            const double y0 = *CY(syfx, ci, j), y1 = *CY(syfx, ci, j + 1);
            num[u] = *Q(ci, j) * ar + f[u] * y0 - f[u + 1] * y1;
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
        } else {
          const int it = item - NY;
          const int rj = it % NRX - 3, ib = (it / NRX) * SEG;
          double f[SEG + 1];
          ppm_line<SEG + 1>(Q(ib, rj), 1, CX(scrx, ib, rj), 1, p1, p2, f);
          double num[SEG], den[SEG], v[SEG];
          bool ok = true;
#pragma unroll
          for (int u = 0; u < SEG; ++u) {
            const int i = ib + u;
            const double ar = sarea[(rj + 3) * L::QW + i + 4];
            const double x0 = *CX(sxfx, i, rj), x1 = *CX(sxfx, i + 1, rj);
            num[u] = *Q(i, rj) * ar + f[u] * x0 - f[u + 1] * x1;
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
        }
      }
    }
    __syncthreads();

    // ---- phase B: xppm(qi) -> fx (smem) ; yppm(qj) -> fy (registers) -----
    if (tid < NX2) {
      const int rj = tid % TJ, ib = (tid / TJ) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(sqi + rj * L::QW + ib + 4, 1, CX(scrx, ib, rj), 1, p1, p2, f);
      const int nf = (ib + SEG == TI) ? SEG + 1 : SEG;
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        if (u < nf) {
          const int i = ib + u;
          const double w = *CX(sxfx, i, rj);
          sfx[rj * L::XW + i] = 0.5 * (f[u] + sfx2[rj * L::XW + i]) * w;
        }
      }
    } else if (yth) {
      ppm_line<SEG + 1>(sqj + (jb2 + 3) * L::JW + ci2, L::JW, CY(scry, ci2, jb2), L::YW, p1, p2, fy);
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        const int j = jb2 + u;
        const double w = *CY(syfx, ci2, j);
        fy[u] = 0.5 * (fy[u] + sfy2[j * TI + ci2]) * w;
      }
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        qc[u] = *Q(ci2, jb2 + u);
      }
    }
    pend_k = k;
    pend_t = t;
    __syncthreads();
  }
  write_pending();
}

// ---------------------------------------------------------------------------
// tracer_2d, group schedule. The tracers of one level are processed TG at a
// time; per group two barrier intervals:
//   A: cell updates of the previous group (one cell per thread: dp2 from
//      registers, q' written straight to HBM) + phase A of all TG tracers
//      (one item per thread covers the group: the tracers share the inner
//      update's denominators, whose reciprocals are refined once);
//   B: phase B of all TG tracers (fluxes fx, fy to shared memory).
// Twice the work per barrier of tp_kernel, every thread busy in phase B, and
// the mass-flux divergence dp2 computed once per level in registers.
constexpr int TG = 2;

template <int TI, int TJ>
struct Tr2Layout {
  using B = TpLayout<TI, TJ, true>;  // tile shapes and TMA boxes as tp_kernel
  static constexpr int NQB = 3;      // q stages (group s in stage s % 3)
  // per-tracer intermediates: qi, qj, fx2, fy2, fx, fy
  static constexpr int s_qi = 0, s_qj = B::n_qi, s_fx2 = s_qj + B::n_qj, s_fy2 = s_fx2 + B::n_fx,
                       s_fx = s_fy2 + B::n_fy, s_fy = s_fx + B::n_fx, n_set = s_fy + B::n_fy;
  static constexpr int o_q = 0;
  static constexpr int o_sh = o_q + NQB * TG * B::n_q;  // 2 per-level stages
  static constexpr int o_area = o_sh + 2 * B::n_shared;
  static constexpr int o_set = o_area + B::n_q;
  static constexpr int total = o_set + TG * n_set;
  static constexpr size_t bytes = total * sizeof(double) + 64;
  static_assert(2 * bytes + 2048 <= 228 * 1024, "two CTAs per SM");
};

template <int TI, int TJ>
__global__ void __launch_bounds__(TI * TJ, 2) tracer2_kernel(const __grid_constant__ TpArgs a) {
  using B = TpLayout<TI, TJ, true>;
  using L = Tr2Layout<TI, TJ>;
  constexpr int NT = TI * TJ;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::total);  // [0..2] q stages, [3] area
  const int tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ;
  const int k0 = blockIdx.z * a.kchunk;
  const int k1 = min(a.nk, k0 + a.kchunk);
  const int ng = (a.nq + TG - 1) / TG;
  const int nsteps = (k1 - k0) * ng;
  const int xq = a.i0 + gi0 - 4, yq = a.j0 + gj0 - 3;
  const int xx = a.i0 + gi0, yy = a.j0 + gj0;
  const double p1 = a.p1, p2 = a.p2;
  auto qstage = [&](int s, int c) { return smem + L::o_q + ((s % L::NQB) * TG + c) * B::n_q; };
  auto shstage = [&](int lv) { return smem + L::o_sh + (lv & 1) * B::n_shared; };

  auto issue = [&](int s) {  // single thread
    const int lv = s / ng, g = s % ng, k = k0 + lv;
    const int t0 = g * TG, cnt = min(TG, a.nq - t0);
    uint64_t* mb = &bar[s % L::NQB];
    mbar_expect_tx(mb, cnt * B::tx_q + (g == 0 ? B::tx_shared : 0));
    for (int c = 0; c < cnt; ++c) tma_load3(qstage(s, c), &a.q[t0 + c], xq, yq, k, mb);
    if (g == 0) {
      double* sh = shstage(lv);
      tma_load3(sh, &a.crx, xx, yq, k, mb);
      tma_load3(sh + B::n_x, &a.xfx, xx, yq, k, mb);
      tma_load3(sh + 2 * B::n_x, &a.cry, xq, yy, k, mb);
      tma_load3(sh + 2 * B::n_x + B::n_y, &a.yfx, xq, yy, k, mb);
      double* m = sh + 2 * B::n_x + 2 * B::n_y;
      tma_load3(m, &a.mfx, xx, yy, k, mb);
      tma_load3(m + B::n_mx, &a.mfy, xx, yy, k, mb);
      tma_load3(m + B::n_mx + B::n_my, &a.dp1, xx, yy, k, mb);
    }
  };

  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && nsteps > 0) {
    mbar_expect_tx(&bar[3], B::tx_area);
    tma_load3(smem + L::o_area, &a.area, xq, yq, 0, &bar[3]);
    issue(0);
  }
  if (nsteps <= 0) return;
  const double* sarea = smem + L::o_area;  // QW, origin (-4, -3)
  mbar_wait(&bar[3], 0);

  // cell owned by this thread in the update pass
  const int li = tid % TI, lj = tid / TI;
  const bool live = gi0 + li < a.ni && gj0 + lj < a.nj;
  const int64_t coff = (gi0 + li) + (int64_t)(gj0 + lj) * a.sj;
  const double rr = live ? a.rarea[coff] : 0.0;
  double dp1c = 0.0, dp2c = 0.0;
  int dp_lv = -1;

  auto update = [&](int s) {  // q' of group s, one cell per thread
    const int lv = s / ng, g = s % ng;
    const int t0 = g * TG, cnt = min(TG, a.nq - t0);
    if (lv != dp_lv) {
      // dp2 = dp1 + (mfx - mfx[1,0,0] + mfy - mfy[0,1,0]) * rarea      (tracer_dp)
      const double* smfx = shstage(lv) + 2 * B::n_x + 2 * B::n_y;
      const double* smfy = smfx + B::n_mx;
      const double* sdp1 = smfy + B::n_my;
      dp1c = sdp1[lj * TI + li];
      dp2c = dp1c + (smfx[lj * B::XW + li] - smfx[lj * B::XW + li + 1] + smfy[lj * TI + li] -
                     smfy[(lj + 1) * TI + li]) * rr;
      dp_lv = lv;
    }
    if (!live) return;
    const int64_t off = coff + (int64_t)(k0 + lv) * a.sk;
#pragma unroll
    for (int c = 0; c < TG; ++c) {
      if (c < cnt) {
        const double* st = smem + L::o_set + c * L::n_set;
        const double* fx = st + L::s_fx;  // XW, origin (0, 0)
        const double* fy = st + L::s_fy;  // TI, origin (0, 0)
        const double div = (fx[lj * B::XW + li] - fx[lj * B::XW + li + 1] + fy[lj * TI + li] -
                            fy[(lj + 1) * TI + li]) * rr;
        const double qc = qstage(s, c)[(lj + 3) * B::QW + li + 4];
        a.qout[t0 + c][off] = (qc * dp1c + div) / dp2c;
      }
    }
  };

  constexpr int NCY = TI + 6, NSY = TJ / SEG;  // phase-A y columns i in [-3, TI+3)
  constexpr int NRX = TJ + 6, NSX = TI / SEG;  // phase-A x rows j in [-3, TJ+3)
  constexpr int NY = NCY * NSY, NX = NRX * NSX;
  constexpr int NX2 = TJ * NSX, NY2 = TI * NSY;  // phase-B x rows / y columns
  static_assert(TG * (NX2 + NY2) <= NT, "one phase-B item per thread");
  // with few tracer groups per level the next level's shared stage may only
  // be refilled once the previous group's cell updates are done (phase B)
  const bool early = ng >= 2;

  int lv = 0, g = 0;
  for (int s = 0; s < nsteps; ++s, (++g == ng ? (g = 0, ++lv) : 0)) {
    const int cnt = min(TG, a.nq - g * TG);
    if (early && tid == 0 && s + 1 < nsteps) {
      fence_async_smem();
      issue(s + 1);
    }
    mbar_wait(&bar[s % L::NQB], (s / L::NQB) & 1);
    const double* sh = shstage(lv);
    const double* scrx = sh;                             // XW, origin (0, -3)
    const double* sxfx = sh + B::n_x;                    // XW, origin (0, -3)
    const double* scry = sh + 2 * B::n_x;                // YW, origin (-4, 0)
    const double* syfx = sh + 2 * B::n_x + B::n_y;       // YW, origin (-4, 0)
    const double* smfx = sh + 2 * B::n_x + 2 * B::n_y;   // XW, origin (0, 0)
    const double* smfy = smfx + B::n_mx;                 // TI, origin (0, 0)
    auto CX = [&](const double* p, int i, int j) { return p + (j + 3) * B::XW + i; };
    auto CY = [&](const double* p, int i, int j) { return p + j * B::YW + (i + 4); };

    // ---- interval A: previous group's cell updates; phase A ------------------
    if (s > 0) update(s - 1);
    // one item for every tracer of the group: the inner-update denominators
    // are the tracers' common ones, so each cell's reciprocal is refined once
    // (fastdiv.cuh: bitwise a / b; an item outside the fast-path range is
    // redone with `/`)
    for (int item = tid; item < NY + NX; item += NT) {
      if (item < NY) {
        const int ci = item % NCY - 3, jb = (item / NCY) * SEG;
        double ar[SEG], y0[SEG], y1[SEG], den[SEG], rd[SEG];
#pragma unroll
        for (int u = 0; u < SEG; ++u) {
          const int j = jb + u;
          ar[u] = sarea[(j + 3) * B::QW + ci + 4];
          y0[u] = *CY(syfx, ci, j);
          y1[u] = *CY(syfx, ci, j + 1);
          den[u] = ar[u] + y0[u] - y1[u];
          rd[u] = rcp_fast(den[u]);
        }
#pragma unroll 1
        for (int c = 0; c < cnt; ++c) {
          const double* sq = qstage(s, c);
          double* st = smem + L::o_set + c * L::n_set;
          double f[SEG + 1];
          ppm_line<SEG + 1>(sq + (jb + 3) * B::QW + ci + 4, B::QW, CY(scry, ci, jb), B::YW, p1, p2, f);
          bool ok = true;
          double v[SEG];
#pragma unroll
          for (int u = 0; u < SEG; ++u)
            v[u] = div_fast_r(sq[(jb + u + 3) * B::QW + ci + 4] * ar[u] + f[u] * y0[u] - f[u + 1] * y1[u], den[u],
                              rd[u], ok);
          if (!ok)
#pragma unroll
            for (int u = 0; u < SEG; ++u)
              v[u] = (sq[(jb + u + 3) * B::QW + ci + 4] * ar[u] + f[u] * y0[u] - f[u + 1] * y1[u]) / den[u];
#pragma unroll
          for (int u = 0; u < SEG; ++u) st[L::s_qi + (jb + u) * B::QW + ci + 4] = v[u];
          if (ci >= 0 && ci < TI) {
#pragma unroll
            for (int u = 0; u < SEG; ++u) st[L::s_fy2 + (jb + u) * TI + ci] = f[u];
            if (jb + SEG == TJ) st[L::s_fy2 + TJ * TI + ci] = f[SEG];
          }
        }
      } else {
        const int it = item - NY;
        const int rj = it % NRX - 3, ib = (it / NRX) * SEG;
        double ar[SEG], x0[SEG], x1[SEG], den[SEG], rd[SEG];
#pragma unroll
        for (int u = 0; u < SEG; ++u) {
          const int i = ib + u;
          ar[u] = sarea[(rj + 3) * B::QW + i + 4];
          x0[u] = *CX(sxfx, i, rj);
          x1[u] = *CX(sxfx, i + 1, rj);
          den[u] = ar[u] + x0[u] - x1[u];
          rd[u] = rcp_fast(den[u]);
        }
#pragma unroll 1
        for (int c = 0; c < cnt; ++c) {
          const double* sq = qstage(s, c);
          double* st = smem + L::o_set + c * L::n_set;
          double f[SEG + 1];
          ppm_line<SEG + 1>(sq + (rj + 3) * B::QW + ib + 4, 1, CX(scrx, ib, rj), 1, p1, p2, f);
          bool ok = true;
          double v[SEG];
#pragma unroll
          for (int u = 0; u < SEG; ++u)
            v[u] = div_fast_r(sq[(rj + 3) * B::QW + ib + u + 4] * ar[u] + f[u] * x0[u] - f[u + 1] * x1[u], den[u],
                              rd[u], ok);
          if (!ok)
#pragma unroll
            for (int u = 0; u < SEG; ++u)
              v[u] = (sq[(rj + 3) * B::QW + ib + u + 4] * ar[u] + f[u] * x0[u] - f[u + 1] * x1[u]) / den[u];
#pragma unroll
          for (int u = 0; u < SEG; ++u) st[L::s_qj + (rj + 3) * B::JW + ib + u] = v[u];
          if (rj >= 0 && rj < TJ) {
#pragma unroll
            for (int u = 0; u < SEG; ++u) st[L::s_fx2 + rj * B::XW + ib + u] = f[u];
            if (ib + SEG == TI) st[L::s_fx2 + rj * B::XW + TI] = f[SEG];
          }
        }
      }
    }
    __syncthreads();

    // ---- interval B: xppm(qi) -> fx, yppm(qj) -> fy (mass-flux weighted) -----
    if (!early && tid == 0 && s + 1 < nsteps) {
      fence_async_smem();
      issue(s + 1);
    }
    if (tid < cnt * NX2) {
      const int c = tid / NX2, it = tid % NX2;
      double* st = smem + L::o_set + c * L::n_set;
      const int rj = it % TJ, ib = (it / TJ) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(st + L::s_qi + rj * B::QW + ib + 4, 1, CX(scrx, ib, rj), 1, p1, p2, f);
      const int nf = (ib + SEG == TI) ? SEG + 1 : SEG;
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        if (u < nf) {
          const int i = ib + u;
          st[L::s_fx + rj * B::XW + i] = 0.5 * (f[u] + st[L::s_fx2 + rj * B::XW + i]) * smfx[rj * B::XW + i];
        }
      }
    } else if (tid < cnt * NX2 + cnt * NY2) {
      const int y = tid - cnt * NX2;
      const int c = y / NY2, it = y % NY2;
      double* st = smem + L::o_set + c * L::n_set;
      const int ci = it % TI, jb = (it / TI) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(st + L::s_qj + (jb + 3) * B::JW + ci, B::JW, CY(scry, ci, jb), B::YW, p1, p2, f);
      const int nf = (jb + SEG == TJ) ? SEG + 1 : SEG;
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        if (u < nf) {
          const int j = jb + u;
          st[L::s_fy + j * TI + ci] = 0.5 * (f[u] + st[L::s_fy2 + j * TI + ci]) * smfy[j * TI + ci];
        }
      }
    }
    __syncthreads();
  }
  update(nsteps - 1);
}

template <int TI, int TJ>
static int launch_tracer2(const TpArgs& a0, cudaStream_t st) {
  using L = Tr2Layout<TI, TJ>;
  FV3B_TRY(ensure_smem((const void*)tracer2_kernel<TI, TJ>, L::bytes, "tracer_2d smem attribute"));
  TpArgs a = a0;
  a.kchunk = level_chunk(FV3B_TUNE_KCHUNK_TRACER, cdiv(a.ni, TI) * cdiv(a.nj, TJ), a.nk, 2);
  dim3 grid(cdiv(a.ni, TI), cdiv(a.nj, TJ), cdiv(a.nk, a.kchunk));
  tracer2_kernel<TI, TJ><<<grid, TI * TJ, L::bytes, st>>>(a);
  return check_launch("tracer_2d");
}

template <int TI, int TJ>
static int launch_tp(const TpArgs& a0, cudaStream_t st) {
  using L = TpLayout<TI, TJ, false>;
  FV3B_TRY(ensure_smem((const void*)tp_kernel<TI, TJ>, L::bytes, "tp smem attribute"));
  TpArgs a = a0;
  const int tiles = cdiv(a.ni, TI) * cdiv(a.nj, TJ);
  a.kchunk = level_chunk(FV3B_TUNE_KCHUNK_FV_TP_2D, tiles, a.nk, cps_of<TJ>());
  dim3 grid(cdiv(a.ni, TI), cdiv(a.nj, TJ), cdiv(a.nk, a.kchunk));
  tp_kernel<TI, TJ><<<grid, nt_of<TJ>(), L::bytes, st>>>(a);
  return check_launch("fv_tp_2d");
}

// Build the tensor maps for one call; boxes match TpLayout.
template <int TI, int TJ, bool MASS>
static int make_maps(TpArgs& a, const Geo& g, const fv3b_field* f3q, int nq, const fv3b_field& crx,
                     const fv3b_field& xfx, const fv3b_field& cry, const fv3b_field& yfx, const fv3b_field* mfx,
                     const fv3b_field* mfy, const fv3b_field* dp1, const fv3b_field& area) {
  using L = TpLayout<TI, TJ, MASS>;
  for (int t = 0; t < nq; ++t) FV3B_TRY(tensor_map(f3q[t].data, g.pitch, g.rows, g.levels, L::QW, L::QH, &a.q[t]));
  FV3B_TRY(tensor_map(crx.data, g.pitch, g.rows, g.levels, L::XW, L::XH, &a.crx));
  FV3B_TRY(tensor_map(xfx.data, g.pitch, g.rows, g.levels, L::XW, L::XH, &a.xfx));
  FV3B_TRY(tensor_map(cry.data, g.pitch, g.rows, g.levels, L::YW, L::YH, &a.cry));
  FV3B_TRY(tensor_map(yfx.data, g.pitch, g.rows, g.levels, L::YW, L::YH, &a.yfx));
  if (MASS) {
    FV3B_TRY(tensor_map(mfx->data, g.pitch, g.rows, g.levels, L::XW, TJ, &a.mfx));
    FV3B_TRY(tensor_map(mfy->data, g.pitch, g.rows, g.levels, TI, L::YH, &a.mfy));
    FV3B_TRY(tensor_map(dp1->data, g.pitch, g.rows, g.levels, TI, TJ, &a.dp1));
  }
  FV3B_TRY(tensor_map(area.data, g.pitch, g.rows, 1, L::QW, L::QH, &a.area));
  return FV3B_OK;
}

// Common argument validation: every 3-D field must have the same dense
// geometry (one TMA box geometry per launch).
static int same_geo(const fv3b_field* fs, int n, const Geo& g, const char* what) {
  for (int i = 0; i < n; ++i) {
    Geo h;
    FV3B_TRY(geo_of(fs[i], &h));
    const bool is2d = fs[i].rank == 2;
    if (h.pitch != g.pitch || h.rows != g.rows || (!is2d && h.levels != g.levels) || h.i0 != g.i0 || h.j0 != g.j0)
      return fail(FV3B_ELAYOUT, "%s: field %d geometry differs from field 0", what, i);
  }
  return FV3B_OK;
}

}  // namespace fv3b

using namespace fv3b;

static constexpr int TP_TI = 32, TP_TJ = 16;

extern "C" int fv3b_fv_tp_2d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                             void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 8 || ns != 2)
    return fail(FV3B_EINVAL, "fv3b_fv_tp_2d: expects 8 fields, 2 scalars (got %d, %d)", nf, ns);
  View q, crx, cry, xfx, yfx, area, rarea, qo;
  const Halo hq = {3, 3, 3, 3, 0, 0}, hx = {0, 1, 3, 3, 0, 0}, hy = {3, 3, 0, 1, 0, 0}, h0 = {0, 0, 0, 0, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, hq, "q", &q));
  FV3B_TRY(view_of(f[1], 3, *d, hx, "crx", &crx));
  FV3B_TRY(view_of(f[2], 3, *d, hy, "cry", &cry));
  FV3B_TRY(view_of(f[3], 3, *d, hx, "xfx", &xfx));
  FV3B_TRY(view_of(f[4], 3, *d, hy, "yfx", &yfx));
  FV3B_TRY(view_of(f[5], 2, *d, hq, "area", &area));
  FV3B_TRY(view_of(f[6], 2, *d, h0, "rarea", &rarea));
  FV3B_TRY(view_of(f[7], 3, *d, h0, "q_out", &qo));
  if (f[7].data == f[0].data) return fail(FV3B_EINVAL, "fv3b_fv_tp_2d: q_out must not alias q");
  Geo g;
  FV3B_TRY(geo_of(f[0], &g));
  FV3B_TRY(same_geo(f, 8, g, "fv3b_fv_tp_2d"));
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  TpArgs a;
  memset(&a, 0, sizeof a);
  FV3B_TRY((make_maps<TP_TI, TP_TJ, false>(a, g, &f[0], 1, f[1], f[3], f[2], f[4], nullptr, nullptr, nullptr, f[5])));
  a.qout[0] = qo.o;
  a.rarea = rarea.o;
  a.sj = q.sj;
  a.sk = q.sk;
  a.i0 = g.i0;
  a.j0 = g.j0;
  a.nq = 1;
  a.ni = d->ni; a.nj = d->nj; a.nk = d->nk;
  a.p1 = s[0];
  a.p2 = s[1];
  return launch_tp<TP_TI, TP_TJ>(a, (cudaStream_t)stream);
}

static constexpr int TR_TI = 32, TR_TJ = 8;

extern "C" int fv3b_tracer_2d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                              void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || ns != 2 || nf < 11 || (nf - 9) % 2 != 0 || (nf - 9) / 2 > NQMAX)
    return fail(FV3B_EINVAL, "fv3b_tracer_2d: expects 9 + 2*nq fields (nq <= %d), 2 scalars", NQMAX);
  const int nq = (nf - 9) / 2;
  View v;
  const Halo hq = {3, 3, 3, 3, 0, 0}, hx = {0, 1, 3, 3, 0, 0}, hy = {3, 3, 0, 1, 0, 0}, h0 = {0, 0, 0, 0, 0, 0};
  const Halo hmx = {0, 1, 0, 0, 0, 0}, hmy = {0, 0, 0, 1, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, hx, "cx", &v));
  FV3B_TRY(view_of(f[1], 3, *d, hy, "cy", &v));
  FV3B_TRY(view_of(f[2], 3, *d, hx, "xfx", &v));
  FV3B_TRY(view_of(f[3], 3, *d, hy, "yfx", &v));
  FV3B_TRY(view_of(f[4], 3, *d, hmx, "mfx", &v));
  FV3B_TRY(view_of(f[5], 3, *d, hmy, "mfy", &v));
  FV3B_TRY(view_of(f[6], 3, *d, h0, "dp1", &v));
  FV3B_TRY(view_of(f[7], 2, *d, hq, "area", &v));
  View rarea;
  FV3B_TRY(view_of(f[8], 2, *d, h0, "rarea", &rarea));
  TpArgs a;
  memset(&a, 0, sizeof a);
  for (int t = 0; t < nq; ++t) {
    View qi, qo;
    FV3B_TRY(view_of(f[9 + t], 3, *d, hq, "q", &qi));
    FV3B_TRY(view_of(f[9 + nq + t], 3, *d, h0, "q_out", &qo));
    if (f[9 + t].data == f[9 + nq + t].data) return fail(FV3B_EINVAL, "fv3b_tracer_2d: q%d_out aliases q%d", t, t);
    a.qout[t] = qo.o;
  }
  Geo g;
  FV3B_TRY(geo_of(f[0], &g));
  FV3B_TRY(same_geo(f, nf, g, "fv3b_tracer_2d"));
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  FV3B_TRY((make_maps<TR_TI, TR_TJ, true>(a, g, &f[9], nq, f[0], f[2], f[1], f[3], &f[4], &f[5], &f[6], f[7])));
  a.rarea = rarea.o;
  a.sj = (int64_t)g.pitch;
  a.sk = (int64_t)g.pitch * g.rows;
  a.i0 = g.i0;
  a.j0 = g.j0;
  a.nq = nq;
  a.ni = d->ni; a.nj = d->nj; a.nk = d->nk;
  a.p1 = s[0];
  a.p2 = s[1];
  return launch_tracer2<TR_TI, TR_TJ>(a, (cudaStream_t)stream);
}
