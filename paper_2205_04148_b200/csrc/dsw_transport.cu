// K3a d_sw transport group (programs/d_sw.stn: d_sw_courant, d_sw_mass,
// d_sw_heat, d_sw_vert and the delp / pt / w / accumulator statements of
// d_sw_update), as one level-marching, TMA-pipelined kernel.
//
// Structure: a CTA owns a TI x TJ column tile and walks a chunk of levels.
// Per level the inputs (delp, pt, w with a 3-cell halo and the C-grid winds
// uc / vc) arrive by TMA into a stage that is refilled for the next level as
// soon as this level's values are in registers; the 2-D metrics arrive once
// per CTA; the accumulators are read by the threads that update them.  Each
// level is three transport chains of the same fv_tp_2d statements:
//
//   delp  weights xfx / yfx   -> fxm, fym (mass fluxes, kept in smem), delpn
//   pt    weights fxm / fym   -> pt' = (pt*delp + div(gxp, gyp)*rarea) / delpn
//   w     weights fxm / fym   -> w'  = (w*delp + div(hxw, hyw)*rarea) / delpn
//
// exactly the tracer_2d update with dp1 = delp and (mfx, mfy) = (fxm, fym),
// so the statement chain, association and operand order are the .stn's and
// the results are bitwise the interpreter's.  Phase A evaluates yppm(q) ->
// fy2, qi and xppm(q) -> fx2, qj over the tile halo (register sliding
// windows, ppm.cuh); phase B the outer xppm(qi) / yppm(qj) and the weighted
// fluxes.  Each flux carries its del6 damping increment (templates.delnflux,
// FV3 deln_flux with nord = 2): the two Laplacian orders d2_1, d2_2 of every
// quantity are cell passes riding in the courant and phase-A intervals (each
// cell forms its four order-0/1 face fluxes itself: same operands, same
// bits as the stored temporaries), and the last order's face fluxes are
// formed by the phase-B items.  Five barriers per level: courant + d2_1 +
// mass weights | phase A + d2_2 | phase B of delp | phase B of pt, w | cell
// updates (d2_1 of the next level borrows the flux arrays they read).
#include "common.cuh"
#include "dsw.cuh"
#include "fastdiv.cuh"
#include "ppm.cuh"
#include "tma.cuh"

namespace fv3b {

namespace {

constexpr int SEG = 4;
// threads per CTA / CTAs per SM by tile height: 32x16 tiles run one CTA of 11
// warps per SM, 32x8 tiles two CTAs of 8 warps (<= 128 registers per thread)
template <int TI, int TJ> constexpr int nt_of() { return TI * TJ; }  // one thread per tile cell
template <int TI, int TJ> constexpr int cps_of() { return TI * TJ >= 512 ? 1 : 2; }

__host__ __device__ constexpr int a16(int n) { return (n + 15) / 16 * 16; }

// ---------------------------------------------------------------------------
// Four-barrier level schedule (the kernel launched): the three quantities'
// phase A run together, then phase B of delp (mass fluxes), then phase B of
// pt and w together, then every thread updates its own cell (delpn, delp',
// pt', w', accumulators) from registers it loaded while the stage was live.
// A single input stage: level k+1's TMA loads are issued as soon as level k's
// stage values are in registers (after phase B of delp), overlapping the
// rest of the level; the second CTA of the SM hides what remains.
// ---------------------------------------------------------------------------
template <int TI, int TJ>
struct Dt2Layout {
  static constexpr int QW = TI + 10, QH = TJ + 6;
  static constexpr int XW = TI + 2, XH = TJ + 6;
  static constexpr int YW = TI + 8, YH = TJ + 1;
  static constexpr int JW = TI + 2;
  static constexpr int D1W = TI + 4, D1H = TJ + 4;  // d2 order 1: [-2, TI+2) x [-2, TJ+2)
  static constexpr int D2W = TI + 2, D2H = TJ + 2;  // d2 order 2: [-1, TI+1) x [-1, TJ+1)
  static constexpr int n_q = a16(QW * QH);
  static constexpr int n_x = a16(XW * XH), n_y = a16(YW * YH);
  static constexpr int n_mx = a16(XW * TJ), n_my = a16(TI * YH);
  static constexpr int n_qi = a16(QW * TJ), n_qj = a16(JW * QH);
  static constexpr int n_d1 = a16(D1W * D1H), n_d2 = a16(D2W * D2H);
  static constexpr int n_set = n_qi + n_qj + n_mx + n_my;  // qi, qj, fx2, fy2 of one quantity
  static constexpr int n_fl = n_mx + n_my;                 // x / y fluxes of one quantity
  static constexpr int o_stage = 0;                        // delp, pt, w, uc, vc
  static constexpr int o_met = 5 * n_q;                    // area, rarea, del6_u, del6_v
  static constexpr int o_crx = o_met + 4 * n_q;
  static constexpr int o_xfx = o_crx + n_x;
  static constexpr int o_cry = o_xfx + n_x;
  static constexpr int o_yfx = o_cry + n_y;
  static constexpr int o_set = o_yfx + n_y;
  static constexpr int o_fl = o_set + 3 * n_set;           // (d2_1 of the three quantities until phase B)
  static constexpr int o_d2 = o_fl + 3 * n_fl;             // d2_2 of delp, pt, w
  static constexpr int o_mw = o_d2 + 3 * n_d2;             // damp4h * (delp[-1] + delp): x faces, y faces
  static constexpr int total = o_mw + n_mx + n_my;
  static constexpr size_t bytes = total * sizeof(double) + 64;
  static_assert(3 * n_d1 <= 3 * n_fl, "d2_1 fits the flux arrays it borrows");
  // two CTAs per SM: 228 KB per SM, 1 KB reserved per CTA
  static_assert(cps_of<TI, TJ>() * (bytes + 1024) <= 228 * 1024, "shared memory budget");
  static_assert(TJ % SEG == 0 && TI % SEG == 0 && QW % 4 == 2 && XW % 4 == 2 && JW % 4 == 2, "tile shape");
  static constexpr uint32_t tx_stage = 5 * QW * QH * 8;
  static constexpr uint32_t tx_met = 4 * QW * QH * 8;
};

template <int TI, int TJ>
__global__ void __launch_bounds__(nt_of<TI, TJ>(), cps_of<TI, TJ>()) dsw_transport2_kernel(
    const __grid_constant__ DswTpArgs a) {
  using L = Dt2Layout<TI, TJ>;
  constexpr int NT = nt_of<TI, TJ>();
  static_assert(NT == TI * TJ, "one thread per tile cell for the update phase");
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::total);  // [0] stage, [1] metrics
  const int tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ;
  const int k0 = blockIdx.z * a.kchunk;
  const int k1 = min(a.nk, k0 + a.kchunk);
  const int xq = a.i0 + gi0 - 4, yq = a.j0 + gj0 - 3;
  const double p1 = a.p1, p2 = a.p2, dt = a.dt;

  auto issue = [&](int k) {
    mbar_expect_tx(&bar[0], L::tx_stage);
#pragma unroll
    for (int f = 0; f < 5; ++f) tma_load3(smem + L::o_stage + f * L::n_q, &a.qbox[f], xq, yq, k, &bar[0]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && k1 > k0) {
    mbar_expect_tx(&bar[1], L::tx_met);
#pragma unroll
    for (int f = 0; f < 4; ++f) tma_load3(smem + L::o_met + f * L::n_q, &a.met[f], xq, yq, 0, &bar[1]);
    issue(k0);
  }
  const double* sdp = smem + L::o_stage;
  const double* suc = sdp + 3 * L::n_q;
  const double* svc = sdp + 4 * L::n_q;
  const double* sarea = smem + L::o_met;
  const double* srarea = sarea + L::n_q;
  const double* sd6u = srarea + L::n_q;
  const double* sd6v = sd6u + L::n_q;
  // courant-only metrics straight from L1 / L2 (tile-local (i, j); 2-D, J stride sj)
  const int64_t moff = gi0 + (int64_t)gj0 * a.sj;
  const double* gdx = a.dx + moff;
  const double* gdy = a.dy + moff;
  const double* grdxa = a.rdxa + moff;
  const double* grdya = a.rdya + moff;
  // a ragged edge tile's box reaches past the allocated halo: its metric
  // loads are clamped into the allocation (those cells lie outside the
  // domain plus the 3-cell halo every owned cell reads, so no owned result
  // sees the clamped values)
  const int64_t mlo = a.mlo - moff, mhi = a.mhi - moff;
  double* scrx = smem + L::o_crx;  // XW, origin (0, -3)
  double* sxfx = smem + L::o_xfx;
  double* scry = smem + L::o_cry;  // YW, origin (-4, 0)
  double* syfx = smem + L::o_yfx;
  auto QB = [&](auto* p, int i, int j) { return p + (j + 3) * L::QW + (i + 4); };
  auto CX = [&](auto* p, int i, int j) { return p + (j + 3) * L::XW + i; };
  auto CY = [&](auto* p, int i, int j) { return p + j * L::YW + (i + 4); };
  auto SQI = [&](int q) { return smem + L::o_set + q * L::n_set; };                // QW, origin (-4, 0)
  auto SQJ = [&](int q) { return SQI(q) + L::n_qi; };                              // JW, origin (0, -3)
  auto SFX2 = [&](int q) { return SQJ(q) + L::n_qj; };                             // XW, origin (0, 0)
  auto SFY2 = [&](int q) { return SFX2(q) + L::n_mx; };                            // TI, origin (0, 0)
  auto FLX = [&](int q) { return smem + L::o_fl + q * L::n_fl; };                  // XW, origin (0, 0)
  auto FLY = [&](int q) { return FLX(q) + L::n_mx; };                              // TI, origin (0, 0)
  auto D1 = [&](int q, int i, int j) { return smem + L::o_fl + q * L::n_d1 + (j + 2) * L::D1W + (i + 2); };
  auto D2 = [&](int q, int i, int j) { return smem + L::o_d2 + q * L::n_d2 + (j + 1) * L::D2W + (i + 1); };
  double* smwx = smem + L::o_mw;  // XW, origin (0, 0)
  double* smwy = smwx + L::n_mx;  // TI, origin (0, 0)
  const double damp4 = a.damp4, damp4h = a.damp4h;
  if (k1 > k0) mbar_wait(&bar[1], 0);

  // this thread's update cell
  const int ci = tid % TI, cj = tid / TI, gi = gi0 + ci, gj = gj0 + cj;
  const bool own = gi < a.ni && gj < a.nj;
  const int64_t sj = a.sj, sk = a.sk;
  const int64_t coff = gi + gj * sj;
  const double ra = *QB(srarea, ci, cj);

  constexpr int NSEG = TI / SEG;
  constexpr int NCY = TI + 6, NSY = TJ / SEG;  // phase-A y items: columns [-3, TI+3)
  constexpr int NRX = TJ + 6, NSX = TI / SEG;  // phase-A x items: rows [-3, TJ+3)
  constexpr int NY = NCY * NSY, NA = NY + NRX * NSX;
  constexpr int NX2 = TJ * NSEG, NB = NX2 + TI * (TJ / SEG);
  static_assert(NA < NT, "one phase-A item per thread, spare threads for del6 order 2");

  // phase A of quantity q, item `it` (0 <= it < NA)
  auto phase_a = [&](int q, int it) {
    const double* Q = sdp + q * L::n_q;
    double* sqi = SQI(q);
    double* sqj = SQJ(q);
    double* sfx2 = SFX2(q);
    double* sfy2 = SFY2(q);
    if (it < NY) {
      const int c = it % NCY - 3, jb = (it / NCY) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(QB(Q, c, jb), L::QW, CY(scry, c, jb), L::YW, p1, p2, f);
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        const int j = jb + u;
        const double ar = *QB(sarea, c, j);
        const double y0 = *CY(syfx, c, j), y1 = *CY(syfx, c, j + 1);
        sqi[j * L::QW + c + 4] = (*QB(Q, c, j) * ar + f[u] * y0 - f[u + 1] * y1) / (ar + y0 - y1);
      }
      if (c >= 0 && c < TI) {
#pragma unroll
        for (int u = 0; u < SEG; ++u) sfy2[(jb + u) * TI + c] = f[u];
        if (jb + SEG == TJ) sfy2[TJ * TI + c] = f[SEG];
      }
    } else {
      const int r = it - NY;
      const int rj = r % NRX - 3, ib = (r / NRX) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(QB(Q, ib, rj), 1, CX(scrx, ib, rj), 1, p1, p2, f);
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        const int i = ib + u;
        const double ar = *QB(sarea, i, rj);
        const double x0 = *CX(sxfx, i, rj), x1 = *CX(sxfx, i + 1, rj);
        sqj[(rj + 3) * L::JW + i] = (*QB(Q, i, rj) * ar + f[u] * x0 - f[u + 1] * x1) / (ar + x0 - x1);
      }
      if (rj >= 0 && rj < TJ) {
#pragma unroll
        for (int u = 0; u < SEG; ++u) sfx2[rj * L::XW + ib + u] = f[u];
        if (ib + SEG == TI) sfx2[rj * L::XW + TI] = f[SEG];
      }
    }
  };
  // phase A of all three quantities for item `it`: the inner-update
  // denominators (area + yfx - yfx[j+1], area + xfx - xfx[i+1]) are the
  // same for delp, pt and w, so each cell's reciprocal is refined once and
  // the three quotients take nvcc's fast-path residual step (fastdiv.cuh:
  // bitwise a / b); an item whose range test fails is redone with `/`.
  auto phase_a3 = [&](int it) {
    if (it < NY) {
      const int c = it % NCY - 3, jb = (it / NCY) * SEG;
      double den[SEG], rd[SEG], ar[SEG], y0[SEG], y1[SEG];
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        const int j = jb + u;
        ar[u] = *QB(sarea, c, j);
        y0[u] = *CY(syfx, c, j);
        y1[u] = *CY(syfx, c, j + 1);
        den[u] = ar[u] + y0[u] - y1[u];
        rd[u] = rcp_fast(den[u]);
      }
      bool ok = true;
#pragma unroll 1
      for (int q = 0; q < 3; ++q) {
        const double* Q = sdp + q * L::n_q;
        double* sqi = SQI(q);
        double* sfy2 = SFY2(q);
        double f[SEG + 1], qc[SEG];
        ppm_line<SEG + 1, SEG>(QB(Q, c, jb), L::QW, CY(scry, c, jb), L::YW, p1, p2, f, qc);
#pragma unroll
        for (int u = 0; u < SEG; ++u) {
          const int j = jb + u;
          const double num = qc[u] * ar[u] + f[u] * y0[u] - f[u + 1] * y1[u];
          double v = div_fast_r(num, den[u], rd[u], ok);
          sqi[j * L::QW + c + 4] = v;
        }
        if (c >= 0 && c < TI) {
#pragma unroll
          for (int u = 0; u < SEG; ++u) sfy2[(jb + u) * TI + c] = f[u];
          if (jb + SEG == TJ) sfy2[TJ * TI + c] = f[SEG];
        }
      }
      if (!ok)
        for (int q = 0; q < 3; ++q) phase_a(q, it);
    } else {
      const int r = it - NY;
      const int rj = r % NRX - 3, ib = (r / NRX) * SEG;
      double den[SEG], rd[SEG], ar[SEG], x0[SEG], x1[SEG];
#pragma unroll
      for (int u = 0; u < SEG; ++u) {
        const int i = ib + u;
        ar[u] = *QB(sarea, i, rj);
        x0[u] = *CX(sxfx, i, rj);
        x1[u] = *CX(sxfx, i + 1, rj);
        den[u] = ar[u] + x0[u] - x1[u];
        rd[u] = rcp_fast(den[u]);
      }
      bool ok = true;
#pragma unroll 1
      for (int q = 0; q < 3; ++q) {
        const double* Q = sdp + q * L::n_q;
        double* sqj = SQJ(q);
        double* sfx2 = SFX2(q);
        double f[SEG + 1], qc[SEG];
        ppm_line<SEG + 1, SEG>(QB(Q, ib, rj), 1, CX(scrx, ib, rj), 1, p1, p2, f, qc);
#pragma unroll
        for (int u = 0; u < SEG; ++u) {
          const int i = ib + u;
          const double num = qc[u] * ar[u] + f[u] * x0[u] - f[u + 1] * x1[u];
          sqj[(rj + 3) * L::JW + i] = div_fast_r(num, den[u], rd[u], ok);
        }
        if (rj >= 0 && rj < TJ) {
#pragma unroll
          for (int u = 0; u < SEG; ++u) sfx2[rj * L::XW + ib + u] = f[u];
          if (ib + SEG == TI) sfx2[rj * L::XW + TI] = f[SEG];
        }
      }
      if (!ok)
        for (int q = 0; q < 3; ++q) phase_a(q, it);
    }
  };
  // del6 order 1 of delp, pt, w (templates.delnflux): d2_0 = damp4 * delp
  // (delp) or q itself (pt, w: mass-weighted chains), dfx_0 = del6_v *
  // (d2_0[-1,0] - d2_0), d2_1 = div(dfx_0, dfy_0) * rarea.  An item is a
  // vertical run of DR cells of one column for all three quantities: the
  // metrics are loaded once for the three, and each y-face flux once for the
  // two cells that share it (the same operands, so the same bits as each
  // cell forming its four face fluxes).  Lanes run along i (conflict-free).
  constexpr int DR = 2;
  static_assert(L::D1H % DR == 0 && L::D2H % DR == 0, "del6 runs tile the rows");
  auto deln1 = [&](int e) {
    const int i = e % L::D1W - 2, j0 = (e / L::D1W) * DR - 2;
    double v0[DR], v1[DR], rr[DR], uf[DR + 1];
#pragma unroll
    for (int r = 0; r < DR; ++r) {
      v0[r] = *QB(sd6v, i, j0 + r);
      v1[r] = *QB(sd6v, i + 1, j0 + r);
      rr[r] = *QB(srarea, i, j0 + r);
    }
#pragma unroll
    for (int f = 0; f <= DR; ++f) uf[f] = *QB(sd6u, i, j0 + f);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double* Q = sdp + q * L::n_q;
      double col[DR + 2], wq[DR], eq[DR];
#pragma unroll
      for (int d = 0; d < DR + 2; ++d) col[d] = *QB(Q, i, j0 - 1 + d);
#pragma unroll
      for (int r = 0; r < DR; ++r) {
        wq[r] = *QB(Q, i - 1, j0 + r);
        eq[r] = *QB(Q, i + 1, j0 + r);
      }
      if (q == 0) {
#pragma unroll
        for (int d = 0; d < DR + 2; ++d) col[d] = damp4 * col[d];
#pragma unroll
        for (int r = 0; r < DR; ++r) {
          wq[r] = damp4 * wq[r];
          eq[r] = damp4 * eq[r];
        }
      }
      double fy[DR + 1];  // face j0 + f: del6_u * (d2[j-1] - d2[j])
#pragma unroll
      for (int f = 0; f <= DR; ++f) fy[f] = uf[f] * (col[f] - col[f + 1]);
#pragma unroll
      for (int r = 0; r < DR; ++r) {
        const double c = col[r + 1];
        const double fx0 = v0[r] * (wq[r] - c), fx1 = v1[r] * (c - eq[r]);
        *D1(q, i, j0 + r) = (fx0 - fx1 + fy[r] - fy[r + 1]) * rr[r];
      }
    }
  };
  // del6 order 2: dfx_1 = del6_v * (d2_1 - d2_1[-1,0]), d2_2 = div(dfx_1, dfy_1) * rarea
  // (vertical runs like order 1)
  auto deln2 = [&](int e) {
    const int i = e % L::D2W - 1, j0 = (e / L::D2W) * DR - 1;
    double v0[DR], v1[DR], rr[DR], uf[DR + 1];
#pragma unroll
    for (int r = 0; r < DR; ++r) {
      v0[r] = *QB(sd6v, i, j0 + r);
      v1[r] = *QB(sd6v, i + 1, j0 + r);
      rr[r] = *QB(srarea, i, j0 + r);
    }
#pragma unroll
    for (int f = 0; f <= DR; ++f) uf[f] = *QB(sd6u, i, j0 + f);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double col[DR + 2], wq[DR], eq[DR];
#pragma unroll
      for (int d = 0; d < DR + 2; ++d) col[d] = *D1(q, i, j0 - 1 + d);
#pragma unroll
      for (int r = 0; r < DR; ++r) {
        wq[r] = *D1(q, i - 1, j0 + r);
        eq[r] = *D1(q, i + 1, j0 + r);
      }
      double fy[DR + 1];  // face j0 + f: del6_u * (d2_1[j] - d2_1[j-1])
#pragma unroll
      for (int f = 0; f <= DR; ++f) fy[f] = uf[f] * (col[f + 1] - col[f]);
#pragma unroll
      for (int r = 0; r < DR; ++r) {
        const double c = col[r + 1];
        const double fx0 = v0[r] * (c - wq[r]), fx1 = v1[r] * (eq[r] - c);
        *D2(q, i, j0 + r) = (fx0 - fx1 + fy[r] - fy[r + 1]) * rr[r];
      }
    }
  };
  // phase B of quantity q, item `it` (0 <= it < NB): weighted fluxes into FLX/FLY(q).
  // Every operand is loaded before the first store (the stores could alias
  // them as far as the compiler knows, which would force reloads).
  auto phase_b = [&](int q, int it) {
    if (it < NX2) {
      const int rj = it % TJ, ib = (it / TJ) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(SQI(q) + rj * L::QW + ib + 4, 1, CX(scrx, ib, rj), 1, p1, p2, f);
      const int nf = (ib + SEG == TI) ? SEG + 1 : SEG;
      const double* fx2 = SFX2(q);
      double* out = FLX(q);
      double wv[SEG + 1], f2[SEG + 1], d6[SEG + 1], mw[SEG + 1], dv[SEG + 2];
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        const int i = ib + u;  // <= TI: inside every face array
        wv[u] = q == 0 ? *CX(sxfx, i, rj) : FLX(0)[rj * L::XW + i];
        f2[u] = fx2[rj * L::XW + i];
        d6[u] = *QB(sd6v, i, rj);
        mw[u] = q == 0 ? 0.0 : smwx[rj * L::XW + i];
      }
#pragma unroll
      for (int u = 0; u < SEG + 2; ++u) dv[u] = *D2(q, ib - 1 + u, rj);
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        if (u < nf) {
          // + dfx_2 = del6_v * (d2_2 - d2_2[-1,0]) (x damp4h * (delp[-1,0] + delp) for pt, w)
          const double dd = d6[u] * (dv[u + 1] - dv[u]);
          const double dinc = q == 0 ? dd : mw[u] * dd;
          out[rj * L::XW + ib + u] = 0.5 * (f[u] + f2[u]) * wv[u] + dinc;
        }
      }
    } else {
      const int r = it - NX2;
      const int c = r % TI, jb = (r / TI) * SEG;
      double f[SEG + 1];
      ppm_line<SEG + 1>(SQJ(q) + (jb + 3) * L::JW + c, L::JW, CY(scry, c, jb), L::YW, p1, p2, f);
      const int nf = (jb + SEG == TJ) ? SEG + 1 : SEG;
      const double* fy2 = SFY2(q);
      double* out = FLY(q);
      double wv[SEG + 1], f2[SEG + 1], d6[SEG + 1], mw[SEG + 1], dv[SEG + 2];
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        const int j = jb + u;  // <= TJ: inside every face array
        wv[u] = q == 0 ? *CY(syfx, c, j) : FLY(0)[j * TI + c];
        f2[u] = fy2[j * TI + c];
        d6[u] = *QB(sd6u, c, j);
        mw[u] = q == 0 ? 0.0 : smwy[j * TI + c];
      }
#pragma unroll
      for (int u = 0; u < SEG + 2; ++u) dv[u] = *D2(q, c, jb - 1 + u);
#pragma unroll
      for (int u = 0; u < SEG + 1; ++u) {
        if (u < nf) {
          const double dd = d6[u] * (dv[u + 1] - dv[u]);
          const double dinc = q == 0 ? dd : mw[u] * dd;
          out[(jb + u) * TI + c] = 0.5 * (f[u] + f2[u]) * wv[u] + dinc;
        }
      }
    }
  };

  for (int k = k0; k < k1; ++k) {
    // accumulator inputs of this thread's cell (consumed in S4)
    double acc[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) acc[f] = (own && !a.acc_reset) ? ld_stream(a.acci[f] + (own ? coff : 0) + (int64_t)k * sk) : 0.0;
    // ---- S0: courant -------------------------------------------------------
    // (this thread's courant metrics are loaded before the stage wait, so
    // their L1 / L2 latency hides behind it; nothing else is live here)
    constexpr int NCX = (L::XW * L::XH + NT - 1) / NT, NCYI = (L::YW * L::YH + NT - 1) / NT;
    double mxd[NCX], mxl[NCX], mxr[NCX], myd[NCYI], myl[NCYI], myr[NCYI];
#pragma unroll
    for (int u = 0; u < NCX; ++u) {  // (spare items load the last item's metrics: always in bounds)
      const int e = min(tid + u * NT, L::XW * L::XH - 1);
      const int i = e % L::XW, j = e / L::XW - 3;
      const int64_t m = min(max(i + j * sj, mlo + 1), mhi);
      mxd[u] = ld_keep(gdy + m);
      mxl[u] = ld_keep(grdxa + m - 1);
      mxr[u] = ld_keep(grdxa + m);
    }
#pragma unroll
    for (int u = 0; u < NCYI; ++u) {
      const int e = min(tid + u * NT, L::YW * L::YH - 1);
      const int i = e % L::YW - 4, j = e / L::YW;
      const int64_t m = min(max(i + j * sj, mlo + sj), mhi);
      myd[u] = ld_keep(gdx + m);
      myl[u] = ld_keep(grdya + m - sj);
      myr[u] = ld_keep(grdya + m);
    }
    mbar_wait(&bar[0], (k - k0) & 1);
#pragma unroll
    for (int u = 0; u < NCX; ++u) {
      const int e = tid + u * NT;
      if (e < L::XW * L::XH) {
        const int i = e % L::XW, j = e / L::XW - 3;
        const double uc = *QB(suc, i, j);
        *CX(sxfx, i, j) = dt * uc * mxd[u];
        *CX(scrx, i, j) = uc > 0.0 ? dt * uc * mxl[u] : dt * uc * mxr[u];
      }
    }
#pragma unroll
    for (int u = 0; u < NCYI; ++u) {
      const int e = tid + u * NT;
      if (e < L::YW * L::YH) {
        const int i = e % L::YW - 4, j = e / L::YW;
        const double vc = *QB(svc, i, j);
        *CY(syfx, i, j) = dt * vc * myd[u];
        *CY(scry, i, j) = vc > 0.0 ? dt * vc * myl[u] : dt * vc * myr[u];
      }
    }
    for (int e = tid; e < L::D1W * (L::D1H / DR); e += NT) deln1(e);
    // mass weights damp4h * (delp[-1] + delp) of the x / y faces (stage delp
    // only; read by phase B of pt and w), dealt from the last thread down so
    // the threads without a del6 order-1 item take the extra ones (measured
    // 0.2% per step faster here than beside phase A)
    for (int e = NT - 1 - tid; e < (TI + 1) * TJ + TI * (TJ + 1); e += NT) {
      if (e < (TI + 1) * TJ) {
        const int i = e % (TI + 1), j = e / (TI + 1);
        smwx[j * L::XW + i] = damp4h * (*QB(sdp, i - 1, j) + *QB(sdp, i, j));
      } else {
        const int i = (e - (TI + 1) * TJ) % TI, j = (e - (TI + 1) * TJ) / TI;
        smwy[j * TI + i] = damp4h * (*QB(sdp, i, j - 1) + *QB(sdp, i, j));
      }
    }
    __syncthreads();
    // ---- S1: phase A of delp, pt, w; del6 order 2 ------------------------------
    // (the phase-A items are the heavy ones: one per thread of the first NA;
    // the remaining threads take del6 order 2)
    if (tid < NA) {
      phase_a3(tid);
    } else {
      const int t = tid - NA;
      constexpr int NR = NT - NA;
      for (int e = t; e < L::D2W * (L::D2H / DR); e += NR) deln2(e);
    }
    __syncthreads();
    // ---- S2: phase B of delp (mass fluxes); stage values of the update cell ---
    if (tid < NB) phase_b(0, tid);
    const double* spt = sdp + L::n_q;
    const double* sww = sdp + 2 * L::n_q;
    const double dp = *QB(sdp, ci, cj), ptc = *QB(spt, ci, cj), wc = *QB(sww, ci, cj);
    const double crx = *CX(scrx, ci, cj), cry = *CY(scry, ci, cj);
    const double xfx = *CX(sxfx, ci, cj), yfx = *CY(syfx, ci, cj);
    __syncthreads();
    // the stage is free: fetch level k+1 while this level finishes
    if (tid == 0 && k + 1 < k1) {
      fence_async_smem();
      issue(k + 1);
    }
    // ---- S3: phase B of pt and w ----------------------------------------------
    for (int e = tid; e < 2 * NB; e += NT) phase_b(1 + e / NB, e % NB);
    __syncthreads();
    // ---- S4: cell updates (d_sw_update) ----------------------------------------
    {
      const double* fxm = FLX(0);
      const double* fym = FLY(0);
      const double fxm0 = fxm[cj * L::XW + ci], fxm1 = fxm[cj * L::XW + ci + 1];
      const double fym0 = fym[cj * TI + ci], fym1 = fym[(cj + 1) * TI + ci];
      // delpn = delp + (fxm - fxm[1,0,0] + fym - fym[0,1,0]) * rarea
      const double dn = dp + (fxm0 - fxm1 + fym0 - fym1) * ra;
      const double* gxp = FLX(1);
      const double* gyp = FLY(1);
      const double* hxw = FLX(2);
      const double* hyw = FLY(2);
      const double divp = (gxp[cj * L::XW + ci] - gxp[cj * L::XW + ci + 1] + gyp[cj * TI + ci] -
                           gyp[(cj + 1) * TI + ci]) * ra;
      const double divw = (hxw[cj * L::XW + ci] - hxw[cj * L::XW + ci + 1] + hyw[cj * TI + ci] -
                           hyw[(cj + 1) * TI + ci]) * ra;
      if (own) {
        const int64_t off = coff + (int64_t)k * sk;
        a.delpo[off] = dn;
        if (a.dp1o) a.dp1o[off] = dp;
        // pt' and w' share the divisor delpn: one refined reciprocal (fastdiv.cuh)
        bool ok = true;
        const double rdn = rcp_fast(dn);
        double ptn = div_fast_r(ptc * dp + divp, dn, rdn, ok);
        double wq = div_fast_r(wc * dp + divw, dn, rdn, ok);
        if (!ok) {
          ptn = (ptc * dp + divp) / dn;
          wq = (wc * dp + divw) / dn;
        }
        a.pto[off] = ptn;
        a.wo[off] = wq;
        // cx += crx, cy += cry, xfa += xfx, yfa += yfx, mfx += fxm, mfy += fym
        a.acco[0][off] = acc[0] + crx;
        a.acco[1][off] = acc[1] + cry;
        a.acco[2][off] = acc[2] + xfx;
        a.acco[3][off] = acc[3] + yfx;
        a.acco[4][off] = acc[4] + fxm0;
        a.acco[5][off] = acc[5] + fym0;
      }
    }
    // the next level's d2_1 reuses the flux arrays this level's updates read
    if (k + 1 < k1) __syncthreads();
  }
}

}  // namespace

constexpr int DT_TI = 32, DT_TJ = 8;  // (32 x 16, one CTA of 16 warps per SM: measured slower, 7.78 -> 8.06 ms per step)

int launch_dsw_transport(const DswTpArgs& a0, cudaStream_t st) {
  using L = Dt2Layout<DT_TI, DT_TJ>;
  FV3B_TRY(ensure_smem((const void*)dsw_transport2_kernel<DT_TI, DT_TJ>, L::bytes, "d_sw transport smem attribute"));
  DswTpArgs a = a0;
  const int tiles = cdiv(a.ni, DT_TI) * cdiv(a.nj, DT_TJ);
  a.kchunk = level_chunk(FV3B_TUNE_KCHUNK_DSW_TRANSPORT, tiles, a.nk, cps_of<DT_TI, DT_TJ>());
  dim3 grid(cdiv(a.ni, DT_TI), cdiv(a.nj, DT_TJ), cdiv(a.nk, a.kchunk));
  dsw_transport2_kernel<DT_TI, DT_TJ><<<grid, nt_of<DT_TI, DT_TJ>(), L::bytes, st>>>(a);
  return check_launch("d_sw transport");
}

int dsw_transport_maps(DswTpArgs& a, const Geo& g, const fv3b_field* qbox5, const fv3b_field* acc6,
                       const fv3b_field* met4) {
  (void)acc6;
  using L = Dt2Layout<DT_TI, DT_TJ>;
  for (int f = 0; f < 5; ++f) FV3B_TRY(tensor_map(qbox5[f].data, g.pitch, g.rows, g.levels, L::QW, L::QH, &a.qbox[f]));
  for (int f = 0; f < 4; ++f) FV3B_TRY(tensor_map(met4[f].data, g.pitch, g.rows, 1, L::QW, L::QH, &a.met[f]));
  return FV3B_OK;
}

}  // namespace fv3b
