// K2 c_sw (programs/c_sw.stn; the c_sw part of c_grid.stn) as a
// TMA-pipelined level-marching kernel (the d_sw kernels' machinery).
//
// A CTA owns a 32 x 16 column tile and walks a chunk of levels; u, v, delp,
// pt, w arrive per level by TMA into a double-buffered stage (fetched one
// level ahead), the nine metrics once per CTA.  Per level:
//   S0  the previous level's c_sw_update (uc, vc) from its kept UCT / VCT /
//       KE / VORT tiles; d2a2c ua, va;
//   S1  uct, vct;
//   S2  ke, vorticity (corner regions fire on owned edges only,
//       lower.py:91-93) and the transportdelp fluxes -> delpc, ptc, wc,
//       written over the -1 extension when EXT (c_grid: the column solver
//       and p_grad_c need them there).
// Statement order, association and select semantics are the .stn's, so the
// results are bitwise the interpreter's.
#include "common.cuh"
#include "csw.cuh"
#include "fastdiv.cuh"
#include "tma.cuh"

namespace fv3b {

namespace {

// 32x8 tiles: two CTAs of 11 warps per SM (112 KB of shared memory each)
#ifndef FV3B_CS_NT
#define FV3B_CS_NT 352  // 11 warps: 0.2% faster per step than 10 (same-box A/B), 10 1% faster than 8, 12 no better
#endif
constexpr int CS_NT = FV3B_CS_NT;

__host__ __device__ constexpr int a16(int n) { return (n + 15) / 16 * 16; }

template <int TI, int TJ>
struct CsLayout {
  static constexpr int BW = TI + 8, BH = TJ + 6;  // box: i in [-4, TI+4), j in [-3, TJ+3)
  static constexpr int n_b = a16(BW * BH);
  static constexpr int n_stage = 5 * n_b;            // u, v, delp, pt, w
  static constexpr int o_met = 2 * n_stage;          // dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc
  static constexpr int o_tmp = o_met + 9 * n_b;      // ua, va, uct, vct, ke, vort
  static constexpr int total = o_tmp + 6 * n_b;
  static constexpr size_t bytes = total * sizeof(double) + 64;
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static constexpr uint32_t tx_stage = 5 * BW * BH * 8;
  static constexpr uint32_t tx_met = 9 * BW * BH * 8;
};

template <int TI, int TJ, bool EXT>
__global__ void __launch_bounds__(CS_NT, 2) csw_kernel(const __grid_constant__ CswTmaArgs a) {
  using L = CsLayout<TI, TJ>;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::total);
  const int tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ;
  const int k0 = blockIdx.z * a.kchunk;
  const int k1 = min(a.nk, k0 + a.kchunk);
  const int xb = a.i0 + gi0 - 4, yb = a.j0 + gj0 - 3;
  const int ni = a.ni, nj = a.nj;
  const double dt2 = a.dt2, a1 = a.a1, a2 = a.a2;

  auto issue = [&](int k) {
    const int b = (k - k0) & 1;
    double* st = smem + b * L::n_stage;
    mbar_expect_tx(&bar[b], L::tx_stage);
#pragma unroll
    for (int f = 0; f < 5; ++f) tma_load3(st + f * L::n_b, &a.in[f], xb, yb, k, &bar[b]);
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
#pragma unroll
    for (int f = 0; f < 9; ++f) tma_load3(smem + L::o_met + f * L::n_b, &a.met[f], xb, yb, 0, &bar[2]);
    issue(k0);
  }
  auto B = [&](auto* p, int i, int j) -> auto& { return p[(j + 3) * L::BW + (i + 4)]; };
  const double* sdx = smem + L::o_met;
  const double* sdy = sdx + L::n_b;
  const double* sdxc = sdy + L::n_b;
  const double* sdyc = sdxc + L::n_b;
  const double* srdxc = sdyc + L::n_b;
  const double* srdyc = srdxc + L::n_b;
  const double* srarea = srdyc + L::n_b;
  const double* srac = srarea + L::n_b;
  const double* sfc = srac + L::n_b;
  double* UA = smem + L::o_tmp;
  double* VA = UA + L::n_b;
  double* UCT = VA + L::n_b;
  double* VCT = UCT + L::n_b;
  double* KE = VCT + L::n_b;
  double* VO = KE + L::n_b;
  if (k1 > k0) mbar_wait(&bar[2], 0);
  const int64_t sj = a.sj, sk = a.sk;
  int pend_k = -1;

  // c_sw_update of level pend_k over the interior tile
  auto update = [&]() {
    if (pend_k < 0) return;
    const double* st = smem + ((pend_k - k0) & 1) * L::n_stage;
    const double* U = st;
    const double* V = st + L::n_b;
    for (int e = tid; e < TI * TJ; e += blockDim.x) {
      const int i = e % TI, j = e / TI, gi = gi0 + i, gj = gj0 + j;
      if (gi >= ni || gj >= nj) continue;
      const int64_t off = gi + gj * sj + (int64_t)pend_k * sk;
      const double fy1c = dt2 * B(V, i, j);
      a.uc[off] = B(UCT, i, j) + fy1c * (fy1c > 0.0 ? B(VO, i, j) : B(VO, i, j + 1)) +
                  B(srdxc, i, j) * (B(KE, i - 1, j) - B(KE, i, j));
      const double fx1c = dt2 * B(U, i, j);
      a.vc[off] = B(VCT, i, j) - fx1c * (fx1c > 0.0 ? B(VO, i, j) : B(VO, i + 1, j)) +
                  B(srdyc, i, j) * (B(KE, i, j - 1) - B(KE, i, j));
    }
  };

  for (int k = k0; k < k1; ++k) {
    const double* st = smem + ((k - k0) & 1) * L::n_stage;
    const double* U = st;
    const double* V = st + L::n_b;
    const double* DP = st + 2 * L::n_b;
    const double* PT = st + 3 * L::n_b;
    const double* WW = st + 4 * L::n_b;
    // ---- S0: previous level's update; d2a2c ua / va ----------------------
    update();
    mbar_wait(&bar[(k - k0) & 1], ((k - k0) >> 1) & 1);
    // ua over [-3, TI+2) x [-1, TJ+1) ; va over [-1, TI+1) x [-3, TJ+2)
    for (int e = tid; e < (TI + 5) * (TJ + 2); e += blockDim.x) {
      const int i = e % (TI + 5) - 3, j = e / (TI + 5) - 1;
      B(UA, i, j) = a2 * (B(U, i, j - 1) + B(U, i, j + 2)) + a1 * (B(U, i, j) + B(U, i, j + 1));
    }
    for (int e = tid; e < (TI + 2) * (TJ + 5); e += blockDim.x) {
      const int i = e % (TI + 2) - 1, j = e / (TI + 2) - 3;
      B(VA, i, j) = a2 * (B(V, i - 1, j) + B(V, i + 2, j)) + a1 * (B(V, i, j) + B(V, i + 1, j));
    }
    __syncthreads();
    // ---- S1: uct / vct over [-1, TI+1) x [-1, TJ+1) ------------------------
    if (tid == 0 && k + 1 < k1) {
      fence_async_smem();
      issue(k + 1);
    }
    for (int e = tid; e < (TI + 2) * (TJ + 2); e += blockDim.x) {
      const int i = e % (TI + 2) - 1, j = e / (TI + 2) - 1;
      B(UCT, i, j) = a2 * (B(UA, i - 2, j) + B(UA, i + 1, j)) + a1 * (B(UA, i - 1, j) + B(UA, i, j));
      B(VCT, i, j) = a2 * (B(VA, i, j - 2) + B(VA, i, j + 1)) + a1 * (B(VA, i, j - 1) + B(VA, i, j));
    }
    __syncthreads();
    // ---- S2: ke, vorticity, transportdelp ---------------------------------
    for (int e = tid; e < (TI + 1) * (TJ + 1); e += blockDim.x) {
      const int i = e % (TI + 1) - 1, j = e / (TI + 1) - 1;  // ke over [-1, TI) x [-1, TJ)
      const double keu = B(UA, i, j) > 0.0 ? B(UCT, i, j) : B(UCT, i + 1, j);
      const double kev = B(VA, i, j) > 0.0 ? B(VCT, i, j) : B(VCT, i, j + 1);
      B(KE, i, j) = 0.5 * dt2 * (B(UA, i, j) * keu + B(VA, i, j) * kev);
    }
    for (int e = tid; e < (TI + 1) * (TJ + 1); e += blockDim.x) {
      const int i = e % (TI + 1), j = e / (TI + 1);  // vorticity over corners [0, TI+1) x [0, TJ+1)
      const int gi = gi0 + i, gj = gj0 + j;
      const double fc = B(sfc, i, j), rac = B(srac, i, j);
      const double ts = B(UCT, i, j - 1) * B(sdxc, i, j - 1);  // south
      const double tn = B(UCT, i, j) * B(sdxc, i, j);          // north
      const double te = B(VCT, i, j) * B(sdyc, i, j);          // east
      const double tw = B(VCT, i - 1, j) * B(sdyc, i - 1, j);  // west
      double v = fc + rac * (ts - tn + te - tw);
      if (gi == 0 && gj == 0 && a.own_is && a.own_js) v = fc + rac * (te - tn - tw);
      if (gi == ni && gj == 0 && a.own_ie && a.own_js) v = fc + rac * (ts - tn - tw);
      if (gi == ni && gj == nj && a.own_ie && a.own_je) v = fc + rac * (ts + te - tw);
      if (gi == 0 && gj == nj && a.own_is && a.own_je) v = fc + rac * (ts - tn + te);
      B(VO, i, j) = v;
    }
    {
      const int loi = (EXT && gi0 == 0) ? -1 : 0, loj = (EXT && gj0 == 0) ? -1 : 0;
      const int w = TI - loi, n = w * (TJ - loj);
      for (int e = tid; e < n; e += blockDim.x) {
        const int i = loi + e % w, j = loj + e / w, gi = gi0 + i, gj = gj0 + j;
        if (gi >= ni || gj >= nj) continue;
        auto xf = [&](int ii, double& f, double& fp, double& fw) {
          const double utc = dt2 * B(UCT, ii, j) * B(sdy, ii, j);
          const bool up = utc > 0.0;
          f = utc * (up ? B(DP, ii - 1, j) : B(DP, ii, j));
          fp = f * (up ? B(PT, ii - 1, j) : B(PT, ii, j));
          fw = f * (up ? B(WW, ii - 1, j) : B(WW, ii, j));
        };
        auto yf = [&](int jj, double& f, double& fp, double& fw) {
          const double vtc = dt2 * B(VCT, i, jj) * B(sdx, i, jj);
          const bool up = vtc > 0.0;
          f = vtc * (up ? B(DP, i, jj - 1) : B(DP, i, jj));
          fp = f * (up ? B(PT, i, jj - 1) : B(PT, i, jj));
          fw = f * (up ? B(WW, i, jj - 1) : B(WW, i, jj));
        };
        double fx0, fxp0, fxw0, fx1, fxp1, fxw1, fy0, fyp0, fyw0, fy1, fyp1, fyw1;
        xf(i, fx0, fxp0, fxw0);
        xf(i + 1, fx1, fxp1, fxw1);
        yf(j, fy0, fyp0, fyw0);
        yf(j + 1, fy1, fyp1, fyw1);
        const double ra = B(srarea, i, j);
        const double dp = B(DP, i, j);
        const double dpc = dp + (fx0 - fx1 + fy0 - fy1) * ra;
        const int64_t off = gi + gj * sj + (int64_t)k * sk;
        a.delpc[off] = dpc;
        // ptc and wc share the divisor delpc: one refined reciprocal (fastdiv.cuh)
        const double np = B(PT, i, j) * dp + (fxp0 - fxp1 + fyp0 - fyp1) * ra;
        const double nw = B(WW, i, j) * dp + (fxw0 - fxw1 + fyw0 - fyw1) * ra;
        bool ok = true;
        const double r = rcp_fast(dpc);
        double vp = div_fast_r(np, dpc, r, ok), vw = div_fast_r(nw, dpc, r, ok);
        if (!ok) {
          vp = np / dpc;
          vw = nw / dpc;
        }
        a.ptc[off] = vp;
        a.wc[off] = vw;
      }
    }
    pend_k = k;
    __syncthreads();
  }
  update();
}

}  // namespace

constexpr int CS_TI = 32, CS_TJ = 8;

int csw_maps(CswTmaArgs& a, const Geo& g, const fv3b_field* in5, const fv3b_field* met9) {
  using L = CsLayout<CS_TI, CS_TJ>;
  for (int f = 0; f < 5; ++f) FV3B_TRY(tensor_map(in5[f].data, g.pitch, g.rows, g.levels, L::BW, L::BH, &a.in[f]));
  for (int f = 0; f < 9; ++f) FV3B_TRY(tensor_map(met9[f].data, g.pitch, g.rows, 1, L::BW, L::BH, &a.met[f]));
  return FV3B_OK;
}

template <bool EXT>
static int launch_t(const CswTmaArgs& a0, cudaStream_t st) {
  using L = CsLayout<CS_TI, CS_TJ>;
  FV3B_TRY(ensure_smem((const void*)csw_kernel<CS_TI, CS_TJ, EXT>, L::bytes, "c_sw smem attribute"));
  CswTmaArgs a = a0;
  const int tiles = cdiv(a.ni, CS_TI) * cdiv(a.nj, CS_TJ);
  a.kchunk = level_chunk(FV3B_TUNE_KCHUNK_CSW, tiles, a.nk, 2);
  dim3 grid(cdiv(a.ni, CS_TI), cdiv(a.nj, CS_TJ), cdiv(a.nk, a.kchunk));
  csw_kernel<CS_TI, CS_TJ, EXT><<<grid, CS_NT, L::bytes, st>>>(a);
  return check_launch("c_sw");
}

int launch_csw(const CswTmaArgs& a, bool ext, cudaStream_t st) { return ext ? launch_t<true>(a, st) : launch_t<false>(a, st); }

}  // namespace fv3b
