// K3a d_sw transport group (programs/d_sw.stn: d_sw_courant, d_sw_mass,
// d_sw_heat, d_sw_vert and the delp / pt / w / accumulator statements of
// d_sw_update), as one level-marching, TMA-pipelined kernel.
//
// Structure (same machinery as the tracer kernel, fv_tp_2d.cu): a CTA owns a
// TI x TJ column tile and walks a chunk of levels.  Per level the inputs
// (delp, pt, w with a 3-cell halo, the C-grid winds uc / vc, the six
// accumulators) arrive by TMA into a double-buffered stage that is fetched
// one level ahead; the 2-D metrics arrive once per CTA.  Each level is three
// transport steps of the same fv_tp_2d chain:
//
//   delp  weights xfx / yfx   -> fxm, fym (mass fluxes, kept in smem), delpn
//   pt    weights fxm / fym   -> pt' = (pt*delp + div(gxp, gyp)*rarea) / delpn
//   w     weights fxm / fym   -> w'  = (w*delp + div(hxw, hyw)*rarea) / delpn + damp_w*lap(w)
//
// exactly the tracer_2d update with dp1 = delp and (mfx, mfy) = (fxm, fym),
// so the statement chain, association and operand order are the .stn's and
// the results are bitwise the interpreter's.  Phase A of a step evaluates
// yppm(q) -> fy2, qi and xppm(q) -> fx2, qj over the tile halo (register
// sliding windows, ppm.cuh); phase B the outer xppm(qi) / yppm(qj) and the
// weighted fluxes; the step's cell update is written during the next step's
// phase A so the y-threads' registers carry it across one barrier.
#include "common.cuh"
#include "dsw.cuh"
#include "ppm.cuh"
#include "tma.cuh"

namespace fv3b {

namespace {

constexpr int SEG = 4;
// threads per CTA / CTAs per SM by tile height: 32x16 tiles run one CTA of 11
// warps per SM, 32x8 tiles two CTAs of 8 warps (<= 128 registers per thread)
template <int TI, int TJ> constexpr int nt_of() { return TI * TJ >= 512 ? 352 : 256; }
template <int TI, int TJ> constexpr int cps_of() { return TI * TJ >= 512 ? 1 : 2; }

__host__ __device__ constexpr int a16(int n) { return (n + 15) / 16 * 16; }

template <int TI, int TJ>
struct DtLayout {
  static constexpr int QW = TI + 10, QH = TJ + 6;  // q-box: i in [-4, TI+6), j in [-3, TJ+3)
  static constexpr int XW = TI + 2, XH = TJ + 6;   // x faces: i in [0, TI+2), j in [-3, TJ+3)
  static constexpr int YW = TI + 8, YH = TJ + 1;   // y faces: i in [-4, TI+4), j in [0, TJ+1)
  static constexpr int JW = TI + 2;                // qj row width
  static constexpr int n_q = a16(QW * QH);
  static constexpr int n_c = a16(TI * TJ);         // interior tile (accumulators, delpn)
  static constexpr int n_x = a16(XW * XH), n_y = a16(YW * YH);
  static constexpr int n_mx = a16(XW * TJ), n_my = a16(TI * YH);
  static constexpr int n_qi = a16(QW * TJ), n_qj = a16(JW * QH);
  // stage: delp, pt, w, uc, vc (q-box); the six accumulators are read by the
  // threads that update them (register prefetch at the level start)
  static constexpr int n_stage = 5 * n_q;
  static constexpr int o_stage = 0;
  static constexpr int o_met = o_stage + 2 * n_stage;  // dx, dy, rdxa, rdya, area (q-box)
  static constexpr int o_crx = o_met + 5 * n_q;
  static constexpr int o_xfx = o_crx + n_x;
  static constexpr int o_cry = o_xfx + n_x;
  static constexpr int o_yfx = o_cry + n_y;
  static constexpr int o_fxm = o_yfx + n_y;
  static constexpr int o_fym = o_fxm + n_mx;
  static constexpr int o_dpn = o_fym + n_my;
  static constexpr int o_qi = o_dpn + n_c;
  static constexpr int o_qj = o_qi + n_qi;
  static constexpr int o_fx2 = o_qj + n_qj;
  static constexpr int o_fy2 = o_fx2 + n_mx;
  static constexpr int o_fx = o_fy2 + n_my;
  static constexpr int total = o_fx + n_mx;
  static constexpr size_t bytes = total * sizeof(double) + 64;
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static_assert(TJ % SEG == 0 && TI % SEG == 0 && QW % 4 == 2 && XW % 4 == 2 && JW % 4 == 2, "tile shape");
  static constexpr uint32_t tx_stage = 5 * QW * QH * 8;
  static constexpr uint32_t tx_met = 5 * QW * QH * 8;
};

template <int TI, int TJ>
__global__ void __launch_bounds__(nt_of<TI, TJ>(), cps_of<TI, TJ>()) dsw_transport_kernel(const __grid_constant__ DswTpArgs a) {
  using L = DtLayout<TI, TJ>;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::total);  // [0],[1] level stages, [2] metrics
  const int tid = threadIdx.x;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ;
  const int k0 = blockIdx.z * a.kchunk;
  const int k1 = min(a.nk, k0 + a.kchunk);
  const int xq = a.i0 + gi0 - 4, yq = a.j0 + gj0 - 3;  // q-box origin (allocated coords)
  const int xx = a.i0 + gi0, yy = a.j0 + gj0;          // interior origin
  const double p1 = a.p1, p2 = a.p2, dt = a.dt;

  auto issue = [&](int k) {  // single thread: level k's stage
    const int b = (k - k0) & 1;
    double* st = smem + L::o_stage + b * L::n_stage;
    mbar_expect_tx(&bar[b], L::tx_stage);
#pragma unroll
    for (int f = 0; f < 5; ++f) tma_load3(st + f * L::n_q, &a.qbox[f], xq, yq, k, &bar[b]);
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
    for (int f = 0; f < 5; ++f) tma_load3(smem + L::o_met + f * L::n_q, &a.met[f], xq, yq, 0, &bar[2]);
    issue(k0);
  }
  const double* sdx = smem + L::o_met;
  const double* sdy = sdx + L::n_q;
  const double* srdxa = sdy + L::n_q;
  const double* srdya = srdxa + L::n_q;
  const double* sarea = srdya + L::n_q;
  double* scrx = smem + L::o_crx;  // XW, origin (0, -3)
  double* sxfx = smem + L::o_xfx;
  double* scry = smem + L::o_cry;  // YW, origin (-4, 0)
  double* syfx = smem + L::o_yfx;
  double* sfxm = smem + L::o_fxm;  // XW, origin (0, 0)
  double* sfym = smem + L::o_fym;  // TI, origin (0, 0)
  double* sdpn = smem + L::o_dpn;  // TI, origin (0, 0)
  double* sqi = smem + L::o_qi;    // QW, origin (-4, 0)
  double* sqj = smem + L::o_qj;    // JW, origin (0, -3)
  double* sfx2 = smem + L::o_fx2;  // XW, origin (0, 0)
  double* sfy2 = smem + L::o_fy2;  // TI, origin (0, 0)
  double* sfx = smem + L::o_fx;    // XW, origin (0, 0)
  auto QB = [&](auto* p, int i, int j) { return p + (j + 3) * L::QW + (i + 4); };
  auto CX = [&](auto* p, int i, int j) { return p + (j + 3) * L::XW + i; };
  auto CY = [&](auto* p, int i, int j) { return p + j * L::YW + (i + 4); };
  if (k1 > k0) mbar_wait(&bar[2], 0);

  constexpr int NSEG = TI / SEG;
  static_assert((TI + 6) * (TJ / SEG) + (TJ + 6) * (TI / SEG) <= nt_of<TI, TJ>(), "one phase-A item per thread");
  constexpr int NX2 = TJ * NSEG, NY2 = TI * (TJ / SEG);
  static_assert(NX2 + NY2 <= nt_of<TI, TJ>(), "one item per thread in phase B");
  // phase-B y threads own a column segment for the whole CTA (as the tracer)
  const bool yth = tid >= NX2 && tid < NX2 + NY2;
  const int ci2 = yth ? (tid - NX2) % TI : 0;
  const int jb2 = yth ? ((tid - NX2) / TI) * SEG : 0;
  const int gi2 = gi0 + ci2;
  // phase-A worker slot: the y threads (which also write the pending cell
  // updates in phase A) take items only after every other thread has one
  const int wslot = tid < NX2 ? tid : (yth ? nt_of<TI, TJ>() - NY2 + (tid - NX2) : tid - NY2);
  double ra[SEG];
#pragma unroll
  for (int u = 0; u < SEG; ++u) {
    const int gj = gj0 + jb2 + u;
    ra[u] = (yth && gi2 < a.ni && gj < a.nj) ? a.rarea[gi2 + (int64_t)gj * a.sj] : 0.0;
  }
  double fy[SEG + 1], dpa[SEG], dpb[SEG];
  int pend_k = -1, pend_q = 0;  // step whose cell update is pending
  constexpr int NT = nt_of<TI, TJ>(), NACC = (6 * TI * TJ + NT - 1) / NT;
  double accv[NACC];  // this thread's accumulator cells of the current level
  const int64_t sj = a.sj, sk = a.sk;

  // cell updates of the previous step (y threads; reads sfx / stage tiles)
  auto write_pending = [&]() {
    if (!yth || pend_k < 0) return;
    const double* st = smem + L::o_stage + ((pend_k - k0) & 1) * L::n_stage;
    const double* Q = st + pend_q * L::n_q;  // pt or w tile
    double* qo = pend_q == 1 ? a.pto : a.wo;
#pragma unroll
    for (int u = 0; u < SEG; ++u) {
      const int j = jb2 + u, gj = gj0 + j;
      if (gi2 < a.ni && gj < a.nj) {
        const int64_t off = gi2 + gj * sj + (int64_t)pend_k * sk;
        const double qc = *QB(Q, ci2, j);
        const double div = (sfx[j * L::XW + ci2] - sfx[j * L::XW + ci2 + 1] + fy[u] - fy[u + 1]) * ra[u];
        double r = (qc * dpa[u] + div) / dpb[u];
        if (pend_q == 2)
          r = r + a.damp_w * (*QB(Q, ci2 - 1, j) + *QB(Q, ci2 + 1, j) + *QB(Q, ci2, j - 1) + *QB(Q, ci2, j + 1) -
                              4.0 * qc);
        qo[off] = r;
      }
    }
  };

  for (int k = k0; k < k1; ++k) {
    const double* st = smem + L::o_stage + ((k - k0) & 1) * L::n_stage;
    const double* sdp = st;
    const double* suc = st + 3 * L::n_q;
    const double* svc = st + 4 * L::n_q;
    for (int q = 0; q < 3; ++q) {
      const double* Q = st + q * L::n_q;
      if (q == 0) {
        // ---- level start: accumulator prefetch; previous level's w update;
        //      this level's courant ------------------------------------------
#pragma unroll
        for (int m = 0; m < NACC; ++m) {
          const int e = tid + m * NT;
          const int f = e / (TI * TJ), c = e % (TI * TJ);
          const int gi = gi0 + c % TI, gj = gj0 + c / TI;
          accv[m] = (e < 6 * TI * TJ && gi < a.ni && gj < a.nj) ? a.acci[f < 6 ? f : 0][gi + gj * sj + (int64_t)k * sk]
                                                                : 0.0;
        }
        write_pending();
        mbar_wait(&bar[(k - k0) & 1], ((k - k0) >> 1) & 1);
        // d_sw_courant: xfx = dt*uc*dy ; crx = select(uc > 0, dt*uc*rdxa[-1,0], dt*uc*rdxa)
        for (int e = tid; e < L::XW * L::XH; e += blockDim.x) {
          const int i = e % L::XW, j = e / L::XW - 3;
          const double uc = *QB(suc, i, j);
          *CX(sxfx, i, j) = dt * uc * *QB(sdy, i, j);
          *CX(scrx, i, j) = uc > 0.0 ? dt * uc * *QB(srdxa, i - 1, j) : dt * uc * *QB(srdxa, i, j);
        }
        // yfx = dt*vc*dx ; cry = select(vc > 0, dt*vc*rdya[0,-1], dt*vc*rdya)
        for (int e = tid; e < L::YW * L::YH; e += blockDim.x) {
          const int i = e % L::YW - 4, j = e / L::YW;
          const double vc = *QB(svc, i, j);
          *CY(syfx, i, j) = dt * vc * *QB(sdx, i, j);
          *CY(scry, i, j) = vc > 0.0 ? dt * vc * *QB(srdya, i, j - 1) : dt * vc * *QB(srdya, i, j);
        }
        __syncthreads();
      } else if (q == 1) {
        // ---- delp step done: delpn, delp', accumulators; prefetch level k+1 --
        if (tid == 0 && k + 1 < k1) {
          fence_async_smem();
          issue(k + 1);
        }
        if (yth) {
#pragma unroll
          for (int u = 0; u < SEG; ++u) {
            const int j = jb2 + u, gj = gj0 + j;
            // delpn = delp + (fxm - fxm[1,0,0] + fym - fym[0,1,0]) * rarea
            const double dp = *QB(sdp, ci2, j);
            const double dn = dp + (sfxm[j * L::XW + ci2] - sfxm[j * L::XW + ci2 + 1] + sfym[j * TI + ci2] -
                                    sfym[(j + 1) * TI + ci2]) * ra[u];
            sdpn[j * TI + ci2] = dn;
            if (gi2 < a.ni && gj < a.nj) a.delpo[gi2 + gj * sj + (int64_t)k * sk] = dn;
          }
        }
        // cx += crx, cy += cry, xfa += xfx, yfa += yfx, mfx += fxm, mfy += fym
#pragma unroll
        for (int m = 0; m < NACC; ++m) {
          const int e = tid + m * NT;
          const int f = e / (TI * TJ), c = e % (TI * TJ);
          const int i = c % TI, j = c / TI, gi = gi0 + i, gj = gj0 + j;
          if (e >= 6 * TI * TJ || gi >= a.ni || gj >= a.nj) continue;
          double d;
          switch (f) {
            case 0: d = *CX(scrx, i, j); break;
            case 1: d = *CY(scry, i, j); break;
            case 2: d = *CX(sxfx, i, j); break;
            case 3: d = *CY(syfx, i, j); break;
            case 4: d = sfxm[j * L::XW + i]; break;
            default: d = sfym[j * TI + i]; break;
          }
          a.acco[f][gi + gj * sj + (int64_t)k * sk] = accv[m] + d;
        }
      } else {
        write_pending();  // pt
      }

      // ---- phase A: yppm(q) -> fy2, qi ; xppm(q) -> fx2, qj -----------------
      {
        constexpr int NCY = TI + 6, NSY = TJ / SEG;  // columns i in [-3, TI+3)
        constexpr int NRX = TJ + 6, NSX = TI / SEG;  // rows j in [-3, TJ+3)
        constexpr int NY = NCY * NSY, NX = NRX * NSX;
        for (int item = wslot; item < NY + NX; item += blockDim.x) {
          if (item < NY) {
            const int ci = item % NCY - 3, jb = (item / NCY) * SEG;
            double f[SEG + 1];
            ppm_line<SEG + 1>(QB(Q, ci, jb), L::QW, CY(scry, ci, jb), L::YW, p1, p2, f);
#pragma unroll
            for (int u = 0; u < SEG; ++u) {
              const int j = jb + u;
              const double ar = *QB(sarea, ci, j);
              const double y0 = *CY(syfx, ci, j), y1 = *CY(syfx, ci, j + 1);
              sqi[j * L::QW + ci + 4] = (*QB(Q, ci, j) * ar + f[u] * y0 - f[u + 1] * y1) / (ar + y0 - y1);
            }
            if (ci >= 0 && ci < TI) {
#pragma unroll
              for (int u = 0; u < SEG; ++u) sfy2[(jb + u) * TI + ci] = f[u];
              if (jb + SEG == TJ) sfy2[TJ * TI + ci] = f[SEG];
            }
          } else {
            const int it = item - NY;
            const int rj = it % NRX - 3, ib = (it / NRX) * SEG;
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
        }
      }
      __syncthreads();

      // ---- phase B: xppm(qi) -> x fluxes ; yppm(qj) -> y fluxes ----------
      if (tid < NX2) {
        const int rj = tid % TJ, ib = (tid / TJ) * SEG;
        double f[SEG + 1];
        ppm_line<SEG + 1>(sqi + rj * L::QW + ib + 4, 1, CX(scrx, ib, rj), 1, p1, p2, f);
        const int nf = (ib + SEG == TI) ? SEG + 1 : SEG;
        double* out = q == 0 ? sfxm : sfx;
#pragma unroll
        for (int u = 0; u < SEG + 1; ++u) {
          if (u < nf) {
            const int i = ib + u;
            const double w = q == 0 ? *CX(sxfx, i, rj) : sfxm[rj * L::XW + i];
            out[rj * L::XW + i] = 0.5 * (f[u] + sfx2[rj * L::XW + i]) * w;
          }
        }
      } else if (yth) {
        ppm_line<SEG + 1>(sqj + (jb2 + 3) * L::JW + ci2, L::JW, CY(scry, ci2, jb2), L::YW, p1, p2, fy);
#pragma unroll
        for (int u = 0; u < SEG + 1; ++u) {
          const int j = jb2 + u;
          const double w = q == 0 ? *CY(syfx, ci2, j) : sfym[j * TI + ci2];
          fy[u] = 0.5 * (fy[u] + sfy2[j * TI + ci2]) * w;
        }
        if (q == 0) {
#pragma unroll
          for (int u = 0; u < SEG; ++u) sfym[(jb2 + u) * TI + ci2] = fy[u];
          if (jb2 + SEG == TJ) sfym[TJ * TI + ci2] = fy[SEG];
        } else {
#pragma unroll
          for (int u = 0; u < SEG; ++u) {
            dpa[u] = *QB(sdp, ci2, jb2 + u);
            dpb[u] = sdpn[(jb2 + u) * TI + ci2];
          }
          pend_k = k;
          pend_q = q;
        }
      }
      __syncthreads();
    }
  }
  write_pending();
}

}  // namespace

constexpr int DT_TI = 32, DT_TJ = 8;

int launch_dsw_transport(const DswTpArgs& a0, cudaStream_t st) {
  using L = DtLayout<DT_TI, DT_TJ>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(dsw_transport_kernel<DT_TI, DT_TJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)L::bytes) != cudaSuccess)
      return check_launch("d_sw transport smem attribute");
    attr = true;
  }
  DswTpArgs a = a0;
  const int tiles = cdiv(a.ni, DT_TI) * cdiv(a.nj, DT_TJ);
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // ~4 waves of one CTA per SM, at least 2 levels per CTA so the prefetch overlaps
  (void)sms;
  a.kchunk = level_chunk(tiles, a.nk, cps_of<DT_TI, DT_TJ>());
  dim3 grid(cdiv(a.ni, DT_TI), cdiv(a.nj, DT_TJ), cdiv(a.nk, a.kchunk));
  dsw_transport_kernel<DT_TI, DT_TJ><<<grid, nt_of<DT_TI, DT_TJ>(), L::bytes, st>>>(a);
  return check_launch("d_sw transport");
}

int dsw_transport_maps(DswTpArgs& a, const Geo& g, const fv3b_field* qbox5, const fv3b_field* acc6,
                       const fv3b_field* met5) {
  using L = DtLayout<DT_TI, DT_TJ>;
  for (int f = 0; f < 5; ++f) FV3B_TRY(tensor_map(qbox5[f].data, g.pitch, g.rows, g.levels, L::QW, L::QH, &a.qbox[f]));
  for (int f = 0; f < 5; ++f) FV3B_TRY(tensor_map(met5[f].data, g.pitch, g.rows, 1, L::QW, L::QH, &a.met[f]));
  return FV3B_OK;
}

}  // namespace fv3b
