// K3 d_sw (programs/d_sw.stn; templates.d_sw_stencils).
//
// Two fused kernels per level tile (32 x 16 columns, halo 4):
//   d_sw_transport  d_sw_courant + d_sw_mass + d_sw_heat + d_sw_vert and the
//                   delp / pt / w / accumulator statements of d_sw_update;
//   d_sw_momentum   d_sw_courant + d_sw_ke + d_sw_vort + d_sw_damp and the
//                   u / v statements of d_sw_update.
// The split is exact: the transport group never reads u/v and the momentum
// group never reads delp/pt/w, and every statement of d_sw_update reads the
// pre-update values (RHS materialised before each store, reference.py:293-299;
// offset reads of u/v/w/delp/pt all precede their writes in the .stn).
// All temporaries are shared-memory tiles computed over the rectangles the
// later statements read (extents.py:128-164 restricted to the tile).
#include <string.h>

#include "dsw.cuh"
#include "tile.cuh"

namespace fv3b {

using GD = TileGeo<32, 16, 4, 4>;
constexpr int DSW_NT = 256;

struct DswArgs {
  View u, v, w, delp, pt, uc, vc;
  View cx, cy, xfa, yfa, mfx, mfy;
  View dx, dy, dxc, dyc, rdx, rdy, rdxa, rdya, area, rarea, rarea_c, f0;
  View uo, vo, wo, delpo, pto, cxo, cyo, xfao, yfao, mfxo, mfyo;
  int ni, nj, nk, hx, hy;
  double p1, p2, dt, dddmp, d2_bg, da_min, damp_w;
};

__device__ __forceinline__ double np_min(double a, double b) {
  if (isnan(a) || isnan(b)) return a + b;
  return b < a ? b : a;
}
__device__ __forceinline__ double np_max2(double a, double b) {
  if (isnan(a) || isnan(b)) return a + b;
  return b > a ? b : a;
}

// Courant numbers and area fluxes (d_sw_courant) on x faces [0, TI+1) x
// rows [ja, jb) and y faces [0, TJ+1) x columns [ia, ib).
template <class G>
__device__ __forceinline__ void courant(const DswArgs& a, const Arr<G>& CRX, const Arr<G>& XFX, const Arr<G>& CRY,
                                        const Arr<G>& YFX, int gi0, int gj0, int k, int ja, int jb, int ia, int ib) {
  constexpr int TI = G::TI, TJ = G::TJ;
  const double dt = a.dt;
  each(0, TI + 1, ja, jb, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    const bool ok = gi >= -a.hx + 1 && gi < a.ni + a.hx && gj >= -a.hy && gj < a.nj + a.hy;
    const double uc = ok ? __ldg(a.uc.ptr(gi, gj, k)) : 0.0;
    XFX(i, j) = ok ? dt * uc * met(a.dy, gi, gj) : 0.0;
    CRX(i, j) = ok ? (uc > 0.0 ? dt * uc * met(a.rdxa, gi - 1, gj) : dt * uc * met(a.rdxa, gi, gj)) : 0.0;
  });
  each(ia, ib, 0, TJ + 1, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    const bool ok = gi >= -a.hx && gi < a.ni + a.hx && gj >= -a.hy + 1 && gj < a.nj + a.hy;
    const double vc = ok ? __ldg(a.vc.ptr(gi, gj, k)) : 0.0;
    YFX(i, j) = ok ? dt * vc * met(a.dx, gi, gj) : 0.0;
    CRY(i, j) = ok ? (vc > 0.0 ? dt * vc * met(a.rdya, gi, gj - 1) : dt * vc * met(a.rdya, gi, gj)) : 0.0;
  });
}

// fv_tp_2d of Q (templates.fv_tp_2d) up to the per-face flux pair; results:
// FXO faces [0, TI+1) x rows [0, TJ), FYO columns [0, TI) x faces [0, TJ+1),
// weighted by WX / WY.  Scratch: FY2, FX2, QI, QJ.  Caller syncs before.
template <class G>
__device__ __forceinline__ void tp2d(const DswArgs& a, const Arr<G>& Q, const Arr<G>& CRX, const Arr<G>& XFX,
                                     const Arr<G>& CRY, const Arr<G>& YFX, const Arr<G>& WX, const Arr<G>& WY,
                                     const Arr<G>& FY2, const Arr<G>& FX2, const Arr<G>& QI, const Arr<G>& QJ,
                                     const Arr<G>& FXO, const Arr<G>& FYO, int gi0, int gj0) {
  constexpr int TI = G::TI, TJ = G::TJ;
  const double p1 = a.p1, p2 = a.p2;
  ppm_y(FY2, Q, CRY, -3, TI + 3, 0, TJ + 1, p1, p2);
  ppm_x(FX2, Q, CRX, 0, TI + 1, -3, TJ + 3, p1, p2);
  __syncthreads();
  fill(QI, -3, TI + 3, 0, TJ, [&](int i, int j) {
    const double ar = met(a.area, gi0 + i, gj0 + j);
    return (Q(i, j) * ar + FY2(i, j) * YFX(i, j) - FY2(i, j + 1) * YFX(i, j + 1)) / (ar + YFX(i, j) - YFX(i, j + 1));
  });
  fill(QJ, 0, TI, -3, TJ + 3, [&](int i, int j) {
    const double ar = met(a.area, gi0 + i, gj0 + j);
    return (Q(i, j) * ar + FX2(i, j) * XFX(i, j) - FX2(i + 1, j) * XFX(i + 1, j)) / (ar + XFX(i, j) - XFX(i + 1, j));
  });
  __syncthreads();
  ppm_x(FXO, QI, CRX, 0, TI + 1, 0, TJ, p1, p2);
  ppm_y(FYO, QJ, CRY, 0, TI, 0, TJ + 1, p1, p2);
  __syncthreads();
  fill(FXO, 0, TI + 1, 0, TJ, [&](int i, int j) { return 0.5 * (FXO(i, j) + FX2(i, j)) * WX(i, j); });
  fill(FYO, 0, TI, 0, TJ + 1, [&](int i, int j) { return 0.5 * (FYO(i, j) + FY2(i, j)) * WY(i, j); });
}

__global__ void __launch_bounds__(DSW_NT, 1) d_sw_momentum_kernel(const DswArgs a) {
  extern __shared__ __align__(128) double smem[];
  using G = GD;
  constexpr int TI = G::TI, TJ = G::TJ;
  int s = 0;
  auto arr = [&]() { return Arr<G>{smem + (s++) * G::NA}; };
  const Arr<G> CRX = arr(), XFX = arr(), CRY = arr(), YFX = arr(), U = arr(), V = arr();
  const Arr<G> UB = arr(), CUB = arr(), VB = arr(), CVB = arr(), UU = arr(), VV = arr();
  const Arr<G> WK = arr(), DDV = arr(), FY2 = arr(), FX2 = arr();
  // dead after the KE statement: reused by the vorticity transport
  const Arr<G> QI = CUB, QJ = CVB, FXV = UU, FYV = VV;
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ, k = blockIdx.z;
  const int ni = a.ni, nj = a.nj;
  const double dt = a.dt;

  load(U, a.u, gi0, gj0, k, -3, TI + 3, -3, TJ + 4, ni, nj, a.hx, a.hy);
  load(V, a.v, gi0, gj0, k, -3, TI + 4, -3, TJ + 3, ni, nj, a.hx, a.hy);
  courant(a, CRX, XFX, CRY, YFX, gi0, gj0, k, -3, TJ + 3, -3, TI + 3);
  // d_sw_ke: ub/cub, vb/cvb at corners [0, TI+1) x [0, TJ+1)
  each(0, TI + 1, 0, TJ + 1, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    const double ub = 0.5 * dt * (__ldg(a.uc.ptr(gi, gj - 1, k)) + __ldg(a.uc.ptr(gi, gj, k)));
    UB(i, j) = ub;
    CUB(i, j) = ub > 0.0 ? ub * met(a.rdx, gi - 1, gj) : ub * met(a.rdx, gi, gj);
    const double vb = 0.5 * dt * (__ldg(a.vc.ptr(gi - 1, gj, k)) + __ldg(a.vc.ptr(gi, gj, k)));
    VB(i, j) = vb;
    CVB(i, j) = vb > 0.0 ? vb * met(a.rdy, gi, gj - 1) : vb * met(a.rdy, gi, gj);
  });
  __syncthreads();
  ppm_x(UU, U, CUB, 0, TI + 1, 0, TJ + 1, a.p1, a.p2);
  ppm_y(VV, V, CVB, 0, TI + 1, 0, TJ + 1, a.p1, a.p2);
  // d_sw_vort: absolute vorticity at centres over the transport halo
  fill(WK, -3, TI + 3, -3, TJ + 3, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    return met(a.f0, gi, gj) + met(a.rarea, gi, gj) * (U(i, j) * met(a.dx, gi, gj) - U(i, j + 1) * met(a.dx, gi, gj + 1) +
                                                       V(i + 1, j) * met(a.dy, gi + 1, gj) - V(i, j) * met(a.dy, gi, gj));
  });
  // d_sw_damp: Smagorinsky-scaled divergence damping at corners
  fill(DDV, 0, TI + 1, 0, TJ + 1, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    const double rac = met(a.rarea_c, gi, gj);
    const double ue = U(i, j) * met(a.dyc, gi, gj), uw = U(i - 1, j) * met(a.dyc, gi - 1, gj);
    const double vn = V(i, j) * met(a.dxc, gi, gj), vs = V(i, j - 1) * met(a.dxc, gi, gj - 1);
    const double divg = rac * (ue - uw + vn - vs);
    const double tens = rac * (ue - uw - vn + vs);
    const double smag = dt * sqrt(divg * divg + tens * tens);
    const double dmp = a.da_min * np_max2(a.d2_bg, np_min(0.2, a.dddmp * smag));
    return dmp * divg;
  });
  __syncthreads();
  // ked = 0.5 * (ub * uu + vb * vv)   (into UB)
  fill(UB, 0, TI + 1, 0, TJ + 1, [&](int i, int j) { return 0.5 * (UB(i, j) * UU(i, j) + VB(i, j) * VV(i, j)); });
  __syncthreads();
  // vorticity transport: fv_tp_2d(wk) -> fxv, fyv (area-flux weighted)
  tp2d(a, WK, CRX, XFX, CRY, YFX, XFX, YFX, FY2, FX2, QI, QJ, FXV, FYV, gi0, gj0);
  __syncthreads();
  each(0, TI, 0, TJ, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    if (gi >= ni || gj >= nj) return;
    const double rdx = met(a.rdx, gi, gj), rdy = met(a.rdy, gi, gj);
    *a.uo.ptr(gi, gj, k) = (U(i, j) * met(a.dx, gi, gj) + UB(i, j) - UB(i + 1, j) + FYV(i, j)) * rdx +
                           (DDV(i + 1, j) - DDV(i, j)) * rdx;
    *a.vo.ptr(gi, gj, k) = (V(i, j) * met(a.dy, gi, gj) + UB(i, j) - UB(i, j + 1) - FXV(i, j)) * rdy +
                           (DDV(i, j + 1) - DDV(i, j)) * rdy;
  });
}

}  // namespace fv3b

using namespace fv3b;

// fields (36): u, v, w, delp, pt, uc, vc, cx, cy, xfa, yfa, mfx, mfy (3-D);
// dx, dy, dxc, dyc, rdx, rdy, rdxa, rdya, area, rarea, rarea_c, f0 (2-D);
// u_out, v_out, w_out, delp_out, pt_out, cx_out, cy_out, xfa_out, yfa_out,
// mfx_out, mfy_out (3-D).  The accumulator outputs may alias their inputs
// (pointwise update); the others must not.  scalars: ppm_p1, ppm_p2, dt,
// dddmp, d2_bg, da_min, damp_w.
extern "C" int fv3b_d_sw(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 36 || ns != 7)
    return fail(FV3B_EINVAL, "fv3b_d_sw: expects 36 fields, 7 scalars (got %d, %d)", nf, ns);
  DswArgs a;
  const Halo h0 = {0, 0, 0, 0, 0, 0}, h3 = {3, 3, 3, 3, 0, 0};
  const Halo hu = {3, 3, 3, 4, 0, 0}, hv = {3, 4, 3, 3, 0, 0}, huc = {0, 1, 3, 3, 0, 0}, hvc = {3, 3, 0, 1, 0, 0};
  View* in3[13] = {&a.u, &a.v, &a.w, &a.delp, &a.pt, &a.uc, &a.vc, &a.cx, &a.cy, &a.xfa, &a.yfa, &a.mfx, &a.mfy};
  const Halo hin[13] = {hu, hv, h3, h3, h3, huc, hvc, h0, h0, h0, h0, h0, h0};
  const char* nin[13] = {"u", "v", "w", "delp", "pt", "uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy"};
  for (int t = 0; t < 13; ++t) FV3B_TRY(view_of(f[t], 3, *d, hin[t], nin[t], in3[t]));
  View* m[12] = {&a.dx, &a.dy, &a.dxc, &a.dyc, &a.rdx, &a.rdy, &a.rdxa, &a.rdya, &a.area, &a.rarea, &a.rarea_c, &a.f0};
  const char* nm[12] = {"dx", "dy", "dxc", "dyc", "rdx", "rdy", "rdxa", "rdya", "area", "rarea", "rarea_c", "f0"};
  const Halo hm[12] = {{3, 3, 3, 4, 0, 0}, {3, 4, 3, 3, 0, 0}, {0, 1, 1, 1, 0, 0}, {1, 1, 0, 1, 0, 0},
                       {1, 1, 0, 1, 0, 0}, {0, 1, 1, 1, 0, 0}, {1, 1, 3, 3, 0, 0}, {3, 3, 1, 1, 0, 0},
                       h3, h3, {0, 1, 0, 1, 0, 0}, h3};
  for (int t = 0; t < 12; ++t) FV3B_TRY(view_of(f[13 + t], 2, *d, hm[t], nm[t], m[t]));
  View* out[11] = {&a.uo, &a.vo, &a.wo, &a.delpo, &a.pto, &a.cxo, &a.cyo, &a.xfao, &a.yfao, &a.mfxo, &a.mfyo};
  for (int t = 0; t < 11; ++t) FV3B_TRY(view_of(f[25 + t], 3, *d, h0, "d_sw output", out[t]));
  for (int t = 0; t < 5; ++t)
    if (f[25 + t].data == f[t].data) return fail(FV3B_EINVAL, "fv3b_d_sw: output %d aliases its input", t);
  View v3[24];
  for (int t = 0; t < 13; ++t) v3[t] = *in3[t];
  for (int t = 0; t < 11; ++t) v3[13 + t] = *out[t];
  FV3B_TRY(same_strides(v3, 24, "fv3b_d_sw"));
  a.hx = f[0].halo_lo[0];
  a.hy = f[0].halo_lo[1];
  const int hi_x = f[0].shape[0] - f[0].halo_lo[0] - d->ni, hi_y = f[0].shape[1] - f[0].halo_lo[1] - d->nj;
  a.hx = a.hx < hi_x ? a.hx : hi_x;
  a.hy = a.hy < hi_y ? a.hy : hi_y;
  if (a.hx < 4 || a.hy < 4) return fail(FV3B_ELAYOUT, "fv3b_d_sw: needs a 4-cell allocated halo");
  a.ni = d->ni; a.nj = d->nj; a.nk = d->nk;
  a.p1 = s[0]; a.p2 = s[1]; a.dt = s[2]; a.dddmp = s[3]; a.d2_bg = s[4]; a.da_min = s[5]; a.damp_w = s[6];
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // transport group (delp, pt, w, accumulators): TMA-pipelined level march
  {
    Geo g;
    FV3B_TRY(geo_of(f[0], &g));
    const int tma_fields[] = {2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 19, 20, 21};
    for (int t : tma_fields) {
      Geo h;
      FV3B_TRY(geo_of(f[t], &h));
      if (h.pitch != g.pitch || h.rows != g.rows || (f[t].rank == 3 && h.levels != g.levels) || h.i0 != g.i0 ||
          h.j0 != g.j0)
        return fail(FV3B_ELAYOUT, "fv3b_d_sw: field %d geometry differs from field 0", t);
    }
    DswTpArgs t;
    memset(&t, 0, sizeof t);
    const fv3b_field qb[5] = {f[3], f[4], f[2], f[5], f[6]};        // delp, pt, w, uc, vc
    const fv3b_field ac[6] = {f[7], f[8], f[9], f[10], f[11], f[12]};  // cx, cy, xfa, yfa, mfx, mfy
    const fv3b_field mt[5] = {f[13], f[14], f[19], f[20], f[21]};      // dx, dy, rdxa, rdya, area
    FV3B_TRY(dsw_transport_maps(t, g, qb, ac, mt));
    t.delpo = a.delpo.o;
    t.pto = a.pto.o;
    t.wo = a.wo.o;
    View* ao[6] = {&a.cxo, &a.cyo, &a.xfao, &a.yfao, &a.mfxo, &a.mfyo};
    for (int u = 0; u < 6; ++u) t.acco[u] = ao[u]->o;
    t.rarea = a.rarea.o;
    t.sj = a.u.sj;
    t.sk = a.u.sk;
    t.i0 = g.i0;
    t.j0 = g.j0;
    t.ni = d->ni; t.nj = d->nj; t.nk = d->nk;
    t.p1 = a.p1; t.p2 = a.p2; t.dt = a.dt; t.damp_w = a.damp_w;
    FV3B_TRY(launch_dsw_transport(t, st));
  }
  static bool attr = false;
  const size_t b2 = 16 * GD::NA * sizeof(double);
  if (!attr) {
    if (cudaFuncSetAttribute(d_sw_momentum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b2) != cudaSuccess)
      return check_launch("d_sw smem attribute");
    attr = true;
  }
  dim3 grid(cdiv(d->ni, GD::TI), cdiv(d->nj, GD::TJ), d->nk);
  d_sw_momentum_kernel<<<grid, DSW_NT, b2, st>>>(a);
  return check_launch("d_sw_momentum");
}
