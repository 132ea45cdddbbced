// K2 c_sw (programs/c_sw.stn) and the fused C-grid program
// (programs/c_grid.stn = c_sw + riem_solver_c + p_grad_c), plus the D-grid
// nonhydrostatic pair (nh_d.stn, p_grad_d.stn).  templates.c_sw_stencils.
//
// c_sw kernel: one CTA = 32 x 16 columns of one level.  u, v, delp, pt, w
// are staged with their halos; ua/va -> uct/vct -> ke/vort are shared-memory
// temporaries computed over the rectangles the later statements read; the
// transport (transportdelp) fluxes are evaluated per output cell.  In the
// fused C-grid program the C-grid thickness / temperature / w are written
// over the one-cell extension (-1) that p_grad_c needs, so the column solver
// runs on the extended domain and no halo exchange separates the stages.
#include "column.cuh"
#include "tile.cuh"

namespace fv3b {

using GC = TileGeo<32, 16, 4, 4>;
constexpr int CSW_NT = 256;
constexpr int CSW_NARR = 11;

struct CswArgs {
  View u, v, delp, pt, w;
  View dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc;
  View uc, vc, delpc, ptc, wc;  // outputs (delpc/ptc/wc over the extension if EXT)
  int ni, nj, nk, hx, hy;       // hx/hy: allocated halo of the inputs
  bool own_is, own_ie, own_js, own_je;
  double dt2, a1, a2;
};

template <bool EXT>
__global__ void __launch_bounds__(CSW_NT, 2) c_sw_kernel(const CswArgs a) {
  extern __shared__ __align__(128) double smem[];
  using G = GC;
  constexpr int TI = G::TI, TJ = G::TJ;
  const Arr<G> U{smem + 0 * G::NA}, V{smem + 1 * G::NA}, DP{smem + 2 * G::NA}, PT{smem + 3 * G::NA},
      WW{smem + 4 * G::NA}, UA{smem + 5 * G::NA}, VA{smem + 6 * G::NA}, UCT{smem + 7 * G::NA},
      VCT{smem + 8 * G::NA}, KE{smem + 9 * G::NA}, VO{smem + 10 * G::NA};
  const int gi0 = blockIdx.x * TI, gj0 = blockIdx.y * TJ, k = blockIdx.z;
  const int ni = a.ni, nj = a.nj;
  const double dt2 = a.dt2, a1 = a.a1, a2 = a.a2;

  load(U, a.u, gi0, gj0, k, -3, TI + 2, -2, TJ + 3, ni, nj, a.hx, a.hy);
  load(V, a.v, gi0, gj0, k, -2, TI + 3, -3, TJ + 2, ni, nj, a.hx, a.hy);
  load(DP, a.delp, gi0, gj0, k, -2, TI + 1, -2, TJ + 1, ni, nj, a.hx, a.hy);
  load(PT, a.pt, gi0, gj0, k, -2, TI + 1, -2, TJ + 1, ni, nj, a.hx, a.hy);
  load(WW, a.w, gi0, gj0, k, -2, TI + 1, -2, TJ + 1, ni, nj, a.hx, a.hy);
  __syncthreads();
  // c_sw_winds: d2a2c (orthogonal)
  fill(UA, -3, TI + 2, -1, TJ + 1, [&](int i, int j) {
    return a2 * (U(i, j - 1) + U(i, j + 2)) + a1 * (U(i, j) + U(i, j + 1));
  });
  fill(VA, -1, TI + 1, -3, TJ + 2, [&](int i, int j) {
    return a2 * (V(i - 1, j) + V(i + 2, j)) + a1 * (V(i, j) + V(i + 1, j));
  });
  __syncthreads();
  fill(UCT, -1, TI + 1, -1, TJ + 1, [&](int i, int j) {
    return a2 * (UA(i - 2, j) + UA(i + 1, j)) + a1 * (UA(i - 1, j) + UA(i, j));
  });
  fill(VCT, -1, TI + 1, -1, TJ + 1, [&](int i, int j) {
    return a2 * (VA(i, j - 2) + VA(i, j + 1)) + a1 * (VA(i, j - 1) + VA(i, j));
  });
  __syncthreads();
  // c_sw_ke_vort
  fill(KE, -1, TI, -1, TJ, [&](int i, int j) {
    const double keu = UA(i, j) > 0.0 ? UCT(i, j) : UCT(i + 1, j);
    const double kev = VA(i, j) > 0.0 ? VCT(i, j) : VCT(i, j + 1);
    return 0.5 * dt2 * (UA(i, j) * keu + VA(i, j) * kev);
  });
  fill(VO, 0, TI + 1, 0, TJ + 1, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    const double fc = met(a.fc, gi, gj), rac = met(a.rarea_c, gi, gj);
    const double ts = UCT(i, j - 1) * met(a.dxc, gi, gj - 1);  // south
    const double tn = UCT(i, j) * met(a.dxc, gi, gj);          // north
    const double te = VCT(i, j) * met(a.dyc, gi, gj);          // east
    const double tw = VCT(i - 1, j) * met(a.dyc, gi - 1, gj);  // west
    double v = fc + rac * (ts - tn + te - tw);
    // tile-corner regions (fire only on owned edges, lower.py:91-93)
    if (gi == 0 && gj == 0 && a.own_is && a.own_js) v = fc + rac * (te - tn - tw);
    if (gi == ni && gj == 0 && a.own_ie && a.own_js) v = fc + rac * (ts - tn - tw);
    if (gi == ni && gj == nj && a.own_ie && a.own_je) v = fc + rac * (ts + te - tw);
    if (gi == 0 && gj == nj && a.own_is && a.own_je) v = fc + rac * (ts - tn + te);
    return v;
  });
  // c_sw_transport (transportdelp), fluxes evaluated per output cell
  {
    // the first tile row/column also owns the -1 extension (EXT)
    const int loi = (EXT && gi0 == 0) ? -1 : 0, loj = (EXT && gj0 == 0) ? -1 : 0;
    each(loi, TI, loj, TJ, [&](int i, int j) {
      const int gi = gi0 + i, gj = gj0 + j;
      if (gi >= ni || gj >= nj) return;
      auto xf = [&](int ii, double& f, double& fp, double& fw) {
        const double utc = dt2 * UCT(ii, j) * met(a.dy, gi0 + ii, gj);
        const bool up = utc > 0.0;
        f = utc * (up ? DP(ii - 1, j) : DP(ii, j));
        fp = f * (up ? PT(ii - 1, j) : PT(ii, j));
        fw = f * (up ? WW(ii - 1, j) : WW(ii, j));
      };
      auto yf = [&](int jj, double& f, double& fp, double& fw) {
        const double vtc = dt2 * VCT(i, jj) * met(a.dx, gi, gj0 + jj);
        const bool up = vtc > 0.0;
        f = vtc * (up ? DP(i, jj - 1) : DP(i, jj));
        fp = f * (up ? PT(i, jj - 1) : PT(i, jj));
        fw = f * (up ? WW(i, jj - 1) : WW(i, jj));
      };
      double fx0, fxp0, fxw0, fx1, fxp1, fxw1, fy0, fyp0, fyw0, fy1, fyp1, fyw1;
      xf(i, fx0, fxp0, fxw0);
      xf(i + 1, fx1, fxp1, fxw1);
      yf(j, fy0, fyp0, fyw0);
      yf(j + 1, fy1, fyp1, fyw1);
      const double ra = met(a.rarea, gi, gj);
      const double dp = DP(i, j);
      const double dpc = dp + (fx0 - fx1 + fy0 - fy1) * ra;
      *a.delpc.ptr(gi, gj, k) = dpc;
      *a.ptc.ptr(gi, gj, k) = (PT(i, j) * dp + (fxp0 - fxp1 + fyp0 - fyp1) * ra) / dpc;
      *a.wc.ptr(gi, gj, k) = (WW(i, j) * dp + (fxw0 - fxw1 + fyw0 - fyw1) * ra) / dpc;
    });
  }
  __syncthreads();
  // c_sw_update
  each(0, TI, 0, TJ, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    if (gi >= ni || gj >= nj) return;
    const double fy1c = dt2 * V(i, j);
    *a.uc.ptr(gi, gj, k) = UCT(i, j) + fy1c * (fy1c > 0.0 ? VO(i, j) : VO(i, j + 1)) +
                           met(a.rdxc, gi, gj) * (KE(i - 1, j) - KE(i, j));
    const double fx1c = dt2 * U(i, j);
    *a.vc.ptr(gi, gj, k) = VCT(i, j) - fx1c * (fx1c > 0.0 ? VO(i, j) : VO(i + 1, j)) +
                           met(a.rdyc, gi, gj) * (KE(i, j - 1) - KE(i, j));
  });
}

// p_grad_c (c_grid.stn, nk+1 domain): uc/vc += C-grid pressure gradient from
// the solver's interface pressure pkc and geopotential gzc (extended by one
// cell), evaluated in place per cell.
struct PgArgs {
  View uc, vc, pk, gz, rdxc, rdyc;
  int ni, nj, nk;  // nk layers
  double dt;
};

__global__ void p_grad_c_kernel(const PgArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= a.ni) return;
  auto P = [&](int di, int dj, int dk) { return *a.pk.ptr(i + di, j + dj, k + dk); };
  auto Z = [&](int di, int dj, int dk) { return *a.gz.ptr(i + di, j + dj, k + dk); };
  const double wk = P(0, 0, 1) - P(0, 0, 0);
  const double wkx = P(-1, 0, 1) - P(-1, 0, 0);
  const double wky = P(0, -1, 1) - P(0, -1, 0);
  double* uc = a.uc.ptr(i, j, k);
  double* vc = a.vc.ptr(i, j, k);
  *uc = *uc + a.dt * met(a.rdxc, i, j) / (wkx + wk) *
                  ((Z(-1, 0, 1) - Z(0, 0, 0)) * (P(0, 0, 1) - P(-1, 0, 0)) +
                   (Z(-1, 0, 0) - Z(0, 0, 1)) * (P(-1, 0, 1) - P(0, 0, 0)));
  *vc = *vc + a.dt * met(a.rdyc, i, j) / (wky + wk) *
                  ((Z(0, -1, 1) - Z(0, 0, 0)) * (P(0, 0, 1) - P(0, -1, 0)) +
                   (Z(0, -1, 0) - Z(0, 0, 1)) * (P(0, -1, 1) - P(0, 0, 0)));
}

// p_grad_d (p_grad_d.stn, nk+1 domain): corner-averaged pressure and
// geopotential, then the D-grid winds' pressure-gradient update.
struct PgdArgs {
  View u, v, pef, gz, rdx, rdy, uo, vo;
  int ni, nj, nk;
  double dt;
};

__global__ void p_grad_d_kernel(const PgdArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= a.ni) return;
  // pkd = 0.25 * (pef + pef[-1,0,0] + pef[0,-1,0] + pef[-1,-1,0])   (corner (i, j))
  auto PK = [&](int ci, int cj, int kk) {
    return 0.25 * (*a.pef.ptr(ci, cj, kk) + *a.pef.ptr(ci - 1, cj, kk) + *a.pef.ptr(ci, cj - 1, kk) +
                   *a.pef.ptr(ci - 1, cj - 1, kk));
  };
  auto GZ = [&](int ci, int cj, int kk) {
    return 0.25 * (*a.gz.ptr(ci, cj, kk) + *a.gz.ptr(ci - 1, cj, kk) + *a.gz.ptr(ci, cj - 1, kk) +
                   *a.gz.ptr(ci - 1, cj - 1, kk));
  };
  const double p00 = PK(i, j, k), p01 = PK(i, j, k + 1);
  const double g00 = GZ(i, j, k), g01 = GZ(i, j, k + 1);
  const double wk = p01 - p00;
  {  // u at (i, j-1/2): corners (i, j) and (i+1, j)
    const double p10 = PK(i + 1, j, k), p11 = PK(i + 1, j, k + 1);
    const double g10 = GZ(i + 1, j, k), g11 = GZ(i + 1, j, k + 1);
    const double wkx = p11 - p10;
    *a.uo.ptr(i, j, k) = *a.u.ptr(i, j, k) + a.dt * met(a.rdx, i, j) / (wk + wkx) *
                                                 ((g01 - g10) * (p11 - p00) + (g00 - g11) * (p01 - p10));
  }
  {  // v at (i-1/2, j): corners (i, j) and (i, j+1)
    const double p10 = PK(i, j + 1, k), p11 = PK(i, j + 1, k + 1);
    const double g10 = GZ(i, j + 1, k), g11 = GZ(i, j + 1, k + 1);
    const double wky = p11 - p10;
    *a.vo.ptr(i, j, k) = *a.v.ptr(i, j, k) + a.dt * met(a.rdy, i, j) / (wk + wky) *
                                                 ((g01 - g10) * (p11 - p00) + (g00 - g11) * (p01 - p10));
  }
}

template <bool EXT>
static int launch_c_sw(const CswArgs& a, cudaStream_t st) {
  const size_t bytes = CSW_NARR * GC::NA * sizeof(double);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(c_sw_kernel<EXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      return check_launch("c_sw smem attribute");
    attr = true;
  }
  dim3 grid(cdiv(a.ni, GC::TI), cdiv(a.nj, GC::TJ), a.nk);
  c_sw_kernel<EXT><<<grid, CSW_NT, bytes, st>>>(a);
  return check_launch("c_sw");
}

static int check_same(const View* v, int n, const char* what) { return same_strides(v, n, what); }

}  // namespace fv3b

using namespace fv3b;

namespace {

const Halo H0 = {0, 0, 0, 0, 0, 0};

int c_sw_common(const fv3b_field* f, const fv3b_domain* d, CswArgs& a, int metric0) {
  // input halos from the program's extents (c_sw.json / c_grid.json)
  const Halo hu = {3, 2, 2, 3, 0, 0}, hv = {2, 3, 3, 2, 0, 0}, hs = {2, 1, 2, 1, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, hu, "u", &a.u));
  FV3B_TRY(view_of(f[1], 3, *d, hv, "v", &a.v));
  FV3B_TRY(view_of(f[2], 3, *d, hs, "delp", &a.delp));
  FV3B_TRY(view_of(f[3], 3, *d, hs, "pt", &a.pt));
  FV3B_TRY(view_of(f[4], 3, *d, hs, "w", &a.w));
  const Halo hdx = {1, 0, 1, 1, 0, 0}, hdy = {1, 1, 1, 0, 0, 0}, hdxc = {0, 1, 1, 1, 0, 0}, hdyc = {1, 1, 0, 1, 0, 0};
  const Halo hc = {0, 1, 0, 1, 0, 0}, hra = {1, 0, 1, 0, 0, 0};
  View* m[9] = {&a.dx, &a.dy, &a.dxc, &a.dyc, &a.rdxc, &a.rdyc, &a.rarea, &a.rarea_c, &a.fc};
  const char* names[9] = {"dx", "dy", "dxc", "dyc", "rdxc", "rdyc", "rarea", "rarea_c", "fc"};
  const Halo hm[9] = {hdx, hdy, hdxc, hdyc, H0, H0, hra, hc, hc};
  for (int t = 0; t < 9; ++t) FV3B_TRY(view_of(f[metric0 + t], 2, *d, hm[t], names[t], m[t]));
  // allocated halo available to the tile loads (uniform device layout)
  a.hx = f[0].halo_lo[0];
  a.hy = f[0].halo_lo[1];
  const int hi_x = f[0].shape[0] - f[0].halo_lo[0] - d->ni, hi_y = f[0].shape[1] - f[0].halo_lo[1] - d->nj;
  a.hx = a.hx < hi_x ? a.hx : hi_x;
  a.hy = a.hy < hi_y ? a.hy : hi_y;
  a.ni = d->ni;
  a.nj = d->nj;
  a.own_is = d->own_i_start;
  a.own_ie = d->own_i_end;
  a.own_js = d->own_j_start;
  a.own_je = d->own_j_end;
  a.a1 = 9.0 / 16.0;
  a.a2 = -1.0 / 16.0;
  return FV3B_OK;
}

}  // namespace

// fields: u, v, delp, pt, w (3-D); dx, dy, dxc, dyc, rdxc, rdyc, rarea,
// rarea_c, fc (2-D); uc, vc, delpc, ptc, wc (3-D outputs).  scalars: dt2.
extern "C" int fv3b_c_sw(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 19 || ns != 1)
    return fail(FV3B_EINVAL, "fv3b_c_sw: expects 19 fields, 1 scalar (got %d, %d)", nf, ns);
  CswArgs a;
  FV3B_TRY(c_sw_common(f, d, a, 5));
  FV3B_TRY(view_of(f[14], 3, *d, H0, "uc", &a.uc));
  FV3B_TRY(view_of(f[15], 3, *d, H0, "vc", &a.vc));
  FV3B_TRY(view_of(f[16], 3, *d, H0, "delpc", &a.delpc));
  FV3B_TRY(view_of(f[17], 3, *d, H0, "ptc", &a.ptc));
  FV3B_TRY(view_of(f[18], 3, *d, H0, "wc", &a.wc));
  const View v3[10] = {a.u, a.v, a.delp, a.pt, a.w, a.uc, a.vc, a.delpc, a.ptc, a.wc};
  FV3B_TRY(check_same(v3, 10, "fv3b_c_sw"));
  a.nk = d->nk;
  a.dt2 = s[0];
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  return launch_c_sw<false>(a, (cudaStream_t)stream);
}

// c_grid.stn (program domain nk = layers + 1).  fields: u, v, delp, pt, w,
// gz (3-D), dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc, ws (2-D),
// uc, vc (3-D outputs), then the scratch temporaries delpcc, ptcc, wcc,
// pkc, gzc (3-D, >= 1-cell halo).  scalars: dt2, ptop, rdgas, grav, gama,
// p_fac.
extern "C" int fv3b_c_grid(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                           void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 23 || ns != 6)
    return fail(FV3B_EINVAL, "fv3b_c_grid: expects 23 fields, 6 scalars (got %d, %d)", nf, ns);
  if (d->nk < 4) return fail(FV3B_EDOMAIN, "fv3b_c_grid: program domain nk=%d below minimum 4", d->nk);
  // c_sw part: f[0..4] = u, v, delp, pt, w; metrics at f[6..14]
  fv3b_field cf[14];
  for (int t = 0; t < 5; ++t) cf[t] = f[t];
  for (int t = 0; t < 9; ++t) cf[5 + t] = f[6 + t];
  CswArgs a;
  FV3B_TRY(c_sw_common(cf, d, a, 5));
  const Halo h1 = {1, 0, 1, 0, 0, 0};
  View gz, ws, uc, vc, delpcc, ptcc, wcc, pkc, gzc;
  FV3B_TRY(view_of(f[5], 3, *d, h1, "gz", &gz));
  FV3B_TRY(view_of(f[15], 2, *d, h1, "ws", &ws));
  FV3B_TRY(view_of(f[16], 3, *d, H0, "uc", &uc));
  FV3B_TRY(view_of(f[17], 3, *d, H0, "vc", &vc));
  FV3B_TRY(view_of(f[18], 3, *d, h1, "delpcc", &delpcc));
  FV3B_TRY(view_of(f[19], 3, *d, h1, "ptcc", &ptcc));
  FV3B_TRY(view_of(f[20], 3, *d, h1, "wcc", &wcc));
  FV3B_TRY(view_of(f[21], 3, *d, h1, "pkc", &pkc));
  FV3B_TRY(view_of(f[22], 3, *d, h1, "gzc", &gzc));
  const View v3[14] = {a.u, a.v, a.delp, a.pt, a.w, gz, uc, vc, delpcc, ptcc, wcc, pkc, gzc, a.u};
  FV3B_TRY(check_same(v3, 13, "fv3b_c_grid"));
  const int nkl = d->nk - 1;
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // 1) c_sw over layers, C-grid state over the -1 extension
  a.uc = uc;
  a.vc = vc;
  a.delpc = delpcc;
  a.ptc = ptcc;
  a.wc = wcc;
  a.nk = nkl;
  a.dt2 = s[0];
  FV3B_TRY(launch_c_sw<true>(a, st));
  // 2) riem_solver_c on the extended columns [-1, n) x [-1, n)
  RiemArgs r;
  r.dm = delpcc; r.pt = ptcc; r.w = wcc; r.gz = gz; r.ws = ws; r.pef = pkc; r.gzo = gzc;
  r.has_wout = false;
  r.ilo = -1; r.jlo = -1; r.ni_ext = d->ni + 1; r.nj_ext = d->nj + 1;
  r.nk = nkl;
  r.dt = s[0]; r.ptop = s[1]; r.rdgas = s[2]; r.grav = s[3]; r.gama = s[4]; r.p_fac = s[5];
  FV3B_TRY(launch_riem(r, st));
  // 3) p_grad_c on the interior
  PgArgs p;
  p.uc = uc; p.vc = vc; p.pk = pkc; p.gz = gzc; p.rdxc = a.rdxc; p.rdyc = a.rdyc;
  p.ni = d->ni; p.nj = d->nj; p.nk = nkl; p.dt = s[0];
  dim3 grid(cdiv(d->ni, 64), d->nj, nkl);
  p_grad_c_kernel<<<grid, 64, 0, st>>>(p);
  return check_launch("p_grad_c");
}

// nh_d.stn (program domain nk = layers + 1): riem solve that writes w back.
// fields: delp, pt, w, gz (3-D), ws (2-D), pef, gz_out, w_out (3-D).
// scalars: ptop, rdgas, grav, gama, p_fac, dt.
extern "C" int fv3b_nh_d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 8 || ns != 6)
    return fail(FV3B_EINVAL, "fv3b_nh_d: expects 8 fields, 6 scalars (got %d, %d)", nf, ns);
  if (d->nk < 4) return fail(FV3B_EDOMAIN, "fv3b_nh_d: program domain nk=%d below minimum 4", d->nk);
  RiemArgs r;
  FV3B_TRY(view_of(f[0], 3, *d, H0, "delp", &r.dm));
  FV3B_TRY(view_of(f[1], 3, *d, H0, "pt", &r.pt));
  FV3B_TRY(view_of(f[2], 3, *d, H0, "w", &r.w));
  FV3B_TRY(view_of(f[3], 3, *d, H0, "gz", &r.gz));
  FV3B_TRY(view_of(f[4], 2, *d, H0, "ws", &r.ws));
  FV3B_TRY(view_of(f[5], 3, *d, H0, "pef", &r.pef));
  FV3B_TRY(view_of(f[6], 3, *d, H0, "gz_out", &r.gzo));
  FV3B_TRY(view_of(f[7], 3, *d, H0, "w_out", &r.wout));
  for (int t = 5; t < 8; ++t)
    for (int u = 0; u < 4; ++u)
      if (f[t].data == f[u].data) return fail(FV3B_EINVAL, "fv3b_nh_d: output %d aliases input %d", t, u);
  r.has_wout = true;
  r.ilo = 0; r.jlo = 0; r.ni_ext = d->ni; r.nj_ext = d->nj;
  r.nk = d->nk - 1;
  r.ptop = s[0]; r.rdgas = s[1]; r.grav = s[2]; r.gama = s[3]; r.p_fac = s[4]; r.dt = s[5];
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  return launch_riem(r, (cudaStream_t)stream);
}

// p_grad_d.stn (program domain nk = layers + 1).  fields: u, v, pef, gz
// (3-D), rdx, rdy (2-D), u_out, v_out (3-D).  scalars: dt.
extern "C" int fv3b_p_grad_d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                             void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 8 || ns != 1)
    return fail(FV3B_EINVAL, "fv3b_p_grad_d: expects 8 fields, 1 scalar (got %d, %d)", nf, ns);
  if (d->nk < 2) return fail(FV3B_EDOMAIN, "fv3b_p_grad_d: program domain nk=%d below minimum 2", d->nk);
  PgdArgs p;
  const Halo h1 = {1, 1, 1, 1, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, H0, "u", &p.u));
  FV3B_TRY(view_of(f[1], 3, *d, H0, "v", &p.v));
  FV3B_TRY(view_of(f[2], 3, *d, h1, "pef", &p.pef));
  FV3B_TRY(view_of(f[3], 3, *d, h1, "gz", &p.gz));
  FV3B_TRY(view_of(f[4], 2, *d, H0, "rdx", &p.rdx));
  FV3B_TRY(view_of(f[5], 2, *d, H0, "rdy", &p.rdy));
  FV3B_TRY(view_of(f[6], 3, *d, H0, "u_out", &p.uo));
  FV3B_TRY(view_of(f[7], 3, *d, H0, "v_out", &p.vo));
  if (f[6].data == f[0].data || f[7].data == f[1].data) return fail(FV3B_EINVAL, "fv3b_p_grad_d: outputs alias inputs");
  p.ni = d->ni; p.nj = d->nj; p.nk = d->nk - 1; p.dt = s[0];
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  dim3 grid(cdiv(d->ni, 64), d->nj, p.nk);
  p_grad_d_kernel<<<grid, 64, 0, (cudaStream_t)stream>>>(p);
  return check_launch("p_grad_d");
}
