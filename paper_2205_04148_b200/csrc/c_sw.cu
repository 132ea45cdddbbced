// K2 c_sw (programs/c_sw.stn) and the fused C-grid program
// (programs/c_grid.stn = c_sw + riem_solver_c + p_grad_c), plus the D-grid
// nonhydrostatic pair (nh_d.stn, p_grad_d.stn).  templates.c_sw_stencils.
//
// c_sw runs as the TMA level-march kernel of csw_tma.cu.  In the fused
// C-grid program the C-grid thickness / temperature / w are written over the
// one-cell extension (-1) that p_grad_c needs, so the column solver runs on
// the extended domain and no halo exchange separates the stages.
#include <string.h>

#include "column.cuh"
#include "csw.cuh"
#include "tile.cuh"

namespace fv3b {


struct CswArgs {
  View u, v, delp, pt, w;
  View dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc;
  View uc, vc, delpc, ptc, wc;  // outputs (delpc/ptc/wc over the extension if EXT)
  int ni, nj, nk, hx, hy;       // hx/hy: allocated halo of the inputs
  bool own_is, own_ie, own_js, own_je;
  double dt2, a1, a2;
};

// p_grad_c (c_grid.stn, nk+1 domain): uc/vc += C-grid pressure gradient from
// the solver's interface pressure pkc and geopotential gzc (extended by one
// cell), evaluated in place per cell.
struct PgArgs {
  View uc, vc, pk, gz, rdxc, rdyc;
  int ni, nj, nk;  // nk layers
  double dt;
};

// p_grad_d tiling (below): 32 x 8 cells and PG_KC levels per CTA.
#ifndef FV3B_PG_KC
#define FV3B_PG_KC 4
#endif
constexpr int PG_TI = 32, PG_TJ = 8, PG_KC = FV3B_PG_KC;
constexpr int PG_CW = PG_TI + 1, PG_CH = PG_TJ + 1, PG_NP = PG_CW * PG_CH;

// one thread per cell (measured faster here than the shared-memory tiling
// used for p_grad_d: only three columns' interface values are reused)
// PGC_K levels per thread: the interface values of level k+1 serve both k and k+1
// (measured 20 us per step faster than one level per thread; 3 or 4 gain nothing more)
constexpr int PGC_K = 2;
__global__ void p_grad_c_kernel(const PgArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k0 = PGC_K * blockIdx.z;
  if (i >= a.ni) return;
  const double rx = met(a.rdxc, i, j), ry = met(a.rdyc, i, j);
  auto P = [&](int di, int dj, int kk) { return __ldg(a.pk.ptr(i + di, j + dj, kk)); };
  auto Z = [&](int di, int dj, int kk) { return __ldg(a.gz.ptr(i + di, j + dj, kk)); };
  double p0 = P(0, 0, k0), px0 = P(-1, 0, k0), py0 = P(0, -1, k0);
  double z0 = Z(0, 0, k0), zx0 = Z(-1, 0, k0), zy0 = Z(0, -1, k0);
#pragma unroll
  for (int l = 0; l < PGC_K; ++l) {
    const int k = k0 + l;
    if (k >= a.nk) break;
    const double p1 = P(0, 0, k + 1), px1 = P(-1, 0, k + 1), py1 = P(0, -1, k + 1);
    const double z1 = Z(0, 0, k + 1), zx1 = Z(-1, 0, k + 1), zy1 = Z(0, -1, k + 1);
    const double wk = p1 - p0, wkx = px1 - px0, wky = py1 - py0;
    double* uc = a.uc.ptr(i, j, k);
    double* vc = a.vc.ptr(i, j, k);
    *uc = *uc + a.dt * rx / (wkx + wk) * ((zx1 - z0) * (p1 - px0) + (zx0 - z1) * (px1 - p0));
    *vc = *vc + a.dt * ry / (wky + wk) * ((zy1 - z0) * (p1 - py0) + (zy0 - z1) * (py1 - p0));
    p0 = p1; px0 = px1; py0 = py1;
    z0 = z1; zx0 = zx1; zy0 = zy1;
  }
}

// p_grad_d (p_grad_d.stn, nk+1 domain): corner-averaged pressure and
// geopotential, then the D-grid winds' pressure-gradient update.
struct PgdArgs {
  View u, v, pef, gz, rdx, rdy, uo, vo;
  int ni, nj, nk;
  double dt;
};

// Tile kernel: a CTA of 32 x 8 threads owns a 32 x 8 cell tile and PG_KC
// levels.  The corner averages of the tile ((TI+1) x (TJ+1) corners x
// (PG_KC+1) levels, all loads independent) are computed once into shared
// memory, then every thread updates its cell's u and v on the PG_KC levels.
__global__ void __launch_bounds__(PG_TI * PG_TJ) p_grad_d_kernel(const PgdArgs a) {
  __shared__ double spk[PG_KC + 1][PG_NP], sgz[PG_KC + 1][PG_NP];
  const int tid = threadIdx.x + threadIdx.y * PG_TI;
  const int i0 = blockIdx.x * PG_TI, j0 = blockIdx.y * PG_TJ, k0 = blockIdx.z * PG_KC;
  const int nl = min(PG_KC, a.nk - k0);
  const int64_t pj = a.pef.sj, zj = a.gz.sj;
  // corners (i0+ci, j0+cj), ci <= TI, cj <= TJ, levels k0 .. k0+nl
  for (int e = tid; e < (nl + 1) * PG_NP; e += PG_TI * PG_TJ) {
    const int l = e / PG_NP, c = e % PG_NP;
    const int gi = i0 + c % PG_CW, gj = j0 + c / PG_CW;
    if (gi <= a.ni && gj <= a.nj) {
      // pkd = 0.25 * (pef + pef[-1,0,0] + pef[0,-1,0] + pef[-1,-1,0])
      const double* p = a.pef.ptr(gi, gj, k0 + l);
      const double* z = a.gz.ptr(gi, gj, k0 + l);
      spk[l][c] = 0.25 * (__ldg(p) + __ldg(p - 1) + __ldg(p - pj) + __ldg(p - 1 - pj));
      sgz[l][c] = 0.25 * (__ldg(z) + __ldg(z - 1) + __ldg(z - zj) + __ldg(z - 1 - zj));
    }
  }
  __syncthreads();
  const int li = threadIdx.x, lj = threadIdx.y, i = i0 + li, j = j0 + lj;
  if (i >= a.ni || j >= a.nj) return;
  const int c = lj * PG_CW + li;
  const double rx = met(a.rdx, i, j), ry = met(a.rdy, i, j);
  for (int l = 0; l < nl; ++l) {
    const int k = k0 + l;
    const double p00 = spk[l][c], p01 = spk[l + 1][c], g00 = sgz[l][c], g01 = sgz[l + 1][c];
    const double wk = p01 - p00;
    {  // u at (i, j-1/2): corners (i, j) and (i+1, j)
      const double p10 = spk[l][c + 1], p11 = spk[l + 1][c + 1];
      const double g10 = sgz[l][c + 1], g11 = sgz[l + 1][c + 1];
      const double wkx = p11 - p10;
      *a.uo.ptr(i, j, k) = __ldg(a.u.ptr(i, j, k)) + a.dt * rx / (wk + wkx) *
                                                         ((g01 - g10) * (p11 - p00) + (g00 - g11) * (p01 - p10));
    }
    {  // v at (i-1/2, j): corners (i, j) and (i, j+1)
      const double p10 = spk[l][c + PG_CW], p11 = spk[l + 1][c + PG_CW];
      const double g10 = sgz[l][c + PG_CW], g11 = sgz[l + 1][c + PG_CW];
      const double wky = p11 - p10;
      *a.vo.ptr(i, j, k) = __ldg(a.v.ptr(i, j, k)) + a.dt * ry / (wk + wky) *
                                                         ((g01 - g10) * (p11 - p00) + (g00 - g11) * (p01 - p10));
    }
  }
}

// c_sw through the TMA level-march kernel (csw_tma.cu).  in5: u, v, delp,
// pt, w; met9: dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc.
static int run_csw(const fv3b_field* in5, const fv3b_field* met9, const CswArgs& a, bool ext, cudaStream_t st) {
  Geo g;
  FV3B_TRY(geo_of(in5[0], &g));
  for (int t = 0; t < 14; ++t) {
    Geo h;
    const fv3b_field& f = t < 5 ? in5[t] : met9[t - 5];
    FV3B_TRY(geo_of(f, &h));
    if (h.pitch != g.pitch || h.rows != g.rows || (f.rank == 3 && h.levels != g.levels) || h.i0 != g.i0 ||
        h.j0 != g.j0)
      return fail(FV3B_ELAYOUT, "c_sw: field %d geometry differs from u", t);
  }
  CswTmaArgs t;
  memset(&t, 0, sizeof t);
  FV3B_TRY(csw_maps(t, g, in5, met9));
  t.uc = a.uc.o; t.vc = a.vc.o; t.delpc = a.delpc.o; t.ptc = a.ptc.o; t.wc = a.wc.o;
  t.sj = a.u.sj; t.sk = a.u.sk;
  t.i0 = g.i0; t.j0 = g.j0;
  t.ni = a.ni; t.nj = a.nj; t.nk = a.nk;
  t.own_is = a.own_is; t.own_ie = a.own_ie; t.own_js = a.own_js; t.own_je = a.own_je;
  t.dt2 = a.dt2; t.a1 = a.a1; t.a2 = a.a2;
  return launch_csw(t, ext, st);
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
  for (int t = 14; t < 19; ++t)
    for (int u = 0; u < 5; ++u)
      if (f[t].data == f[u].data) return fail(FV3B_EINVAL, "fv3b_c_sw: output %d aliases input %d", t, u);
  return run_csw(f, f + 5, a, false, (cudaStream_t)stream);
}

// c_grid.stn (program domain nk = layers + 1).  fields: u, v, delp, pt, w,
// gz (3-D), dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc, ws (2-D),
// uc, vc (3-D outputs), then the scratch temporaries delpcc, ptcc, wcc,
// pkc, gzc (3-D, >= 1-cell halo).  scalars: dt2, ptop, rdgas, grav, gama,
// p_fac.
extern "C" int fv3b_c_grid(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                           void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 24 || ns != 6)
    return fail(FV3B_EINVAL, "fv3b_c_grid: expects 24 fields, 6 scalars (got %d, %d)", nf, ns);
  if (d->nk < 4) return fail(FV3B_EDOMAIN, "fv3b_c_grid: program domain nk=%d below minimum 4", d->nk);
  // c_sw part: f[0..4] = u, v, delp, pt, w; metrics at f[6..14]
  fv3b_field cf[14];
  for (int t = 0; t < 5; ++t) cf[t] = f[t];
  for (int t = 0; t < 9; ++t) cf[5 + t] = f[6 + t];
  CswArgs a;
  FV3B_TRY(c_sw_common(cf, d, a, 5));
  const Halo h1 = {1, 0, 1, 0, 0, 0};
  View gz, ws, uc, vc, delpcc, ptcc, wcc, pkc, gzc, rsc;
  FV3B_TRY(view_of(f[5], 3, *d, h1, "gz", &gz));
  FV3B_TRY(view_of(f[15], 2, *d, h1, "ws", &ws));
  FV3B_TRY(view_of(f[16], 3, *d, H0, "uc", &uc));
  FV3B_TRY(view_of(f[17], 3, *d, H0, "vc", &vc));
  FV3B_TRY(view_of(f[18], 3, *d, h1, "delpcc", &delpcc));
  FV3B_TRY(view_of(f[19], 3, *d, h1, "ptcc", &ptcc));
  FV3B_TRY(view_of(f[20], 3, *d, h1, "wcc", &wcc));
  FV3B_TRY(view_of(f[21], 3, *d, h1, "pkc", &pkc));
  FV3B_TRY(view_of(f[22], 3, *d, h1, "gzc", &gzc));
  FV3B_TRY(view_of(f[23], 3, *d, h1, "riem scratch", &rsc));
  const View v3[14] = {a.u, a.v, a.delp, a.pt, a.w, gz, uc, vc, delpcc, ptcc, wcc, pkc, gzc, rsc};
  FV3B_TRY(check_same(v3, 14, "fv3b_c_grid"));
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
  FV3B_TRY(run_csw(cf, cf + 5, a, true, st));
  // 2) riem_solver_c on the extended columns [-1, n) x [-1, n)
  RiemArgs r;
  r.dm = delpcc; r.pt = ptcc; r.w = wcc; r.gz = gz; r.ws = ws; r.pef = pkc; r.gzo = gzc; r.scr = rsc;
  r.has_wout = false;
  r.ilo = -1; r.jlo = -1; r.ni_ext = d->ni + 1; r.nj_ext = d->nj + 1;
  r.nk = nkl;
  r.dt = s[0]; r.ptop = s[1]; r.rdgas = s[2]; r.grav = s[3]; r.gama = s[4]; r.p_fac = s[5];
  FV3B_TRY(launch_riem(r, st));
  // 3) p_grad_c on the interior
  PgArgs p;
  p.uc = uc; p.vc = vc; p.pk = pkc; p.gz = gzc; p.rdxc = a.rdxc; p.rdyc = a.rdyc;
  p.ni = d->ni; p.nj = d->nj; p.nk = nkl; p.dt = s[0];
  dim3 grid(cdiv(d->ni, 64), d->nj, cdiv(nkl, PGC_K));
  p_grad_c_kernel<<<grid, 64, 0, st>>>(p);
  return check_launch("p_grad_c");
}

// nh_d.stn (program domain nk = layers + 1): riem solve that writes w back.
// fields: delp, pt, w, gz (3-D), ws (2-D), pef, gz_out, w_out (3-D).
// scalars: ptop, rdgas, grav, gama, p_fac, dt.
extern "C" int fv3b_nh_d(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 9 || ns != 6)
    return fail(FV3B_EINVAL, "fv3b_nh_d: expects 9 fields, 6 scalars (got %d, %d)", nf, ns);
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
  FV3B_TRY(view_of(f[8], 3, *d, H0, "scratch", &r.scr));
  for (int t = 5; t < 9; ++t)
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
  dim3 grid(cdiv(d->ni, PG_TI), cdiv(d->nj, PG_TJ), cdiv(p.nk, PG_KC));
  p_grad_d_kernel<<<grid, dim3(PG_TI, PG_TJ), 0, (cudaStream_t)stream>>>(p);
  return check_launch("p_grad_d");
}
