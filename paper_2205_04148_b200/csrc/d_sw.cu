// K3 d_sw (programs/d_sw.stn; templates.d_sw_stencils): ABI entry point.
//
// Two fused, TMA-pipelined level-marching kernels:
//   dsw_transport.cu  d_sw_courant + d_sw_mass + d_sw_heat + d_sw_vert and the
//                     delp / pt / w / accumulator statements of d_sw_update;
//   dsw_momentum.cu   d_sw_courant + d_sw_ke + d_sw_vort + d_sw_damp and the
//                     u / v statements of d_sw_update.
// The split is exact: the transport group never reads u/v and the momentum
// group never reads delp/pt/w, and every statement of d_sw_update reads the
// pre-update values (RHS materialised before each store, reference.py:293-299;
// offset reads of u/v/w/delp/pt all precede their writes in the .stn).
#include <string.h>

#include "dsw.cuh"

namespace fv3b {

struct DswArgs {
  View u, v, w, delp, pt, uc, vc;
  View cx, cy, xfa, yfa, mfx, mfy;
  View dx, dy, dxc, dyc, rdx, rdy, rdxa, rdya, area, rarea, rarea_c, f0, del6_u, del6_v;
  View uo, vo, wo, delpo, pto, cxo, cyo, xfao, yfao, mfxo, mfyo;
  int ni, nj, nk, hx, hy;
  double p1, p2, dt, dddmp, d2_bg, da_min, damp4, damp4h, dampv;
};

}  // namespace fv3b

using namespace fv3b;

// fields (38): u, v, w, delp, pt, uc, vc, cx, cy, xfa, yfa, mfx, mfy (3-D);
// dx, dy, dxc, dyc, rdx, rdy, rdxa, rdya, area, rarea, rarea_c, f0, del6_u,
// del6_v (2-D); u_out, v_out, w_out, delp_out, pt_out, cx_out, cy_out,
// xfa_out, yfa_out, mfx_out, mfy_out (3-D).  The accumulator outputs may
// alias their inputs (pointwise update); the others must not.  scalars:
// ppm_p1, ppm_p2, dt, dddmp, d2_bg, da_min, damp4, damp4h, dampv (the del6
// coefficients of templates.D_CONSTS), and optionally acc_reset: nonzero
// reads the accumulator inputs as 0.0 (the first substep of a timestep,
// where the step zeroes them: 0.0 + x is the same sum, so the zero fill is
// skipped).  An optional 39th field receives a copy of the input delp (the
// timestep's dp1, saved by the first substep instead of a separate copy).
extern "C" int fv3b_d_sw(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || (nf != 38 && nf != 39) || (ns != 9 && ns != 10))
    return fail(FV3B_EINVAL, "fv3b_d_sw: expects 38 or 39 fields, 9 or 10 scalars (got %d, %d)", nf, ns);
  DswArgs a;
  const Halo h0 = {0, 0, 0, 0, 0, 0}, h3 = {3, 3, 3, 3, 0, 0};
  const Halo hu = {3, 3, 3, 4, 0, 0}, hv = {3, 4, 3, 3, 0, 0}, huc = {0, 1, 3, 3, 0, 0}, hvc = {3, 3, 0, 1, 0, 0};
  View* in3[13] = {&a.u, &a.v, &a.w, &a.delp, &a.pt, &a.uc, &a.vc, &a.cx, &a.cy, &a.xfa, &a.yfa, &a.mfx, &a.mfy};
  const Halo hin[13] = {hu, hv, h3, h3, h3, huc, hvc, h0, h0, h0, h0, h0, h0};
  const char* nin[13] = {"u", "v", "w", "delp", "pt", "uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy"};
  for (int t = 0; t < 13; ++t) FV3B_TRY(view_of(f[t], 3, *d, hin[t], nin[t], in3[t]));
  constexpr int NM = 14, O = 13 + NM;
  View* m[NM] = {&a.dx, &a.dy, &a.dxc, &a.dyc, &a.rdx, &a.rdy, &a.rdxa, &a.rdya, &a.area, &a.rarea, &a.rarea_c, &a.f0,
                 &a.del6_u, &a.del6_v};
  const char* nm[NM] = {"dx", "dy", "dxc", "dyc", "rdx", "rdy", "rdxa", "rdya", "area", "rarea", "rarea_c", "f0",
                        "del6_u", "del6_v"};
  const Halo hm[NM] = {{3, 3, 3, 4, 0, 0}, {3, 4, 3, 3, 0, 0}, {0, 1, 1, 1, 0, 0}, {1, 1, 0, 1, 0, 0},
                       {1, 1, 0, 1, 0, 0}, {0, 1, 1, 1, 0, 0}, {1, 1, 3, 3, 0, 0}, {3, 3, 1, 1, 0, 0},
                       h3, h3, {0, 1, 0, 1, 0, 0}, h3, {2, 2, 2, 3, 0, 0}, {2, 3, 2, 2, 0, 0}};
  for (int t = 0; t < NM; ++t) FV3B_TRY(view_of(f[13 + t], 2, *d, hm[t], nm[t], m[t]));
  View* out[11] = {&a.uo, &a.vo, &a.wo, &a.delpo, &a.pto, &a.cxo, &a.cyo, &a.xfao, &a.yfao, &a.mfxo, &a.mfyo};
  for (int t = 0; t < 11; ++t) FV3B_TRY(view_of(f[O + t], 3, *d, h0, "d_sw output", out[t]));
  for (int t = 0; t < 5; ++t)
    if (f[O + t].data == f[t].data) return fail(FV3B_EINVAL, "fv3b_d_sw: output %d aliases its input", t);
  View v3[24];
  for (int t = 0; t < 13; ++t) v3[t] = *in3[t];
  for (int t = 0; t < 11; ++t) v3[13 + t] = *out[t];
  FV3B_TRY(same_strides(v3, 24, "fv3b_d_sw"));
  for (int t = 0; t < NM; ++t)
    if (m[t]->sj != a.u.sj) return fail(FV3B_ELAYOUT, "fv3b_d_sw: metric %s J stride differs", nm[t]);
  a.hx = f[0].halo_lo[0];
  a.hy = f[0].halo_lo[1];
  const int hi_x = f[0].shape[0] - f[0].halo_lo[0] - d->ni, hi_y = f[0].shape[1] - f[0].halo_lo[1] - d->nj;
  a.hx = a.hx < hi_x ? a.hx : hi_x;
  a.hy = a.hy < hi_y ? a.hy : hi_y;
  if (a.hx < 4 || a.hy < 4) return fail(FV3B_ELAYOUT, "fv3b_d_sw: needs a 4-cell allocated halo");
  a.ni = d->ni; a.nj = d->nj; a.nk = d->nk;
  a.p1 = s[0]; a.p2 = s[1]; a.dt = s[2]; a.dddmp = s[3]; a.d2_bg = s[4]; a.da_min = s[5];
  a.damp4 = s[6]; a.damp4h = s[7]; a.dampv = s[8];
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // transport group (delp, pt, w, accumulators): TMA-pipelined level march
  {
    Geo g;
    FV3B_TRY(geo_of(f[0], &g));
    const int tma_fields[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23, 24,
                              25, 26};
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
    const fv3b_field mt[4] = {f[21], f[22], f[25], f[26]};             // area, rarea, del6_u, del6_v
    FV3B_TRY(dsw_transport_maps(t, g, qb, ac, mt));
    t.delpo = a.delpo.o;
    t.pto = a.pto.o;
    t.wo = a.wo.o;
    View* ao[6] = {&a.cxo, &a.cyo, &a.xfao, &a.yfao, &a.mfxo, &a.mfyo};
    View* ai[6] = {&a.cx, &a.cy, &a.xfa, &a.yfa, &a.mfx, &a.mfy};
    for (int u = 0; u < 6; ++u) {
      t.acco[u] = ao[u]->o;
      t.acci[u] = ai[u]->o;
    }
    t.dx = a.dx.o;
    t.dy = a.dy.o;
    t.rdxa = a.rdxa.o;
    t.rdya = a.rdya.o;
    t.sj = a.u.sj;
    t.sk = a.u.sk;
    t.i0 = g.i0;
    t.j0 = g.j0;
    t.mlo = -(g.i0 + g.j0 * t.sj);
    t.mhi = g.rows * t.sj + t.mlo - 1;
    t.ni = d->ni; t.nj = d->nj; t.nk = d->nk;
    t.p1 = a.p1; t.p2 = a.p2; t.dt = a.dt; t.damp4 = a.damp4; t.damp4h = a.damp4h;
    t.acc_reset = ns == 10 && s[9] != 0.0;
    t.dp1o = nullptr;
    if (nf == 39) {
      View v;
      FV3B_TRY(view_of(f[38], 3, *d, h0, "dp1_out", &v));
      if (v.sj != a.u.sj || v.sk != a.u.sk) return fail(FV3B_ELAYOUT, "fv3b_d_sw: dp1_out strides differ");
      if (f[38].data == f[3].data) return fail(FV3B_EINVAL, "fv3b_d_sw: dp1_out aliases delp");
      t.dp1o = v.o;
    }
    FV3B_TRY(launch_dsw_transport(t, st));
  }
  // momentum group (u, v): TMA-pipelined level march
  DswMoArgs mo;
  memset(&mo, 0, sizeof mo);
  {
    Geo g;
    FV3B_TRY(geo_of(f[0], &g));
    const fv3b_field mt[12] = {f[13], f[14], f[19], f[20], f[21], f[24], f[22], f[17], f[18], f[15], f[16], f[23]};
    FV3B_TRY(dsw_momentum_maps(mo, g, f[0], f[1], f[5], f[6], mt));
    mo.i0 = g.i0;
    mo.j0 = g.j0;
    mo.mlo = -(g.i0 + g.j0 * a.u.sj);
    mo.mhi = g.rows * a.u.sj + mo.mlo - 1;
  }
  mo.uo = a.uo.o;
  mo.vo = a.vo.o;
  mo.del6_u = a.del6_u.o;
  mo.del6_v = a.del6_v.o;
  mo.sj = a.u.sj;
  mo.sk = a.u.sk;
  mo.ni = d->ni; mo.nj = d->nj; mo.nk = d->nk;
  mo.p1 = a.p1; mo.p2 = a.p2; mo.dt = a.dt; mo.dddmp = a.dddmp; mo.d2_bg = a.d2_bg; mo.da_min = a.da_min;
  mo.dampv = a.dampv;
  return launch_dsw_momentum(mo, st);
}
