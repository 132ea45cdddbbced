// Pressure and heat-capacity diagnostics of the remapped state (the pe / pk
// / moist_cv part of FV3's Lagrangian-to-Eulerian step, SURVEY 8(f) row 1;
// CPU counterpart oracle/thermo.py, bitwise):
//
//   pe[0] = ptop,  pe[k+1] = pe[k] + delp[k]          (interfaces)
//   peln = log(pe),  pk = exp(akap * peln)            (det_log / det_exp)
//   pkz[k] = (pk[k+1] - pk[k]) / (akap * (peln[k+1] - peln[k]))
//   cvm = (1 - (qv + ql + qs)) cv_air + qv cv_vap + ql c_liq + qs c_ice
//         with ql = liquid + rain, qs = ice + snow + graupel
//
// A CTA owns 32 columns.  All eight warps stage delp in shared memory, one
// warp forms the running sum pe there; then all eight warps evaluate the
// levels in parallel (log / exp per interface, pkz and cvm per layer), so the
// per-level transcendental chains overlap across warps instead of running
// down one column thread.
// HBM-bound: delp + the moist tracers in, five fields out.
#include "common.cuh"
#include "detmath.cuh"
#include "fastdiv.cuh"

namespace fv3b {

struct MoistArgs {
  View delp, q[6], pe, peln, pk, pkz, cvm;
  int nw, ni, nj, nk;  // nk layers
  double ptop, akap, cv_air, cv_vap, c_liq, c_ice;
};

constexpr int MK_COLS = 32, MK_TY = 8;

__global__ void __launch_bounds__(MK_COLS * MK_TY) moist_pk_kernel(const MoistArgs a) {
  extern __shared__ double sm[];  // [nk + 1][32]: pe, then peln in place; pk
  const int nk = a.nk, L = nk + 1;
  double* slog = sm;
  double* spk = sm + L * MK_COLS;
  const int c = threadIdx.x, ty = threadIdx.y;
  const int col = blockIdx.x * MK_COLS + c;
  const bool live = col < a.ni * a.nj;
  const int i = live ? col % a.ni : 0, j = live ? col / a.ni : 0;
  // every warp stages delp (independent loads in flight together), then one
  // warp forms the running sum in place (the oracle's order of additions)
  for (int k = ty; k < nk; k += MK_TY) slog[(k + 1) * MK_COLS + c] = live ? __ldg(a.delp.ptr(i, j, k)) : 0.0;
  __syncthreads();
  if (ty == 0) {
    double p = a.ptop;
    slog[c] = p;
    for (int k = 0; k < nk; ++k) {
      p = p + slog[(k + 1) * MK_COLS + c];
      slog[(k + 1) * MK_COLS + c] = p;
    }
  }
  __syncthreads();
  for (int k = ty; k <= nk; k += MK_TY) {
    const double pe = slog[k * MK_COLS + c];
    const double ln = det_log(pe);
    const double pk = det_exp(a.akap * ln);
    slog[k * MK_COLS + c] = ln;
    spk[k * MK_COLS + c] = pk;
    if (live) {
      *a.pe.ptr(i, j, k) = pe;
      *a.peln.ptr(i, j, k) = ln;
      *a.pk.ptr(i, j, k) = pk;
    }
  }
  __syncthreads();
  if (!live) return;
  for (int k = ty; k < nk; k += MK_TY) {
    const double l0 = slog[k * MK_COLS + c], l1 = slog[(k + 1) * MK_COLS + c];
    const double k0 = spk[k * MK_COLS + c], k1 = spk[(k + 1) * MK_COLS + c];
    *a.pkz.ptr(i, j, k) = (k1 - k0) / (a.akap * (l1 - l0));
    double q[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) q[t] = t < a.nw ? __ldg(a.q[t].ptr(i, j, k)) : 0.0;
    const double qv = q[0], ql = q[1] + q[2], qs = q[3] + q[4] + q[5];
    const double qd = ql + qs;
    *a.cvm.ptr(i, j, k) = (1.0 - (qv + qd)) * a.cv_air + qv * a.cv_vap + ql * a.c_liq + qs * a.c_ice;
  }
}

}  // namespace fv3b

// fields: delp, the nw (0..6) moist tracers (vapour, liquid, rain, ice, snow,
// graupel; absent ones count as 0), then pe, peln, pk (interfaces), pkz, cvm
// (layers).  scalars: ptop, akap, cv_air, cv_vap, c_liq, c_ice.  Domain nk =
// interface levels.
extern "C" int fv3b_moist_pk(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                             void* stream) {
  using namespace fv3b;
  if (f == nullptr || d == nullptr || s == nullptr || ns != 6 || nf < 6 || nf > 12)
    return fail(FV3B_EINVAL, "fv3b_moist_pk: expects delp, 0..6 moist tracers, pe, peln, pk, pkz, cvm; 6 scalars");
  if (d->nk < 2 || d->nk > 4096) return fail(FV3B_EDOMAIN, "fv3b_moist_pk: program domain nk=%d outside [2, 4096]", d->nk);
  MoistArgs a;
  a.nw = nf - 6;
  const Halo h0 = {0, 0, 0, 0, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, h0, "delp", &a.delp));
  for (int t = 0; t < a.nw; ++t) FV3B_TRY(view_of(f[1 + t], 3, *d, h0, "moist tracer", &a.q[t]));
  for (int t = a.nw; t < 6; ++t) a.q[t] = a.delp;  // never read
  View* outs[5] = {&a.pe, &a.peln, &a.pk, &a.pkz, &a.cvm};
  for (int u = 0; u < 5; ++u) FV3B_TRY(view_of(f[1 + a.nw + u], 3, *d, h0, "moist_pk output", outs[u]));
  for (int u = 0; u < 5; ++u)
    for (int g = 0; g < nf; ++g)
      if (g != 1 + a.nw + u && f[g].data == f[1 + a.nw + u].data)
        return fail(FV3B_EINVAL, "fv3b_moist_pk: output %d aliases field %d", u, g);
  a.ni = d->ni;
  a.nj = d->nj;
  a.nk = d->nk - 1;
  a.ptop = s[0];
  a.akap = s[1];
  a.cv_air = s[2];
  a.cv_vap = s[3];
  a.c_liq = s[4];
  a.c_ice = s[5];
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  const size_t bytes = (size_t)2 * d->nk * MK_COLS * sizeof(double);
  if (bytes > 48 * 1024 &&
      cudaFuncSetAttribute(moist_pk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return check_launch("moist_pk smem attribute");
  moist_pk_kernel<<<cdiv(d->ni * d->nj, MK_COLS), dim3(MK_COLS, MK_TY), bytes, (cudaStream_t)stream>>>(a);
  return check_launch("fv3b_moist_pk");
}

// ---------------------------------------------------------------------------
// Log-pressure coordinate for remapping pt in log(p) (FV3 fv_mapz with
// kord_tm < 0: pt is profiled and mapped in the log-pressure coordinate):
//   pe1[0] = ak[0] (ptop), pe1[k+1] = pe1[k] + delp[k],  ps = pe1[nk]
//   pe2 = pe1[0] | ak[k] + bk[k] * ps | ps       (the mapping's target)
//   lnpe1 = log(pe1), lnpe2 = log(pe2),  dlnp[k] = lnpe1[k+1] - lnpe1[k]
// with the deterministic det_log; oracle/remap_map.py log_thickness /
// log_edges, bitwise.  dlnp is the thickness remap_profile takes for pt,
// lnpe1 / lnpe2 the interfaces fv3b_remap_map's log group maps between.
// One thread per column; the logs of consecutive levels are independent.
// ---------------------------------------------------------------------------
namespace fv3b {
// FAST: det_log_fast (branch-free, fastdiv.cuh) with a validity flag; a
// column whose flag fails is redone with det_log.  Inputs are never written.
template <bool FAST>
__device__ __forceinline__ bool log_column(const double* d, int64_t sd, double* o, int64_t so, double* x1, int64_t s1,
                                           double* x2, int64_t s2, const double* ak, const double* bk, int64_t skk,
                                           int nk) {
  ColArith<FAST> ar;
  double pe = __ldg(ak), lp = ar.log(pe);
  x1[0] = lp;
  x2[0] = lp;
#pragma unroll 4
  for (int k = 0; k < nk; ++k) {
    pe = pe + __ldg(d + k * sd);
    const double ln = ar.log(pe);
    o[k * so] = ln - lp;
    x1[(k + 1) * s1] = ln;
    lp = ln;
  }
  const double ps = pe;
  x2[nk * s2] = lp;  // log(ps)
#pragma unroll 4
  for (int k = 1; k < nk; ++k) x2[k * s2] = ar.log(__ldg(ak + k * skk) + __ldg(bk + k * skk) * ps);
  return ar.ok;
}

__global__ void __launch_bounds__(128) log_thickness_kernel(View dp, View dl, View l1, View l2, const double* ak,
                                                            const double* bk, int64_t skk, int ni, int nj, int nk) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ni * nj) return;
  const int i = col % ni, j = col / ni;
  const double* d = dp.ptr(i, j, 0);
  double *o = dl.ptr(i, j, 0), *x1 = l1.ptr(i, j, 0), *x2 = l2.ptr(i, j, 0);
  if (!log_column<true>(d, dp.sk, o, dl.sk, x1, l1.sk, x2, l2.sk, ak, bk, skk, nk))
    log_column<false>(d, dp.sk, o, dl.sk, x1, l1.sk, x2, l2.sk, ak, bk, skk, nk);
}
}  // namespace fv3b

// fields: delp (3-D), ak, bk (K, nk+1), dlnp (3-D layers), lnpe1, lnpe2 (3-D
// interfaces) outputs.  No scalars.  Domain nk = layers.
extern "C" int fv3b_log_thickness(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                  void* stream) {
  using namespace fv3b;
  (void)s;
  if (f == nullptr || d == nullptr || nf != 6 || ns != 0)
    return fail(FV3B_EINVAL, "fv3b_log_thickness: expects delp, ak, bk, dlnp, lnpe1, lnpe2; no scalars");
  View dp, ak, bk, dl, l1, l2;
  const Halo h0 = {0, 0, 0, 0, 0, 0};
  fv3b_domain di = *d;
  di.nk = d->nk + 1;  // (interfaces)
  FV3B_TRY(view_of(f[0], 3, *d, h0, "delp", &dp));
  FV3B_TRY(view_of(f[1], 1, di, h0, "ak", &ak));
  FV3B_TRY(view_of(f[2], 1, di, h0, "bk", &bk));
  FV3B_TRY(view_of(f[3], 3, *d, h0, "dlnp", &dl));
  FV3B_TRY(view_of(f[4], 3, di, h0, "lnpe1", &l1));
  FV3B_TRY(view_of(f[5], 3, di, h0, "lnpe2", &l2));
  for (int x = 3; x < 6; ++x)
    for (int y = 0; y < 6; ++y)
      if (x != y && f[x].data == f[y].data) return fail(FV3B_EINVAL, "fv3b_log_thickness: output %d aliases field %d", x, y);
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  const int cols = d->ni * d->nj;
  log_thickness_kernel<<<cdiv(cols, 128), 128, 0, (cudaStream_t)stream>>>(dp, dl, l1, l2, ak.o, bk.o, ak.sk, d->ni,
                                                                          d->nj, d->nk);
  return check_launch("fv3b_log_thickness");
}
