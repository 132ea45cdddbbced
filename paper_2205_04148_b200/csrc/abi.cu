// ABI plumbing: version, thread-local error text, argument validation.
#include <string>

#include "common.cuh"

namespace fv3b {

static thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int view_of(const fv3b_field& f, int rank, const fv3b_domain& d, const Halo& need, const char* name, View* out) {
  if (f.data == nullptr) return fail(FV3B_EINVAL, "%s: null data pointer", name);
  if (f.rank != rank) return fail(FV3B_ELAYOUT, "%s: rank %d, expected %d", name, f.rank, rank);
  const int n[3] = {d.ni, d.nj, d.nk};
  const int lo[3] = {need.ilo, need.jlo, need.klo};
  const int hi[3] = {need.ihi, need.jhi, need.khi};
  int axes[3];
  int na = 0;
  if (rank == 3) { axes[0] = 0; axes[1] = 1; axes[2] = 2; na = 3; }
  else if (rank == 2) { axes[0] = 0; axes[1] = 1; na = 2; }
  else { axes[0] = 2; na = 1; }
  if (rank >= 2 && f.stride[0] != 1) return fail(FV3B_ELAYOUT, "%s: I must be unit stride (got %lld)", name, (long long)f.stride[0]);
  int64_t off = 0;
  for (int p = 0; p < na; ++p) {
    const int a = axes[p];
    const int have_hi = f.shape[p] - f.halo_lo[p] - n[a];
    if (f.halo_lo[p] < lo[a] || have_hi < hi[a])
      return fail(FV3B_ELAYOUT, "%s: axis %c halo (%d,%d) smaller than required (%d,%d)", name, "IJK"[a],
                  f.halo_lo[p], have_hi, lo[a], hi[a]);
    off += (int64_t)f.halo_lo[p] * f.stride[p];
  }
  out->o = f.data + off;
  if (rank == 3) { out->sj = f.stride[1]; out->sk = f.stride[2]; }
  else if (rank == 2) { out->sj = f.stride[1]; out->sk = 0; }
  else { out->sj = 0; out->sk = f.stride[0]; }
  return FV3B_OK;
}

int same_strides(const View* v, int n, const char* what) {
  for (int i = 1; i < n; ++i)
    if (v[i].sj != v[0].sj || (v[i].sk != v[0].sk && v[i].sk != 0 && v[0].sk != 0))
      return fail(FV3B_ELAYOUT, "%s: field %d strides (%lld,%lld) differ from field 0 (%lld,%lld)", what, i,
                  (long long)v[i].sj, (long long)v[i].sk, (long long)v[0].sj, (long long)v[0].sk);
  return FV3B_OK;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FV3B_ELAUNCH, "%s: %s", what, cudaGetErrorString(e));
  return FV3B_OK;
}

}  // namespace fv3b

extern "C" int fv3b_abi_version(void) { return FV3B_ABI_VERSION; }

extern "C" const char* fv3b_last_error(void) { return fv3b::g_err.c_str(); }
