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

// ---------------------------------------------------------------------------
// Launch-configuration knobs, SM count, per-device shared-memory attributes.
// ---------------------------------------------------------------------------
#include <atomic>
#include <map>
#include <mutex>
#include <utility>

namespace fv3b {

static std::atomic<int> g_tune[FV3B_TUNE_COUNT];

int tune_get(int knob) { return (knob >= 0 && knob < FV3B_TUNE_COUNT) ? g_tune[knob].load() : 0; }

int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load();
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n);
  }
  return n;
}

int ensure_smem(const void* fn, size_t bytes, const char* what) {
  // the largest size set so far per (kernel, device): a kernel whose dynamic
  // shared memory depends on the call (the column solvers: levels) raises it
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({fn, dev});
  if (it != done.end() && it->second >= bytes) return FV3B_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess ||
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
    return check_launch(what);
  done[{fn, dev}] = bytes;
  return FV3B_OK;
}

}  // namespace fv3b

extern "C" int fv3b_abi_version(void) { return FV3B_ABI_VERSION; }

extern "C" int fv3b_tune_set(int knob, int value) {
  if (knob < 0 || knob >= FV3B_TUNE_COUNT || value < 0)
    return fv3b::fail(FV3B_EINVAL, "fv3b_tune_set: unknown knob %d or negative value %d", knob, value);
  fv3b::g_tune[knob].store(value);
  return FV3B_OK;
}

extern "C" int fv3b_tune_get(int knob) {
  return (knob >= 0 && knob < FV3B_TUNE_COUNT) ? fv3b::g_tune[knob].load() : -1;
}

extern "C" const char* fv3b_last_error(void) { return fv3b::g_err.c_str(); }

// ---------------------------------------------------------------------------
// TMA tensor maps (driver entry point fetched through the runtime, so the
// library does not link libcuda directly).  Cached by geometry + pointer.
// ---------------------------------------------------------------------------
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>

#include "tma.cuh"

namespace fv3b {

int tensor_map(const double* base, int64_t pitch, int64_t rows, int64_t levels, int bw, int bh, CUtensorMap* out) {
  using Key = std::tuple<const void*, int64_t, int64_t, int64_t, int, int>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  const Key key{base, pitch, rows, levels, bw, bh};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return FV3B_OK;
  }
  if (encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      return fail(FV3B_ELAUNCH, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (((uintptr_t)base) % 16 != 0 || (pitch * 8) % 16 != 0)
    return fail(FV3B_ELAYOUT, "TMA needs 16-B aligned base and row pitch (pitch=%lld)", (long long)pitch);
  cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)rows, (cuuint64_t)levels};
  cuuint64_t strides[2] = {(cuuint64_t)(pitch * 8), (cuuint64_t)(pitch * rows * 8)};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FV3B_ELAYOUT, "cuTensorMapEncodeTiled failed (%d) box %dx%d", (int)r, bw, bh);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return FV3B_OK;
}

int geo_of(const fv3b_field& f, Geo* g) {
  if (f.rank == 3) {
    if (f.stride[0] != 1 || f.stride[2] != f.stride[1] * f.shape[1] || f.stride[1] != f.shape[0])
      return fail(FV3B_ELAYOUT, "TMA path needs a dense (pitch, rows, levels) field layout");
    g->pitch = f.stride[1];
    g->rows = f.shape[1];
    g->levels = f.shape[2];
  } else if (f.rank == 2) {
    if (f.stride[0] != 1 || f.stride[1] != f.shape[0]) return fail(FV3B_ELAYOUT, "TMA path needs dense 2-D fields");
    g->pitch = f.stride[1];
    g->rows = f.shape[1];
    g->levels = 1;
  } else {
    return fail(FV3B_ELAYOUT, "TMA path needs 2-D or 3-D fields");
  }
  g->i0 = f.halo_lo[0];
  g->j0 = f.halo_lo[1];
  return FV3B_OK;
}

}  // namespace fv3b

// ---------------------------------------------------------------------------
// Self-test of the branch-free fast paths (fastdiv.cuh) against the exact
// operators (IEEE division, det_log): counts, over n operand pairs, the
// results that differ although the fast path reported them valid (must be
// 0), and the fast-path rejections (operands the kernels re-evaluate with
// the exact operators).
#include "fastdiv.cuh"

namespace fv3b {
__global__ void selftest_fastmath_kernel(const double* x, const double* y, int n, unsigned long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ok = true;
  const double q = div_fast(x[i], y[i], ok);
  const double e = x[i] / y[i];
  if (ok && __double_as_longlong(q) != __double_as_longlong(e)) atomicAdd(&out[0], 1ull);
  if (!ok) atomicAdd(&out[1], 1ull);
  bool ok2 = true;
  const double lg = det_log_fast(fabs(x[i]), ok2);
  const double el = det_log(fabs(x[i]));
  if (ok2 && __double_as_longlong(lg) != __double_as_longlong(el)) atomicAdd(&out[2], 1ull);
  if (!ok2) atomicAdd(&out[3], 1ull);
}
}  // namespace fv3b

extern "C" int fv3b_selftest_fastmath(const double* x, const double* y, int n, unsigned long long* counts,
                                      void* stream) {
  if (x == nullptr || y == nullptr || counts == nullptr || n < 0)
    return fv3b::fail(FV3B_EINVAL, "fv3b_selftest_fastmath: bad arguments");
  if (n == 0) return FV3B_OK;
  fv3b::selftest_fastmath_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(x, y, n, counts);
  return fv3b::check_launch("fv3b_selftest_fastmath");
}
