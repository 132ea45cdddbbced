// K0: copy stencil `out = inp` (programs/copy.stn).
// The bandwidth ceiling of the stencil path: 16 B per interior cell.
// Rows are 64-B aligned at the interior origin (Layout pre_pad,
// scheduling.py:377-407), so an even-width row moves as 16-B vectors.
#include "common.cuh"

namespace fv3b {

// One CTA iteration handles `ROWS_PER_ITER` rows of the interior; each lane
// moves 16-B vectors.  Grid-stride over rows keeps the grid at a multiple
// of the SM count.
__global__ void __launch_bounds__(256) copy_vec2_kernel(View in, View out, int ni, int nj, int nk) {
  const int nv = ni >> 1;  // 16-B vectors per row
  const long long nrows = (long long)nj * nk;
  const long long total = nrows * nv;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // 4 independent vectors in flight per thread per iteration
  for (; t + 3 * stride < total; t += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long e = t + u * stride;
      const long long row = e / nv;
      const int c = (int)(e - row * nv);
      const int j = (int)(row % nj), k = (int)(row / nj);
      v[u] = __ldcs(reinterpret_cast<const double2*>(in.ptr(2 * c, j, k)));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long e = t + u * stride;
      const long long row = e / nv;
      const int c = (int)(e - row * nv);
      const int j = (int)(row % nj), k = (int)(row / nj);
      __stcs(reinterpret_cast<double2*>(out.ptr(2 * c, j, k)), v[u]);
    }
  }
  for (; t < total; t += stride) {
    const long long row = t / nv;
    const int c = (int)(t - row * nv);
    const int j = (int)(row % nj), k = (int)(row / nj);
    __stcs(reinterpret_cast<double2*>(out.ptr(2 * c, j, k)), __ldcs(reinterpret_cast<const double2*>(in.ptr(2 * c, j, k))));
  }
}

// Dense fast path (halo-free fields with pitch == ni: the copy is one flat
// vector): 16-B streaming loads / stores, 64 CTAs of 256 threads per SM.
// Swept on B200 (tools/bw_probe.py, profiles/r2_copy_bandwidth.txt): one
// vector per thread per iteration at 64 CTAs / SM reaches 0.945-0.976 of the
// measured HBM copy peak; deeper unrolling with fewer CTAs reaches 0.84-0.95.
__global__ void __launch_bounds__(256) copy_flat_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                        long long n) {
#ifndef FV3B_COPY_U
#define FV3B_COPY_U 1
#endif
  constexpr int U = FV3B_COPY_U;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; t + (U - 1) * stride < n; t += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(in + t + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + t + u * stride, v[u]);
  }
  for (; t < n; t += stride) __stcs(out + t, __ldcs(in + t));
}

__global__ void __launch_bounds__(256) copy_scalar_kernel(View in, View out, int ni, int nj, int nk) {
  const long long total = (long long)ni * nj * nk;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % ni);
    const long long r = t / ni;
    const int j = (int)(r % nj), k = (int)(r / nj);
    out(i, j, k) = in(i, j, k);
  }
}


}  // namespace fv3b

using namespace fv3b;

extern "C" int fv3b_copy(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream) {
  (void)s;
  if (f == nullptr || d == nullptr || nf != 2 || ns != 0) return fail(FV3B_EINVAL, "fv3b_copy: expects 2 fields, 0 scalars");
  const Halo h0 = {0, 0, 0, 0, 0, 0};
  View in, out;
  FV3B_TRY(view_of(f[0], 3, *d, h0, "copy.inp", &in));
  FV3B_TRY(view_of(f[1], 3, *d, h0, "copy.out", &out));
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = (d->ni % 2 == 0) && ((uintptr_t)in.o % 16 == 0) && ((uintptr_t)out.o % 16 == 0) &&
                   (in.sj % 2 == 0) && (in.sk % 2 == 0) && (out.sj % 2 == 0) && (out.sk % 2 == 0);
#ifndef FV3B_COPY_G
#define FV3B_COPY_G 64
#endif
  const int grid = num_sms() * FV3B_COPY_G;
  const bool flat = vec && in.sj == d->ni && out.sj == d->ni && in.sk == (int64_t)d->ni * d->nj &&
                    out.sk == (int64_t)d->ni * d->nj;
  if (flat)
    copy_flat_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(in.o), reinterpret_cast<double2*>(out.o),
                                           (long long)d->ni * d->nj * d->nk / 2);
  else if (vec)
    copy_vec2_kernel<<<grid, 256, 0, st>>>(in, out, d->ni, d->nj, d->nk);
  else
    copy_scalar_kernel<<<grid, 256, 0, st>>>(in, out, d->ni, d->nj, d->nk);
  return check_launch("fv3b_copy");
}

// ---------------------------------------------------------------------------
// Reference array convention (I, J, K with K unit stride: the numpy C-order
// arrays of the reference's run_reference / fieldio) <-> the I-unit-stride
// Layout.  Per J row a 32 x 32 (I, K) tile goes through shared memory, so
// loads run along the source's unit axis and stores along the destination's:
// both sides coalesced (the host<->device state path of Dycore.step_host).
namespace fv3b {

template <bool K2I>  // true: source K-unit -> destination I-unit
__global__ void __launch_bounds__(256) transpose_ik_kernel(const double* __restrict__ src, int64_t s0, int64_t s1,
                                                           int64_t s2, double* __restrict__ dst, int64_t d0,
                                                           int64_t d1, int64_t d2, int ni, int nk) {
  __shared__ double t[32][33];
  const int64_t j = blockIdx.z;
  const int ib = blockIdx.y * 32, kb = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int i = K2I ? ib + r : ib + tx, k = K2I ? kb + tx : kb + r;
    if (i < ni && k < nk) t[r][tx] = __ldcs(src + i * s0 + j * s1 + k * s2);
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int i = K2I ? ib + tx : ib + r, k = K2I ? kb + r : kb + tx;
    if (i < ni && k < nk) __stcs(dst + i * d0 + j * d1 + k * d2, t[tx][r]);
  }
}

}  // namespace fv3b

extern "C" int fv3b_transpose(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                              void* stream) {
  (void)s;
  (void)ns;
  if (f == nullptr || d == nullptr || nf != 2)
    return fv3b::fail(FV3B_EINVAL, "fv3b_transpose: expects 2 fields (src, dst)");
  const fv3b_field &a = f[0], &b = f[1];
  if (a.data == nullptr || b.data == nullptr || a.rank != 3 || b.rank != 3)
    return fv3b::fail(FV3B_EINVAL, "fv3b_transpose: src and dst must be 3-D fields");
  const bool k2i = a.stride[2] == 1 && b.stride[0] == 1, i2k = a.stride[0] == 1 && b.stride[2] == 1;
  if (!k2i && !i2k)
    return fv3b::fail(FV3B_ELAYOUT, "fv3b_transpose: one field must be K-unit-stride, the other I-unit-stride");
  for (int x = 0; x < 3; ++x) {
    const int n = x == 0 ? d->ni : (x == 1 ? d->nj : d->nk);
    if (n > a.shape[x] || n > b.shape[x])
      return fv3b::fail(FV3B_EDOMAIN, "fv3b_transpose: region axis %d (%d) exceeds a field's shape", x, n);
  }
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  dim3 grid(fv3b::cdiv(d->nk, 32), fv3b::cdiv(d->ni, 32), d->nj), block(32, 8);
  auto st = (cudaStream_t)stream;
  if (k2i)
    fv3b::transpose_ik_kernel<true><<<grid, block, 0, st>>>(a.data, a.stride[0], a.stride[1], a.stride[2], b.data,
                                                            b.stride[0], b.stride[1], b.stride[2], d->ni, d->nk);
  else
    fv3b::transpose_ik_kernel<false><<<grid, block, 0, st>>>(a.data, a.stride[0], a.stride[1], a.stride[2], b.data,
                                                             b.stride[0], b.stride[1], b.stride[2], d->ni, d->nk);
  return fv3b::check_launch("fv3b_transpose");
}

// ---------------------------------------------------------------------------
// Layer thickness at the D-grid wind points for the vertical remapping of u
// and v: u(i, j) sits between cells (i, j-1) and (i, j), v(i, j) between
// (i-1, j) and (i, j) (p_grad_d.stn), so
//   du = 0.5 * (delp[0,-1,0] + delp),  dv = 0.5 * (delp[-1,0,0] + delp)
// over the interior (oracle/remap_map.py face_thickness).
namespace fv3b {
__global__ void __launch_bounds__(256) face_thickness_kernel(View dp, View du, View dv, int ni, int nj) {
  const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y, k = blockIdx.z;
  if (i >= ni || j >= nj) return;
  const double c = __ldg(dp.ptr(i, j, k));
  *du.ptr(i, j, k) = 0.5 * (__ldg(dp.ptr(i, j - 1, k)) + c);
  *dv.ptr(i, j, k) = 0.5 * (__ldg(dp.ptr(i - 1, j, k)) + c);
}
}  // namespace fv3b

extern "C" int fv3b_face_thickness(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                   void* stream) {
  (void)s;
  if (f == nullptr || d == nullptr || nf != 3 || ns != 0)
    return fv3b::fail(FV3B_EINVAL, "fv3b_face_thickness: expects 3 fields (delp, du, dv), 0 scalars");
  fv3b::View dp, du, dv;
  const fv3b::Halo h1 = {1, 0, 1, 0, 0, 0}, h0 = {0, 0, 0, 0, 0, 0};
  FV3B_TRY(fv3b::view_of(f[0], 3, *d, h1, "delp", &dp));
  FV3B_TRY(fv3b::view_of(f[1], 3, *d, h0, "du", &du));
  FV3B_TRY(fv3b::view_of(f[2], 3, *d, h0, "dv", &dv));
  if (f[1].data == f[0].data || f[2].data == f[0].data || f[1].data == f[2].data)
    return fv3b::fail(FV3B_EINVAL, "fv3b_face_thickness: outputs alias");
  if (d->ni <= 0 || d->nj <= 0 || d->nk <= 0) return FV3B_OK;
  dim3 grid(fv3b::cdiv(d->ni, 32), fv3b::cdiv(d->nj, 8), d->nk);
  fv3b::face_thickness_kernel<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(dp, du, dv, d->ni, d->nj);
  return fv3b::check_launch("fv3b_face_thickness");
}

// Host-I/O helper: one strided copy of `height` rows of `width` bytes
// (pitches in bytes) between pinned host and device memory, on `stream`
// (cudaMemcpy2DAsync, direction from the unified address space).  Measured
// for moving only the interior columns of the host state (tools/io_variants.py):
// 8% fewer bytes but no faster than whole arrays with both directions busy.
extern "C" int fv3b_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                             int64_t height, void* stream) {
  if (dst == nullptr || src == nullptr || width < 0 || height < 0 || dpitch < width || spitch < width)
    return fv3b::fail(FV3B_EINVAL, "fv3b_memcpy2d: bad arguments");
  if (width == 0 || height == 0) return FV3B_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                                          cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return fv3b::fail(FV3B_ELAUNCH, "fv3b_memcpy2d: %s", cudaGetErrorString(e));
  return FV3B_OK;
}

// Multi-GPU helper of parallel.IpcPeers: let kernels on the current device
// load / store the memory of `peer` (NVLink P2P).  Already enabled is fine.
extern "C" int fv3b_enable_peer_access(int peer) {
  int dev = -1, ok = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fv3b::fail(FV3B_ELAUNCH, "fv3b_enable_peer_access: no device");
  if (peer == dev) return FV3B_OK;
  if (cudaDeviceCanAccessPeer(&ok, dev, peer) != cudaSuccess || !ok)
    return fv3b::fail(FV3B_ELAUNCH, "fv3b_enable_peer_access: device %d cannot access device %d", dev, peer);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // (not sticky: clear it)
    return FV3B_OK;
  }
  if (e != cudaSuccess) return fv3b::fail(FV3B_ELAUNCH, "fv3b_enable_peer_access: %s", cudaGetErrorString(e));
  return FV3B_OK;
}
