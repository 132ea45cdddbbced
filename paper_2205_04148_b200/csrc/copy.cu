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

__global__ void __launch_bounds__(256) copy_scalar_kernel(View in, View out, int ni, int nj, int nk) {
  const long long total = (long long)ni * nj * nk;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % ni);
    const long long r = t / ni;
    const int j = (int)(r % nj), k = (int)(r / nj);
    out(i, j, k) = in(i, j, k);
  }
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
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
  const int grid = num_sms() * 8;
  if (vec)
    copy_vec2_kernel<<<grid, 256, 0, st>>>(in, out, d->ni, d->nj, d->nk);
  else
    copy_scalar_kernel<<<grid, 256, 0, st>>>(in, out, d->ni, d->nj, d->nk);
  return check_launch("fv3b_copy");
}
