// Shared-memory tile toolkit for the fused horizontal kernels (c_sw, d_sw,
// p_grad).  A CTA owns a TI x TJ tile of one level; each temporary of the
// .stn source lives in a shared-memory array with the common halo'd
// geometry [-HX, TI+HX) x [-HY, TJ+HY) and is computed over exactly the
// rectangle the later statements read (the reference's extension,
// extents.py:128-164, restricted to the tile).  One fill() per statement
// group, a barrier between dependent groups.
#pragma once

#include "common.cuh"
#include "ppm.cuh"

namespace fv3b {

template <int TI_, int TJ_, int HX_, int HY_>
struct TileGeo {
  static constexpr int TI = TI_, TJ = TJ_, HX = HX_, HY = HY_;
  // row width = 2 (mod 4) doubles: row-segment threads of a warp hit
  // distinct bank pairs
  static constexpr int W0 = TI + 2 * HX;
  static constexpr int W = W0 + ((2 - W0 % 4) + 4) % 4;
  static constexpr int H = TJ + 2 * HY;
  static constexpr int N = W * H;
  // allocation stride per array: 4 slack rows so partial 4-wide PPM
  // segments near the tile edge may read (never store) past the last row
  static constexpr int NA = (N + 4 * W + 8 + 15) / 16 * 16;
};

// A tile array: element (i, j) in tile-local coordinates.
template <class G>
struct Arr {
  double* p;
  __device__ __forceinline__ double& operator()(int i, int j) const { return p[(j + G::HY) * G::W + (i + G::HX)]; }
  __device__ __forceinline__ double* at(int i, int j) const { return p + (j + G::HY) * G::W + (i + G::HX); }
};

// a(i, j) = f(i, j) over [ia, ib) x [ja, jb)
template <class G, class F>
__device__ __forceinline__ void fill(const Arr<G>& a, int ia, int ib, int ja, int jb, F f) {
  const int w = ib - ia, n = w * (jb - ja);
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int i = ia + e % w, j = ja + e / w;
    a(i, j) = f(i, j);
  }
}

// for each (i, j) in the rectangle: f(i, j)  (no store)
template <class F>
__device__ __forceinline__ void each(int ia, int ib, int ja, int jb, F f) {
  const int w = ib - ia, n = w * (jb - ja);
  for (int e = threadIdx.x; e < n; e += blockDim.x) f(ia + e % w, ja + e / w);
}

// Load a rectangle of a field at level k; cells outside the allocated
// range [-hlo, n+hhi) are zero (never consumed by an in-domain output).
template <class G>
__device__ __forceinline__ void load(const Arr<G>& a, const View& v, int gi0, int gj0, int k, int ia, int ib, int ja,
                                     int jb, int ni, int nj, int hx, int hy) {
  fill(a, ia, ib, ja, jb, [&](int i, int j) {
    const int gi = gi0 + i, gj = gj0 + j;
    return (gi >= -hx && gi < ni + hx && gj >= -hy && gj < nj + hy) ? __ldg(v.ptr(gi, gj, k)) : 0.0;
  });
}

// PPM faces along x over faces [ia, ib) of rows [ja, jb): out(i, j) from
// q(i-3 .. i+2, j) and Courant c(i, j).  Work item = 4 faces of one row.
template <class G>
__device__ __forceinline__ void ppm_x(const Arr<G>& out, const Arr<G>& q, const Arr<G>& c, int ia, int ib, int ja,
                                      int jb, double p1, double p2) {
  constexpr int S = 4;
  const int nseg = (ib - ia + S - 1) / S, nrow = jb - ja, n = nseg * nrow;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int j = ja + e % nrow, i = ia + (e / nrow) * S;
    double f[S];
    ppm_line<S>(q.at(i, j), 1, c.at(i, j), 1, p1, p2, f);
#pragma unroll
    for (int u = 0; u < S; ++u)
      if (i + u < ib) out(i + u, j) = f[u];
  }
}

// PPM faces along y over faces [ja, jb) of columns [ia, ib).
template <class G>
__device__ __forceinline__ void ppm_y(const Arr<G>& out, const Arr<G>& q, const Arr<G>& c, int ia, int ib, int ja,
                                      int jb, double p1, double p2) {
  constexpr int S = 4;
  const int nseg = (jb - ja + S - 1) / S, ncol = ib - ia, n = nseg * ncol;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int i = ia + e % ncol, j = ja + (e / ncol) * S;
    double f[S];
    ppm_line<S>(q.at(i, j), G::W, c.at(i, j), G::W, p1, p2, f);
#pragma unroll
    for (int u = 0; u < S; ++u)
      if (j + u < jb) out(i, j + u) = f[u];
  }
}

// 2-D metric at (i, j) of the tile (read-only path; reused across levels).
__device__ __forceinline__ double met(const View& v, int gi, int gj) { return __ldg(v.ptr(gi, gj, 0)); }

}  // namespace fv3b
