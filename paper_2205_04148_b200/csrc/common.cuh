// Shared helpers for the fv3b kernels: ABI argument checking, error state,
// device views.  See include/fv3b.h for the ABI contract.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdint.h>

#include "../../include/fv3b.h"

namespace fv3b {

// Sets the thread-local error text and returns `code`.
int fail(int code, const char* fmt, ...);

// Device-side view of a field: interior-origin pointer + J/K strides
// (I is unit stride).  For 2-D (I,J) fields sk == 0.
struct View {
  double* o;
  int64_t sj, sk;
  __device__ __forceinline__ double& operator()(int i, int j, int k) const { return o[i + j * sj + k * sk]; }
  __device__ __forceinline__ double* ptr(int i, int j, int k) const { return o + i + j * sj + k * sk; }
};

struct Halo {
  int ilo, ihi, jlo, jhi, klo, khi;  // allocated halo widths
};

// Validate one field and produce its view.  `rank` 3 = IJK, 2 = IJ, 1 = K.
// Checks unit I stride, non-null data and that the allocation covers
// `need` (lo/hi halo widths per axis) around the domain.
int view_of(const fv3b_field& f, int rank, const fv3b_domain& d, const Halo& need, const char* name, View* out);

// All 3-D views must share strides (one tile geometry per launch).
int same_strides(const View* v, int n, const char* what);

int check_launch(const char* what);

inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// SM count of the current device (cached per device).
int num_sms();

// Launch-configuration knob (fv3b_tune_set); 0 = automatic.
int tune_get(int knob);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `fn` once per
// (kernel, device): the attribute is per device context, so a process that
// launches on several GPUs sets it on each.
int ensure_smem(const void* fn, size_t bytes, const char* what);

// Levels per CTA of a level-marching tile kernel: a single wave when the
// tiles fit the resident CTA slots (every CTA gets an equal chunk of levels,
// no tail wave), otherwise one whole column of levels per CTA.  `knob` (and
// FV3B_TUNE_KCHUNK) override the choice.
inline int level_chunk(int knob, int tiles, int nk, int ctas_per_sm) {
  if (nk <= 0 || tiles <= 0) return 1;
  int forced = tune_get(knob);
  if (forced <= 0) forced = tune_get(FV3B_TUNE_KCHUNK);
  if (forced > 0) return forced < nk ? forced : nk;
  const int slots = num_sms() * ctas_per_sm;
  int per_tile = tiles >= slots ? 1 : slots / tiles;
  if (per_tile > nk) per_tile = nk;
  return cdiv(nk, per_tile);
}

// Global loads with an L1 policy: streaming operands read once per level
// (no_allocate: they do not evict the tile's 2-D metrics) and the 2-D
// metrics every level re-reads (evict_last).  The asm is a pure expression
// to the compiler, which may evaluate it outside the guard of its call site:
// callers pass addresses that are valid whether or not the value is used.
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Tile-local shared-memory array covering [i0, i1) x [j0, j1) (tile coords).
struct STile {
  double* p;
  int i0, j0, w;
  __device__ __forceinline__ double& operator()(int i, int j) const { return p[(j - j0) * w + (i - i0)]; }
};

}  // namespace fv3b

#define FV3B_TRY(expr)        \
  do {                        \
    int _rc = (expr);         \
    if (_rc != FV3B_OK) return _rc; \
  } while (0)
