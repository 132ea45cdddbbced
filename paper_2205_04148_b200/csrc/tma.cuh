// TMA (cp.async.bulk.tensor) + mbarrier helpers for the tiled stencil
// kernels.  Tiles of a level are fetched as 3-D boxes (I, J, 1) of the
// device Layout; out-of-bounds box elements are zero-filled by the TMA unit.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace fv3b {

// Host: tensor map of a field tensor (pitch, rows, levels) with a (bw, bh, 1)
// box.  Cached by (pointer, geometry, box); returns FV3B_OK or an error.
int tensor_map(const double* base, int64_t pitch, int64_t rows, int64_t levels, int bw, int bh, CUtensorMap* out);

// Field geometry shared by a launch, in elements.
struct Geo {
  int64_t pitch, rows, levels;  // allocated extents of a 3-D field
  int i0, j0;                   // allocated column / row of interior (0, 0)
};

// Geometry of a validated 3-D fv3b_field (I unit stride, strides == extents).
int geo_of(const fv3b_field& f, Geo* g);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// Box load of (x, y, z) (allocated-element coordinates) into smem.  The box's
// first element must be 16-B aligned in global memory: for fp64 fields x is
// even (measured on B200: an odd x raises an illegal-instruction fault).
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Order generic-proxy smem reads of a buffer before the async proxy
// overwrites it with the next TMA load.
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace fv3b
