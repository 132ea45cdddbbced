// c_sw launch interface (c_sw.cu entry points -> csw_tma.cu kernel).
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace fv3b {

struct CswTmaArgs {
  CUtensorMap in[5];   // u, v, delp, pt, w   (box i in [-4, TI+4), j in [-3, TJ+3))
  CUtensorMap met[9];  // dx, dy, dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc (level 0)
  double* uc;          // interior origins of the outputs
  double* vc;
  double* delpc;
  double* ptc;
  double* wc;
  int64_t sj, sk;
  int i0, j0, ni, nj, nk, kchunk;
  bool own_is, own_ie, own_js, own_je;
  double dt2, a1, a2;
};

int csw_maps(CswTmaArgs& a, const Geo& g, const fv3b_field* in5, const fv3b_field* met9);
int launch_csw(const CswTmaArgs& a, bool ext, cudaStream_t st);

}  // namespace fv3b
