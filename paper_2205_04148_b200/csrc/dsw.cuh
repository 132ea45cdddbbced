// d_sw launch interfaces (d_sw.cu entry point -> dsw_transport.cu kernel).
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace fv3b {

struct DswTpArgs {
  CUtensorMap qbox[5];  // delp, pt, w, uc, vc     (q-box: i in [-4, TI+6), j in [-3, TJ+3))
  CUtensorMap acc[6];   // cx, cy, xfa, yfa, mfx, mfy (interior tile)
  CUtensorMap met[5];   // dx, dy, rdxa, rdya, area (q-box, level 0)
  double* delpo;
  double* pto;
  double* wo;
  double* acco[6];      // interior origins of the accumulator outputs (may alias inputs)
  const double* rarea;  // interior origin (2-D)
  int64_t sj, sk;
  int i0, j0;           // allocated column / row of the interior origin
  int ni, nj, nk, kchunk;
  double p1, p2, dt, damp_w;
};

int dsw_transport_maps(DswTpArgs& a, const Geo& g, const fv3b_field* qbox5, const fv3b_field* acc6,
                       const fv3b_field* met5);
int launch_dsw_transport(const DswTpArgs& a, cudaStream_t st);

}  // namespace fv3b
