// d_sw launch interfaces (d_sw.cu entry point -> dsw_transport.cu kernel).
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace fv3b {

struct DswTpArgs {
  CUtensorMap qbox[5];  // delp, pt, w, uc, vc     (q-box: i in [-4, TI+6), j in [-3, TJ+3))
  CUtensorMap met[4];   // area, rarea, del6_u, del6_v (q-box, level 0)
  const double* dx;     // courant metrics, interior origins (2-D, the 3-D fields' J stride)
  const double* dy;
  const double* rdxa;
  const double* rdya;
  double* delpo;
  double* pto;
  double* wo;
  const double* acci[6];  // interior origins of cx, cy, xfa, yfa, mfx, mfy
  bool acc_reset;         // read the accumulator inputs as 0.0
  double* dp1o;           // optional: copy of the input delp (interior origin)
  double* acco[6];        // and of their outputs (may alias the inputs)
  const double* rarea;  // interior origin (2-D)
  int64_t sj, sk;
  int64_t mlo, mhi;     // offsets (from the interior origin) of a 2-D metric's first / last allocated element
  int i0, j0;           // allocated column / row of the interior origin
  int ni, nj, nk, kchunk;
  double p1, p2, dt, damp4, damp4h;  // del6 coefficient, half of it (mass-weighted chains)
};

int dsw_transport_maps(DswTpArgs& a, const Geo& g, const fv3b_field* qbox5, const fv3b_field* acc6,
                       const fv3b_field* met4);
int launch_dsw_transport(const DswTpArgs& a, cudaStream_t st);

}  // namespace fv3b

namespace fv3b {

// d_sw momentum group: d_sw_courant + d_sw_ke + d_sw_vort + d_sw_damp and the
// u / v statements of d_sw_update.
struct DswMoArgs {
  CUtensorMap u, v, uc, vc;  // u: q-box + 1 row; v, uc, vc: q-box
  CUtensorMap met[12];       // dx (+1 row), dy, rdxa, rdya, area, f0, rarea, rdx, rdy, dxc, dyc, rarea_c
  double* uo;
  double* vo;
  const double* del6_u;  // interior origins (2-D, the 3-D fields' J stride)
  const double* del6_v;
  int64_t sj, sk;
  int64_t mlo, mhi;  // offsets (from the interior origin) of a 2-D metric's first / last allocated element
  int i0, j0, ni, nj, nk, kchunk;
  double p1, p2, dt, dddmp, d2_bg, da_min, dampv;
};

int dsw_momentum_maps(DswMoArgs& a, const Geo& g, const fv3b_field& u, const fv3b_field& v, const fv3b_field& uc,
                      const fv3b_field& vc, const fv3b_field* met12);
int launch_dsw_momentum(const DswMoArgs& a, cudaStream_t st);

}  // namespace fv3b
