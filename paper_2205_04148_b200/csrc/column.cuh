// Column-solver launch interface shared by column.cu and the fused
// C-grid / D-grid programs.
#pragma once

#include "common.cuh"

namespace fv3b {

struct RiemArgs {
  View dm, pt, w, gz, ws, pef, gzo, wout;
  View scr;                      // 3-D scratch: one level array per column (gam -> aa -> gw)
  bool has_wout;                 // nh_d: the solver's w2 is written back (w = w2)
  int ilo, jlo, ni_ext, nj_ext;  // column range [ilo, ilo+ni_ext) x [jlo, jlo+nj_ext)
  int nk;                        // layers; interfaces 0..nk
  double dt, ptop, rdgas, grav, gama, p_fac;
};

int launch_riem(const RiemArgs& a, cudaStream_t st);

}  // namespace fv3b
