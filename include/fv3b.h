/*
 * fv3b.h — C ABI of the B200 FV3 dycore engine (libfv3b.so).
 *
 * This is the boundary below the Python drop-in for the reference engine
 * slot.  The reference declares, but does not ship, the engine modules
 * `stencilkit.executor.scheduled` (run_scheduled / benchmark / TimingStats /
 * BenchmarkResult / timings_to_csv) and `stencilkit.executor.bandwidth`
 * (measure_bandwidth)  — reference pkg/src/stencilkit/executor/__init__.py:6-13,
 * contracts SPEC.md:366-427 — and its executing engine is
 * `run_reference(program, inputs, domain, placement)` (executor/reference.py:307-339).
 * Each entry point below executes one shipped stencil program (or one fused
 * group of its stencils) with exactly the semantics of run_reference on that
 * program; the Python layer (paper_2205_04148_b200.executor) binds them with
 * ctypes.  A ctypes binding is the reference-side integration: see
 * INTEGRATION.md.
 *
 * Conventions
 *  - All arithmetic is IEEE fp64, no FMA contraction (built with -fmad=false),
 *    statement order and association as in the .stn source.
 *  - Fields are borrowed device pointers in the reference Layout
 *    (scheduling.py:323-407): I unit-stride, rows padded, strides in
 *    elements.  `data` is the address of the first allocated element;
 *    the interior origin is data + sum(halo_lo[a] * stride[a]).
 *  - Every 3-D field passed to one call must share strides; 2-D fields share
 *    the J stride.  Output fields must not alias inputs (the reference
 *    materialises every right-hand side before its store, reference.py:10-12).
 *  - Device buffers that are not fields (halo message buffers, index lists,
 *    barrier flag words) are passed as BUFFER FIELDS: rank 1, `data` = the
 *    buffer's address, shape[0] = its capacity in elements of its type
 *    (doubles, int32 or 64-bit words as the entry states), stride[0] = 1.
 *    Entries check the capacity they need; no address travels in a scalar.
 *  - Status 0 = OK.  Negative = error; fv3b_last_error() has the message.
 *    No exceptions or aborts cross the ABI; no implicit synchronisation:
 *    work is enqueued on `stream` (a cudaStream_t, NULL = legacy default).
 *  - Reentrant; callable from any host thread; one process per GPU.
 */
#ifndef FV3B_H
#define FV3B_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FV3B_ABI_VERSION 5

enum {
  FV3B_OK = 0,
  FV3B_EINVAL = -1,   /* bad argument count / null pointer */
  FV3B_ELAYOUT = -2,  /* stride, halo or alignment mismatch */
  FV3B_EDOMAIN = -3,  /* domain below the program minimum */
  FV3B_ELAUNCH = -4,  /* CUDA launch or runtime error */
};

/* One borrowed field view.  rank = number of declared axes (3 for I,J,K,
 * 2 for I,J, 1 for K).  Axes are in I, J, K order, I unit-stride. */
typedef struct {
  double* data;
  int64_t stride[3];
  int32_t shape[3];
  int32_t halo_lo[3];
  int32_t rank;
} fv3b_field;

/* Compute domain and edge ownership (== RankPlacement, ir/graph.py:226-239):
 * horizontal regions anchored on an edge fire only when it is owned. */
typedef struct {
  int32_t ni, nj, nk;
  uint8_t own_i_start, own_i_end, own_j_start, own_j_end;
} fv3b_domain;

int fv3b_abi_version(void);
const char* fv3b_last_error(void);

/* Launch-configuration knobs (the launch-config tuner, tools/tune.py, and the
 * parity tests that force a level-march shape).  Process-wide; a value of 0
 * restores the automatic choice.  The level-marching tile kernels give each
 * CTA a chunk of `kchunk` consecutive levels; automatically the chunk makes
 * the launch one wave of equal chunks.  A kernel-specific knob wins over
 * FV3B_TUNE_KCHUNK.  Replaces the reference's schedule menu
 * (scheduling.py:28 tile sizes, :266-315 enumerate_schedules) for the knobs
 * that are run-time choices here. */
enum {
  FV3B_TUNE_KCHUNK = 0,               /* every level-marching tile kernel */
  FV3B_TUNE_KCHUNK_DSW_TRANSPORT = 1, /* d_sw delp / pt / w transport */
  FV3B_TUNE_KCHUNK_DSW_MOMENTUM = 2,  /* d_sw u / v momentum */
  FV3B_TUNE_KCHUNK_CSW = 3,           /* c_sw (c_grid) */
  FV3B_TUNE_KCHUNK_TRACER = 4,        /* tracer_2d */
  FV3B_TUNE_KCHUNK_FV_TP_2D = 5,      /* fv_tp_2d program */
  FV3B_TUNE_RIEM_COLS = 6,            /* columns per CTA of the vertical solver (0 = automatic) */
  FV3B_TUNE_COUNT = 7
};
int fv3b_tune_set(int knob, int value); /* value >= 0; FV3B_EINVAL for an unknown knob */
int fv3b_tune_get(int knob);            /* current value (0 = automatic), -1 for an unknown knob */

/* K0  copy.stn — `out = inp` over the interior (PAPER.md:589 copy stencil).
 *     fields: inp, out.  scalars: none. */
int fv3b_copy(const fv3b_field* f, int nf, const double* s, int ns,
              const fv3b_domain* d, void* stream);

/* K1  fv_tp_2d.stn — FV3 fv_tp_2d (x/y PPM fluxes + inner updates) and the
 *     flux-form update of q.  fields: q, crx, cry, xfx, yfx (3-D),
 *     area, rarea (2-D), q_out (3-D).  scalars: ppm_p1, ppm_p2. */
int fv3b_fv_tp_2d(const fv3b_field* f, int nf, const double* s, int ns,
                  const fv3b_domain* d, void* stream);

/* K7  tracer_2d.stn — nq tracers advected with accumulated Courant numbers
 *     and mass fluxes, batched in one launch.  fields: cx, cy, xfx, yfx, mfx,
 *     mfy, dp1 (3-D), area, rarea (2-D), then q_in[0..nq), q_out[0..nq).
 *     scalars: ppm_p1, ppm_p2. */
int fv3b_tracer_2d(const fv3b_field* f, int nf, const double* s, int ns,
                   const fv3b_domain* d, void* stream);

/* K4  riem_solver_c.stn — semi-implicit vertical acoustic solve per column.
 *     Program domain nk = interface levels (layers + 1).  fields: dm, pt, w
 *     (layers), gz (interfaces), ws (2-D), pef, gz_out (interfaces), scratch
 *     (3-D, one level array per column).  The outputs and the scratch stage
 *     column intermediates and must not alias the inputs.
 *     scalars: ptop, rdgas, grav, gama, p_fac, dt. */
int fv3b_riem_solver_c(const fv3b_field* f, int nf, const double* s, int ns,
                       const fv3b_domain* d, void* stream);

/* K5  remap_profile.stn / remap_tracers.stn — PPM edge solve + limited
 *     sub-grid coefficients.  Program domain nk = interface levels.
 *     fields: delp, then per tracer: q, a4_2, a4_3, a4_4 (outputs must not
 *     alias the inputs).  scalars: none.  Grouped form (fields at several
 *     layer thicknesses, one launch): scalars s[g] = fields in group g, and
 *     the field list is, per group, its thickness then 4 per member. */
int fv3b_remap_profile(const fv3b_field* f, int nf, const double* s, int ns,
                       const fv3b_domain* d, void* stream);

/* K5b remap mapping (FV3 map1_ppm; oracle/remap_map.py): integrate each
 *     tracer's remap_profile parabolas over the target layers of
 *     pe2 = ak + bk * ps (ps = ptop + sum of delp), then delp <- pe2
 *     differences in place.  Program domain nk = interface levels.
 *     fields: delp, ak (K), bk (K), then per tracer: q, a4_2, a4_3, a4_4,
 *     q_out (q_out must not alias any other field).  scalars: none.
 *     Grouped form: scalars s[g] = fields in group g; fields ak, bk, then
 *     per group its thickness (rewritten with its pe2 differences) and 5
 *     per member.  s[g] < 0: group g (of -s[g] fields) maps in log pressure
 *     (FV3 pt, kord_tm < 0): its thickness slot holds log(pe1) and is
 *     followed by log(pe2) (interfaces, fv3b_log_thickness), nothing is
 *     rewritten, and its profiles were formed at the log-pressure thickness. */
int fv3b_remap_map(const fv3b_field* f, int nf, const double* s, int ns,
                   const fv3b_domain* d, void* stream);

/* K5d log-pressure coordinate: pe1[0] = ak[0], pe1[k+1] = pe1[k] +
 *     delp[k], ps = pe1[nk], pe2 = (pe1[0], ak + bk * ps, ps); lnpe1 =
 *     det_log(pe1), lnpe2 = det_log(pe2), dlnp[k] = lnpe1[k+1] - lnpe1[k]
 *     (the thickness remap_profile takes for a field remapped in log
 *     pressure, and the interfaces fv3b_remap_map's log group maps between).
 *     fields: delp (3-D), ak, bk (K), dlnp (3-D layers), lnpe1, lnpe2 (3-D
 *     interfaces).  No scalars.  Domain nk = layers. */
int fv3b_log_thickness(const fv3b_field* f, int nf, const double* s, int ns,
                       const fv3b_domain* d, void* stream);

/* K5c pressure / heat-capacity diagnostics of the remapped state (FV3
 *     fv_mapz pe, pk, pkz and moist_cv; oracle/thermo.py):
 *     pe[0] = ptop, pe[k+1] = pe[k] + delp[k]; peln = log(pe); pk =
 *     exp(akap * peln) (deterministic fdlibm log / exp, detmath.cuh); pkz =
 *     (pk[k+1] - pk[k]) / (akap * (peln[k+1] - peln[k])); cvm = (1 - (qv + ql
 *     + qs)) cv_air + qv cv_vap + ql c_liq + qs c_ice (ql = liquid + rain,
 *     qs = ice + snow + graupel).  Program domain nk = interface levels.
 *     fields: delp, 0..6 moist tracers (vapour, liquid, rain, ice, snow,
 *     graupel; absent ones are 0), pe, peln, pk (interfaces), pkz, cvm
 *     (layers; outputs must not alias).  scalars: ptop, akap, cv_air,
 *     cv_vap, c_liq, c_ice. */
int fv3b_moist_pk(const fv3b_field* f, int nf, const double* s, int ns,
                  const fv3b_domain* d, void* stream);

/* K2  c_sw.stn — C-grid half step.  fields: u, v, delp, pt, w (3-D); dx, dy,
 *     dxc, dyc, rdxc, rdyc, rarea, rarea_c, fc (2-D); uc, vc, delpc, ptc, wc
 *     (3-D outputs).  scalars: dt2. */
int fv3b_c_sw(const fv3b_field* f, int nf, const double* s, int ns,
              const fv3b_domain* d, void* stream);

/* K2+K4  c_grid.stn — c_sw + riem_solver_c + p_grad_c fused (program domain
 *     nk = layers + 1).  fields: u, v, delp, pt, w, gz (3-D); the 9 c_sw
 *     metrics, ws (2-D); uc, vc (3-D outputs); scratch delpcc, ptcc, wcc, pkc,
 *     gzc, riem (3-D, >= 1-cell halo).  scalars: dt2, ptop, rdgas, grav, gama,
 *     p_fac. */
int fv3b_c_grid(const fv3b_field* f, int nf, const double* s, int ns,
                const fv3b_domain* d, void* stream);

/* K3  d_sw.stn — D-grid Lagrangian step (two fused kernels), with del6 flux
 *     damping (FV3 delnflux, nord = 2) of delp, pt, w and the vorticity.
 *     fields: u, v, w, delp, pt, uc, vc, cx, cy, xfa, yfa, mfx, mfy (3-D);
 *     dx, dy, dxc, dyc, rdx, rdy, rdxa, rdya, area, rarea, rarea_c, f0,
 *     del6_u, del6_v (2-D); u, v, w, delp, pt, cx, cy, xfa, yfa, mfx, mfy
 *     outputs (3-D; accumulators may alias).  [optional 39th: dp1_out,
 *     receives the input delp].  scalars: ppm_p1, ppm_p2, dt, dddmp, d2_bg,
 *     da_min, damp4, damp4h (= damp4 / 2), dampv [, acc_reset: nonzero reads
 *     the accumulator inputs as 0.0]. */
int fv3b_d_sw(const fv3b_field* f, int nf, const double* s, int ns,
              const fv3b_domain* d, void* stream);

/* nh_d.stn — D-grid vertical solve (riem_solver3 role), program domain
 *     nk = layers + 1.  fields: delp, pt, w, gz (3-D), ws (2-D), pef,
 *     gz_out, w_out, scratch (3-D; outputs and scratch must not alias
 *     inputs).  scalars: ptop, rdgas, grav, gama, p_fac, dt. */
int fv3b_nh_d(const fv3b_field* f, int nf, const double* s, int ns,
              const fv3b_domain* d, void* stream);

/* p_grad_d.stn — D-grid pressure-gradient force (nh_p_grad role), program
 *     domain nk = layers + 1.  fields: u, v, pef, gz (3-D), rdx, rdy (2-D),
 *     u_out, v_out (3-D).  scalars: dt. */
int fv3b_p_grad_d(const fv3b_field* f, int nf, const double* s, int ns,
                  const fv3b_domain* d, void* stream);

/* K6  halo_update, on-device parts.
 *   fv3b_halo_periodic  fill the I/J halos of up to 32 fields of a doubly
 *                       periodic single-rank domain.  scalars: [halo width].
 *   fv3b_halo_pack / fv3b_halo_unpack  copy an edge strip (all levels) of up
 *                       to 32 fields to / from one contiguous buffer for the
 *                       NCCL neighbour exchange.  fields: the fields, then
 *                       the message buffer (buffer field, doubles).
 *                       scalars: [i0, j0, w, h]. */
int fv3b_halo_periodic(const fv3b_field* f, int nf, const double* s, int ns,
                       const fv3b_domain* d, void* stream);
int fv3b_halo_pack(const fv3b_field* f, int nf, const double* s, int ns,
                   const fv3b_domain* d, void* stream);
int fv3b_halo_unpack(const fv3b_field* f, int nf, const double* s, int ns,
                     const fv3b_domain* d, void* stream);

/*   fv3b_halo_pack_rects / fv3b_halo_unpack_rects  every edge and corner
 *                       strip of one decomposed-domain halo update (up to 8
 *                       rectangles, all levels, up to 32 fields sharing one
 *                       level count) to / from one message buffer in one
 *                       launch.  fields: the fields, then the message
 *                       buffer (buffer field, doubles).  scalars: [nrect,
 *                       then (i0, j0, w, h, element offset) per rectangle,
 *                       interior-relative].  Rectangle r of
 *                       field t, level k is at offset_r + (t*levels + k)*w*h,
 *                       row-major.  Replaces the paper's Python halo updater
 *                       pack/unpack. */
int fv3b_halo_pack_rects(const fv3b_field* f, int nf, const double* s, int ns,
                         const fv3b_domain* d, void* stream);
int fv3b_halo_unpack_rects(const fv3b_field* f, int nf, const double* s, int ns,
                           const fv3b_domain* d, void* stream);

/*   fv3b_halo_peer_rects  the same strips without a message buffer: each
 *                       rectangle goes from a source field straight into a
 *                       destination field that may be another rank's
 *                       allocation (CUDA IPC / peer-mapped over NVLink, or
 *                       another block on the same device).  fields: nf
 *                       sources, then rectangle r's destination of field t
 *                       at index nf + r*nf + t (all with the sources'
 *                       strides and level count).  scalars: [nf, nrect,
 *                       then (src i0, src j0, dst i0, dst j0, w, h) per
 *                       rectangle, interior-relative].  Up to 32 fields, 8
 *                       rectangles.  Replaces pack + send/recv + unpack of
 *                       the paper's halo updater. */
int fv3b_halo_peer_rects(const fv3b_field* f, int nf, const double* s, int ns,
                         const fv3b_domain* d, void* stream);

/*   fv3b_halo_peer_idx  the cubed-sphere update without message buffers:
 *                       up to 8 destination sets (a neighbour tile's fields,
 *                       peer-mapped, or this tile's own for the corner
 *                       fill).  Entry s of set r's device int32 list is
 *                       (source slot, source offset, destination slot,
 *                       destination offset, sign +/-1), offsets
 *                       interior-relative; all levels.  fields: nf sources,
 *                       then set r's destination of slot t at nf + r*nf + t,
 *                       then set r's list (buffer field, int32, 5 per
 *                       entry) at nf*(1+nset) + r.  scalars: [nf, nset].
 *                       Up to 32 fields sharing one level count. */
int fv3b_halo_peer_idx(const fv3b_field* f, int nf, const double* s, int ns,
                       const fv3b_domain* d, void* stream);

/*   fv3b_peer_barrier  stream-ordered barrier of a rank with its neighbours
 *                       over peer-mapped 64-bit flag words (the ordering of
 *                       fv3b_halo_peer_rects without host synchronisation).
 *                       One thread bumps (bump != 0) or reads the rank's
 *                       counter e, release-stores e into its word in every
 *                       neighbour's flag array, then acquire-spins until each
 *                       neighbour's word in its own array is >= e; after 10 s
 *                       it sets the error word and traps (the stream fails
 *                       loudly instead of storing into a halo a neighbour
 *                       may still read).  fields (buffer fields of one
 *                       element): the counter (u64), the error word
 *                       (int32), then (remote word, local word) per
 *                       neighbour, up to 8 neighbours.  scalars: [bump,
 *                       npeer].  d may be NULL. */
int fv3b_peer_barrier(const fv3b_field* f, int nf, const double* s, int ns,
                      const fv3b_domain* d, void* stream);

/*   fv3b_halo_gather / fv3b_halo_scatter  index-list halo movement for the
 *                       cubed-sphere update (edge strips arrive rotated and,
 *                       for vector pairs, component-swapped with a sign;
 *                       corner fill).  fields: the fields, then the
 *                       message buffer (buffer field, doubles) and the index
 *                       list (buffer field, int32).  scalars: [n].  Gather entries
 *                       are (field slot, interior-relative cell offset);
 *                       scatter entries (field slot, offset, sign +/-1).
 *                       Level k of entry s is buf[k*n + s]; all levels of up
 *                       to 32 fields sharing one level count. */
int fv3b_halo_gather(const fv3b_field* f, int nf, const double* s, int ns,
                     const fv3b_domain* d, void* stream);
int fv3b_halo_scatter(const fv3b_field* f, int nf, const double* s, int ns,
                      const fv3b_domain* d, void* stream);

/*   fv3b_memcpy2d  host I/O helper: `height` rows of `width` bytes from src
 *                  (row pitch spitch bytes) to dst (pitch dpitch) on `stream`,
 *                  host or device pointers (unified addressing; pinned host
 *                  memory for asynchrony).  Used by tools/io_variants.py to
 *                  measure interior-column transfers of halo-inclusive
 *                  (I, J, K) arrays (not faster than whole arrays: the
 *                  bidirectional PCIe rate drops with row-wise DMA). */
int fv3b_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                  int64_t width, int64_t height, void* stream);

/*   fv3b_enable_peer_access  multi-GPU helper: kernels on the current
 *                  device may access device `peer`'s memory (NVLink P2P;
 *                  parallel.IpcPeers calls it for every neighbour on another
 *                  GPU).  Already enabled is not an error. */
int fv3b_enable_peer_access(int peer);

/*   fv3b_transpose  state layout conversion for host I/O: copy the d->ni x
 *                   d->nj x d->nk region at f[0].data to f[1].data where one
 *                   field has unit K stride (the reference's numpy (I, J, K)
 *                   C-order arrays, fieldio / run_reference) and the other
 *                   unit I stride (the Layout).  fields: src, dst (rank 3,
 *                   data = region origin, halo_lo ignored).  scalars: none. */
int fv3b_transpose(const fv3b_field* f, int nf, const double* s, int ns,
                   const fv3b_domain* d, void* stream);

/*   fv3b_face_thickness  layer thickness at the D-grid wind points for the
 *                   remapping of u and v: du = 0.5 * (delp[0,-1,0] + delp),
 *                   dv = 0.5 * (delp[-1,0,0] + delp) over the interior.
 *                   fields: delp (I / J halo >= 1), du, dv.  scalars: none. */
int fv3b_face_thickness(const fv3b_field* f, int nf, const double* s, int ns,
                        const fv3b_domain* d, void* stream);

/*   fv3b_selftest_fastmath  diagnostic: over n device operand pairs, adds to
 *                   counts[0..3] (device, zeroed by the caller) the fast-path
 *                   quotients x/y that differ from IEEE division although
 *                   valid, the rejected ones, and the same two counts for
 *                   det_log(|x|).  counts[0] and counts[2] must stay 0. */
int fv3b_selftest_fastmath(const double* x, const double* y, int n,
                           unsigned long long* counts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FV3B_H */
