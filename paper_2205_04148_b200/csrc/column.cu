// K4 riem_solver_c and K5 remap_profile: vertical column solvers
// (programs/riem_solver_c.stn, remap_profile.stn, remap_tracers.stn;
// templates.riem_stencils / remap_stencils).
//
// One thread owns one column (i, j) and marches in K; consecutive threads
// own consecutive i, so every level's loads/stores are coalesced 256-B rows
// of the I-unit-stride Layout.  The DSL expresses each tridiagonal solve as a
// FORWARD stencil followed by a BACKWARD stencil (validate.py:171-186); the
// values a backward sweep consumes are staged per column in shared memory
// (up to 32 columns x (nk+1) levels per array) so nothing round-trips through HBM.
// Every statement is evaluated with the .stn's operation order, so results
// are bitwise the interpreter's (log is the deterministic det_log of the
// oracle extension, detmath.cuh).
#include <math.h>

#include <type_traits>

#include "column.cuh"
#include "detmath.cuh"
#include "fastdiv.cuh"

namespace fv3b {

constexpr int NC_MAX = 32;  // columns per CTA (at most one warp; see cols_per_cta)

// numpy.maximum semantics (NaN-propagating, reference.py:247-257)
__device__ __forceinline__ double np_max(double a, double b) {
  if (isnan(a) || isnan(b)) return a + b;
  return a > b ? a : (b > a ? b : a);
}


// Software-pipelined level streaming for the column sweeps: step s = 0..n-1
// of a pass loads its per-level global operands U steps ahead into a
// register double buffer, so the loop-carried recurrence never waits on
// HBM/L2 latency (the reference interpreter's level loop, reference.py:293,
// becomes a register pipeline).  load(s) -> T must be side-effect free;
// use(s, T) runs strictly in step order.
template <int U, class T, class LoadF, class UseF>
__device__ __forceinline__ void pipelined(int n, LoadF load, UseF use) {
  // ring of U register slots; step s uses the value loaded U steps earlier.
  // Loads are clamped to the last step (always a valid level) so the main
  // loop carries no guards and the compiler can interleave the independent
  // work (logs, divisions) of U consecutive levels around the recurrence.
  // The body is instantiated U + 1 times only: the kernels are large and a
  // few warps per SM cannot hide instruction-cache misses.
  T a[U];
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = load(min(u, n - 1));
  int s0 = 0;
  for (; s0 + U <= n; s0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T v = a[u];
      a[u] = load(min(s0 + U + u, n - 1));
      use(s0 + u, v);
    }
  }
#pragma unroll 1
  for (int s = s0; s < n; ++s) use(s, load(s));
}

struct D1 { double x; };
struct D2 { double x, y; };
struct D3 { double x, y, z; };

// Level streaming through a per-thread shared-memory ring filled by
// cp.async (LDGSTS): the operands of the next RD levels are in flight
// without holding registers, so the sweeps' loads run far ahead of the
// recurrence at the 8 warps per SM the column count allows.  A Stream
// gives the NF operand addresses of step 0 and their per-step element
// deltas (negative for the backward sweeps); use(s, T) runs strictly in step
// order.  The thread's slot (l, f) is ring[(l * NF + f) * 32] (stride of a
// full warp of columns: consecutive threads, consecutive banks).  Steps are
// consumed in batches of RU (one wait per batch; the batch's independent
// work interleaves like pipelined()'s).
#ifndef FV3B_RD
#define FV3B_RD 8
#endif
#ifndef FV3B_RU
#define FV3B_RU 2
#endif
constexpr int RD = FV3B_RD, RU = FV3B_RU;
constexpr int RING = RD * 3 * NC_MAX;  // doubles of one CTA's operand ring
static_assert(RD % RU == 0 && RD > RU, "ring depth is a multiple of the batch");

template <int NF>
struct Stream {
  const double* p[NF];
  int64_t d[NF];
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The ring is addressed by 32-bit shared-window byte offsets (no generic ->
// shared conversion per copy, immediate field offsets in LDGSTS / LDS).
__device__ __forceinline__ void cp_async8_s(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}

template <int NF, class T, class UseF>
__device__ __forceinline__ void staged(double* ring, int n, Stream<NF> st, UseF use) {
  constexpr uint32_t SSB = NF * NC_MAX * sizeof(double);  // bytes per slot
  constexpr uint32_t FB = NC_MAX * sizeof(double);         // bytes between a slot's fields
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t last = base + (RD - 1) * SSB;
  uint32_t wr = base;  // next slot to fill
  auto fill = [&]() {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      cp_async8_s(wr + f * FB, st.p[f]);
      st.p[f] += st.d[f];
    }
    wr = wr == last ? base : wr + SSB;
  };
  uint32_t rp = base;  // next slot to read
  auto read = [&]() {
    T v;
    if constexpr (NF == 1) v = T{lds64(rp)};
    else if constexpr (NF == 2) v = T{lds64(rp), lds64(rp + FB)};
    else v = T{lds64(rp), lds64(rp + FB), lds64(rp + 2 * FB)};
    rp = rp == last ? base : rp + SSB;
    return v;
  };
#pragma unroll
  for (int s = 0; s < RD; ++s) {
    if (s < n) fill();
    cp_async_commit();
  }
  // main batches: every step's refill (step s + RD) exists, so no guards
  int s0 = 0;
#pragma unroll 1
  for (; s0 + RU <= n - RD; s0 += RU) {
    cp_async_wait<RD - RU>();  // the batch's RU groups have landed
    T v[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) v[u] = read();
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      use(s0 + u, v[u]);
      fill();  // into a slot this batch has read
      cp_async_commit();
    }
  }
  // the last < RD + RU steps, one group per step (empty once the refills end)
#pragma unroll 1
  for (; s0 < n; ++s0) {
    cp_async_wait<RD - 1>();
    const T v = read();
    use(s0, v);
    if (s0 + RD < n) fill();
    cp_async_commit();
  }
  cp_async_wait<0>();
}

#ifndef FV3B_PF  // (overridable for tuning sweeps, tools/build_variant.py)
#define FV3B_PF 4
#define FV3B_PFS 12
#endif
[[maybe_unused]] constexpr int PF = FV3B_PF;    // prefetch distance (levels), riem passes with long bodies (A, C)
[[maybe_unused]] constexpr int PFS = FV3B_PFS;  // riem passes with short bodies (B, D, E, F): L2-resident staging reads

// Statement-for-statement restatement of templates.riem_stencils for one
// column.  FAST: branch-free divisions/logs (fastdiv.cuh), returns false if
// any of them left nvcc's fast-path range, in which case the caller
// re-evaluates the column with EXACT.
//
// One level array per column lives in shared memory (S0); the others the
// sweeps carry between passes live in global memory in the column's own
// slots (L2-resident: written and re-read by the same thread within the
// kernel, prefetched through the register ring like every other operand):
//   scr  gam (riem_pp_fwd) -> aa (riem_w_fwd) -> gw (riem_w_sweep);
//   pef  holds pem (riem_pem) from pass A until pass E writes pe2 + pem;
//   gzo  holds pmc (riem_layer) from pass A until pass F, which reads it
//        instead of re-evaluating dm / log(pem[k+1] / pem[k]) (the same
//        IEEE operations on the same operands, so the same bits).
// With 648 B of shared memory per column every column of a C2 call is
// resident at once.  Outputs and scratch must not alias the inputs.
template <bool FAST>
__device__ __forceinline__ bool riem_column(const RiemArgs& a, int i, int j, int c, int NC, double* sm) {
  ColArith<FAST> ar;
  const int nk = a.nk;
  double* S0 = sm + c;  // pp -> w2 -> pe2 (shifted one level down)
#ifndef FV3B_RIEM_REGRING
  double* ring = sm - RING + c;  // staged() operand ring (RD levels x 3) below S0
#endif
#define AT(S, k) (S)[(k) * NC]
  const double dt = a.dt, ptop = a.ptop, rdgas = a.rdgas, grav = a.grav, gama = a.gama;
  const double* __restrict__ dm = a.dm.ptr(i, j, 0);
  const double* __restrict__ pt = a.pt.ptr(i, j, 0);
  const double* __restrict__ w = a.w.ptr(i, j, 0);
  const double* __restrict__ gz = a.gz.ptr(i, j, 0);
  double* pf = a.pef.ptr(i, j, 0);
  double* go = a.gzo.ptr(i, j, 0);
  double* S1 = a.scr.ptr(i, j, 0);  // gam -> aa -> gw
  const int64_t sk = a.dm.sk, sp = a.pef.sk, sg = a.gzo.sk, s1 = a.scr.sk;

  // ---- pass A (forward): riem_pem, riem_layer, riem_coef, riem_pp_fwd ----
  // Level 0 and level nk-1 are peeled so the pipelined body is branch-free
  // (the scheduler interleaves the independent logs / divisions of
  // consecutive levels around the bet / pp recurrence).  For k >= 1 the
  // statement ppc = (ddc[k-1] - ppc[k-1]) / betp[k-1] also covers k = 1,
  // where the reference has ddc[0] / betp[0]: ppc[0] = 0 and x - 0.0 == x.
  {
    double pem0 = ptop;  // pem(k)
    pf[0] = pem0;
    double pe_prev = 0.0, grat_prev = 0.0, bet_prev = 0.0, pp_prev = 0.0;
    double dm_k = __ldg(dm), gzk = __ldg(gz);
    auto level = [&](int k, const D3& v, auto first, auto last) {
      const double dm_n = v.x, gzk1 = v.y;
      const double pem1 = pem0 + dm_k;  // pem(k+1) = pem + dm
      pf[(k + 1) * sp] = pem1;
      const double pmk = ar.div(dm_k, ar.log(ar.div(pem1, pem0)));
      go[k * sg] = pmk;
      const double pek = ar.div(dm_k * rdgas * v.z, gzk - gzk1) - pmk;
      // layer k coefficients (riem_coef)
      double grat = 0.0, bb = 2.0;
      if constexpr (!decltype(last)::value) {
        grat = ar.div(dm_k, dm_n);
        bb = 2.0 * (1.0 + grat);
      }
      // interface k of riem_pp_fwd (uses layer k-1's dd, needing pe(k))
      if constexpr (decltype(first)::value) {
        bet_prev = bb;
        pp_prev = 0.0;
        AT(S0, 0) = 0.0;
      } else {
        const double dd_prev = 3.0 * (pe_prev + grat_prev * pek);
        const double rb = ar.rcp(bet_prev);
        const double ppk = ar.div_r(dd_prev - pp_prev, bet_prev, rb);
        const double gam = ar.div_r(grat_prev, bet_prev, rb);
        bet_prev = bb - gam;
        pp_prev = ppk;
        AT(S0, k) = ppk;
        S1[k * s1] = gam;
      }
      pe_prev = pek;
      grat_prev = grat;
      pem0 = pem1;
      dm_k = dm_n;
      gzk = gzk1;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    level(0, D3{__ldg(dm + sk), __ldg(gz + sk), __ldg(pt)}, T_{}, F_{});
#ifdef FV3B_RIEM_REGRING
    pipelined<PF, D3>(
        nk - 2,
        [&](int s) {  // k = s + 1: dm(k+1), gz(k+1), pt(k)
          return D3{__ldg(dm + (s + 2) * sk), __ldg(gz + (s + 2) * sk), __ldg(pt + (s + 1) * sk)};
        },
        [&](int s, const D3& v) { level(s + 1, v, F_{}, F_{}); });
#else
    staged<3, D3>(ring, nk - 2, Stream<3>{{dm + 2 * sk, gz + 2 * sk, pt + sk}, {sk, sk, sk}},
                  [&](int s, const D3& v) { level(s + 1, v, F_{}, F_{}); });
#endif
    level(nk - 1, D3{0.0, __ldg(gz + nk * sk), __ldg(pt + (nk - 1) * sk)}, F_{}, T_{});
    // interface nk: pp = (dd[nk-1] - pp[nk-1]) / bet[nk-1], dd[nk-1] = 3*pe[nk-1]
    const double dd_prev = 3.0 * pe_prev;
    AT(S0, nk) = ar.div(dd_prev - pp_prev, bet_prev);
  }

  // ---- pass B (backward): riem_pp_bwd, then aa (riem_w_fwd) -------------
  const double t1g = gama * 2.0 * dt * dt;
  {
    double ppn = AT(S0, nk);
    double gzn = __ldg(gz + (nk - 1) * sk);
    const double rgrav = ar.rcp(grav);
    double dz_n = ar.div_r(__ldg(gz + nk * sk) - gzn, grav, rgrav);  // dz(nk-1)
    S1[nk * s1] = ar.div(t1g, dz_n) * (pf[nk * sp] + ppn);   // aa(nk)
#ifdef FV3B_RIEM_REGRING
    pipelined<PFS, D3>(
        nk - 1,
        [&](int s) {  // gz(k-1), pem(k), gam(k)
          return D3{__ldg(gz + (nk - 2 - s) * sk), pf[(nk - 1 - s) * sp], S1[(nk - 1 - s) * s1]};
        },
#else
    staged<3, D3>(  // gz(k-1), pem(k), gam(k) for k = nk-1-s
        ring, nk - 1, Stream<3>{{gz + (nk - 2) * sk, pf + (nk - 1) * sp, S1 + (nk - 1) * s1}, {-sk, -sp, -s1}},
#endif
        [&](int s, const D3& v) {
          const int k = nk - 1 - s;
          const double ppk = AT(S0, k) - v.z * ppn;
          AT(S0, k) = ppk;
          const double dz_k = ar.div_r(gzn - v.x, grav, rgrav);      // dz(k-1)
          S1[k * s1] = ar.div(t1g, dz_k + dz_n) * (v.y + ppk);      // aa(k) = t1g/(dz(k-1)+dz(k))*(pem+pp)
          dz_n = dz_k;
          ppn = ppk;
          gzn = v.x;
        });
  }

  // ---- pass C (forward): riem_w_sweep (w2 replaces pp level by level) ----
  // (levels 0 and nk-1 peeled: their statements differ)
  const double ws = a.ws(i, j, 0);
  {
    double bw = 0.0, w2p = 0.0, aal = S1[0], rbw = 0.0;
    auto level = [&](int l, const D3& v, auto first, auto last) {
      const double dml = v.x, wl = v.y;
      const double aan = v.z;  // aa(l+1); aa(l) carried from the previous level
      double w2l;
      if constexpr (decltype(first)::value) {
        bw = dml - aan;
        rbw = ar.rcp(bw);
        w2l = ar.div_r(dml * wl + dt * AT(S0, 1), bw, rbw);
      } else {
        const double gw = ar.div_r(aal, bw, rbw);
        bw = dml - (aal + aan + aal * gw);
        rbw = ar.rcp(bw);
        if constexpr (decltype(last)::value)
          w2l = ar.div_r(dml * wl + dt * (AT(S0, l + 1) - AT(S0, l)) - aan * ws - aal * w2p, bw, rbw);
        else
          w2l = ar.div_r(dml * wl + dt * (AT(S0, l + 1) - AT(S0, l)) - aal * w2p, bw, rbw);
        S1[l * s1] = gw;  // aa(l) no longer needed
      }
      AT(S0, l) = w2l;  // pp(l) no longer needed
      w2p = w2l;
      aal = aan;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    auto ld = [&](int l) { return D3{__ldg(dm + l * sk), __ldg(w + l * sk), S1[(l + 1) * s1]}; };
    level(0, ld(0), T_{}, F_{});
#ifdef FV3B_RIEM_REGRING
    pipelined<PF, D3>(nk - 2, [&](int s) { return ld(s + 1); }, [&](int s, const D3& v) { level(s + 1, v, F_{}, F_{}); });
#else
    staged<3, D3>(ring, nk - 2, Stream<3>{{dm + sk, w + sk, S1 + 2 * s1}, {sk, sk, s1}},
                  [&](int s, const D3& v) { level(s + 1, v, F_{}, F_{}); });
#endif
    level(nk - 1, ld(nk - 1), F_{}, T_{});
  }

  // ---- pass D (backward): riem_w_back ----------------------------------
  {
    double w2n = AT(S0, nk - 1);
    double* wo = a.has_wout ? a.wout.ptr(i, j, 0) : nullptr;
    const int64_t so = a.wout.sk;
    if (wo) wo[(nk - 1) * so] = w2n;
#ifdef FV3B_RIEM_REGRING
    pipelined<PFS, D1>(
        nk - 1, [&](int s) { return D1{S1[(nk - 1 - s) * s1]}; },  // l = nk-2-s: gw(l+1)
#else
    staged<1, D1>(ring, nk - 1, Stream<1>{{S1 + (nk - 1) * s1}, {-s1}},  // gw(l+1), l = nk-2-s
#endif
        [&](int s, const D1& v) {
          const int l = nk - 2 - s;
          const double w2l = AT(S0, l) - v.x * w2n;
          AT(S0, l) = w2l;
          if (wo) wo[l * so] = w2l;
          w2n = w2l;
        });
  }

  // ---- pass E (forward): riem_pe, riem_out (pem recomputed in order) -----
  {
    double pe2 = 0.0, pem = ptop;
    const double rdt = ar.rcp(dt);
    pf[0] = pe2 + pem;
#ifdef FV3B_RIEM_REGRING
    pipelined<PFS, D2>(
        nk, [&](int s) { return D2{__ldg(dm + s * sk), __ldg(w + s * sk)}; },  // k = s+1: layer k-1
#else
    staged<2, D2>(ring, nk, Stream<2>{{dm, w}, {sk, sk}},  // k = s+1: layer k-1
#endif
        [&](int s, const D2& v) {
          const int k = s + 1;
          pe2 = pe2 + ar.div_r(v.x * (AT(S0, k - 1) - v.y), dt, rdt);
          pem = pem + v.x;
          AT(S0, k - 1) = pe2;  // pe2(k) (w2(k-1) consumed)
          pf[k * sp] = pe2 + pem;
        });
  }

  // ---- pass F (backward): riem_gz (pmc from pass A, in gz_out) ------------
  {
    double gzn = __ldg(gz + nk * sk);
    go[nk * sg] = gzn;
#ifdef FV3B_RIEM_REGRING
    pipelined<PFS, D3>(
        nk,
        [&](int s) {
          const int l = nk - 1 - s;
          return D3{__ldg(dm + l * sk), __ldg(pt + l * sk), go[l * sg]};
        },
#else
    staged<3, D3>(ring, nk, Stream<3>{{dm + (nk - 1) * sk, pt + (nk - 1) * sk, go + (nk - 1) * sg}, {-sk, -sk, -sg}},
#endif
        [&](int s, const D3& v) {
          const int l = nk - 1 - s;
          const double dml = v.x, pm = v.z;
          const double pe2l = l > 0 ? AT(S0, l - 1) : 0.0, pe2n = AT(S0, l);
          const double g = gzn + ar.div(dml * rdgas * v.y, np_max(a.p_fac * pm, pm + 0.5 * (pe2l + pe2n)));
          go[l * sg] = g;
          gzn = g;
        });
  }
#undef AT
  return ar.ok;
}

#ifdef FV3B_EXACT_NOINLINE
__device__ __noinline__ void riem_exact(const RiemArgs& a, int i, int j, int c, int NC, double* sm) {
  riem_column<false>(a, i, j, c, NC, sm);
}
#endif

// (minBlocks 1: without it ptxas settles on 128 registers and spills; 177
// registers cost no residency, which shared memory caps at 8 CTAs per SM)
__global__ void __launch_bounds__(NC_MAX, 1) riem_kernel(const RiemArgs a) {
  extern __shared__ double sm_[];
#ifdef FV3B_RIEM_REGRING
  double* sm = sm_;
#else
  double* sm = sm_ + RING;  // [operand ring | S0]
#endif
  const int c = threadIdx.x, NC = blockDim.x;
  const int cidx = blockIdx.x * NC + c;
  if (cidx >= a.ni_ext * a.nj_ext) return;
  const int i = a.ilo + cidx % a.ni_ext;
  const int j = a.jlo + cidx / a.ni_ext;
  // outputs never alias inputs: a failed fast evaluation is simply redone
#ifdef FV3B_EXACT_NOINLINE
  if (!riem_column<true>(a, i, j, c, NC, sm)) riem_exact(a, i, j, c, NC, sm);
#else
  if (!riem_column<true>(a, i, j, c, NC, sm)) riem_column<false>(a, i, j, c, NC, sm);
#endif
}

// ---------------------------------------------------------------------------
// remap_profile (templates.remap_stencils): edge values by a tridiagonal
// solve, then the Colella-Woodward limited PPM coefficients, fused into the
// backward sweep (layer k needs final edges k and k+1).
// ---------------------------------------------------------------------------
struct RemapArgs {
  View delp;                // thickness of the first group (strides shared by every field)
  const double* dp[16];     // per field: the interior origin of its group's thickness
  double* q[16];
  double* a2[16];
  double* a3[16];
  double* a4[16];
  int pair0[16];       // first field of each pair (a pair never spans two groups)
  int pairn[16];       // fields in the pair (1 or 2)
  int64_t sj, sk;
  int nq, npair, ni, nj, nk;  // nk layers (program domain nk+1)
};

// One (column, tracer) per thread: 8x the independent recurrences of a
// column-per-thread solver (the tracers' sweeps share nothing but delp), so
// the latency of the division chains is hidden by occupancy.  gam (delp
// only) is re-derived per tracer inside the forward sweep (its statement
// shares bet and d4 with the edge recurrence: same operands, same bits).
// The values the backward sweep consumes are staged in the tracer's own
// output slots (gam in a4_2[k], the forward edge in a4_3[k], both read back
// before level k's coefficients overwrite them; L2-resident).
template <bool FAST>
__device__ __forceinline__ bool remap_column(const RemapArgs& a, int i, int j, int t0, int nf) {
  // fields t0 and t0 + 1 (if any): gam depends on delp only, so it is
  // computed and staged once (in t0's a4_2 slots) for both
  constexpr int F = 2;
  ColArith<FAST> ar;
  const int nk = a.nk;

  const int64_t off = i + (int64_t)j * a.sj, sk = a.sk;
  const double* __restrict__ dp = a.dp[t0] + off;  // (t0 and t0 + 1 share a group: same thickness)
  const double* __restrict__ q[F];
  double* o2[F];
  double* o3[F];
  double* o4[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const int t = f < nf ? t0 + f : t0;
    q[f] = a.q[t] + off;
    o2[f] = a.a2[t] + off;  // t0's: gam(k), then a4_2; others: a4_2
    o3[f] = a.a3[t] + off;  // forward edge qe(k), then a4_3
    o4[f] = a.a4[t] + off;
  }
  double* G = o2[0];
  // forward: remap_edge_fwd (gam and qe)
  const double dp0 = __ldg(dp), dp1 = __ldg(dp + sk);
  const double grat0 = ar.div(dp1, dp0);
  const double bet0 = grat0 * (grat0 + 0.5);
  const double rb0 = ar.rcp(bet0);
  double gprev = ar.div_r(1.0 + grat0 * (grat0 + 1.5), bet0, rb0);
  double eprev[F], qprev[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const double q0 = __ldg(q[f]), q1 = __ldg(q[f] + sk);
    eprev[f] = ar.div_r((grat0 + grat0) * (grat0 + 1.0) * q0 + q1, bet0, rb0);
    qprev[f] = q0;
  }
  G[0] = gprev;
#pragma unroll
  for (int f = 0; f < F; ++f)
    if (f < nf) o3[f][0] = eprev[f];
  double dprev = dp0, d4last = 0.0;
#ifndef FV3B_RM_PF
#define FV3B_RM_PF 4  // measured with two fields per thread: 4 > 8
#endif
  pipelined<FV3B_RM_PF, D3>(
      nk - 1, [&](int s) { return D3{__ldg(dp + (s + 1) * sk), __ldg(q[0] + (s + 1) * sk), __ldg(q[1] + (s + 1) * sk)}; },
      [&](int s, const D3& v) {
        const int k = s + 1;
        const double d4 = ar.div(dprev, v.x);
        const double bet = 2.0 + d4 + d4 - gprev;  // gam(k-1)
        const double rb = ar.rcp(bet);
        const double qv[F] = {v.y, v.z};
#pragma unroll
        for (int f = 0; f < F; ++f) {
          eprev[f] = ar.div_r(3.0 * (qprev[f] + d4 * qv[f]) - eprev[f], bet, rb);
          qprev[f] = qv[f];
        }
        gprev = ar.div_r(d4, bet, rb);
        G[k * sk] = gprev;
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (f < nf) o3[f][k * sk] = eprev[f];
        dprev = v.x;
        d4last = d4;
      });
  const double d4p = d4last;
  const double abot = 1.0 + d4p * (d4p + 1.5);
  // gam(nk-1) = gprev
  double qen[F];
#pragma unroll
  for (int f = 0; f < F; ++f)
    qen[f] = ar.div(2.0 * d4p * (d4p + 1.0) * qprev[f] + __ldg(q[f] + (nk - 2) * sk) - abot * eprev[f],
                    d4p * (d4p + 0.5) - abot * gprev);
  // backward: remap_edge_bwd fused with remap_a4 for layer k
  struct D5 { double g, q0, q1, e0, e1; };
  pipelined<FV3B_RM_PF, D5>(
      nk,
      [&](int s) {
        const int k = nk - 1 - s;
        return D5{G[k * sk], __ldg(q[0] + k * sk), __ldg(q[1] + k * sk), o3[0][k * sk], o3[1][k * sk]};
      },
      [&](int s, const D5& v) {
        const int k = nk - 1 - s;
        const double qv[F] = {v.q0, v.q1}, ev[F] = {v.e0, v.e1};
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const double qek = ev[f] - v.g * qen[f];
          const double qc = qv[f];
          const double al = qek, ar_ = qen[f];
          const double ext = (ar_ - qc) * (qc - al);
          const double da1 = ar_ - al;
          const double a6 = 3.0 * (2.0 * qc - (al + ar_));
          const double a6da = a6 * da1;
          const double da2 = da1 * da1;
          const double v2 = (ext <= 0.0) ? qc : ((a6da > da2) ? 3.0 * qc - 2.0 * ar_ : al);
          const double v3 = (ext <= 0.0) ? qc : ((a6da < -da2) ? 3.0 * qc - 2.0 * al : ar_);
          if (f < nf) {
            o2[f][k * sk] = v2;
            o3[f][k * sk] = v3;
            o4[f][k * sk] = 3.0 * (2.0 * qc - (v2 + v3));
          }
          qen[f] = qek;
        }
      });
  return ar.ok;
}

constexpr int RM_COLS = 32, RM_TQ = 4;  // CTA: 32 columns x 4 tracers
#ifndef FV3B_RM_MINB
#define FV3B_RM_MINB 1
#endif

__global__ void __launch_bounds__(RM_COLS * RM_TQ, FV3B_RM_MINB) remap_kernel(const RemapArgs a) {
  const int cidx = blockIdx.x * RM_COLS + threadIdx.x;
  const int p = blockIdx.y * RM_TQ + threadIdx.y;  // field pair p: fields pair0[p] and pair0[p] + 1
  if (cidx >= a.ni * a.nj || p >= a.npair) return;
  const int t = a.pair0[p], n = a.pairn[p];
  const int i = cidx % a.ni, j = cidx / a.ni;
  // inputs are never written: a failed fast evaluation is simply redone
  if (!remap_column<true>(a, i, j, t, n)) remap_column<false>(a, i, j, t, n);
}

static int set_smem(const void* fn, size_t bytes) {
  // shared memory bounds how many column recurrences are in flight per SM:
  // take the whole 228 KB carve-out
  if ((bytes > 48 * 1024 &&
       cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) ||
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
    return check_launch("smem attribute");
  return FV3B_OK;
}

// Columns per CTA (<= 32, one warp) for a column kernel staging
// `bytes_per_col` of shared memory: maximise resident columns per SM with a
// CTA count that is a multiple of the 4 SM sub-partitions, so every warp
// scheduler owns the same number of recurrences.
static int cols_per_cta(size_t bytes_per_col, int64_t columns) {
  const size_t per_sm = 228 * 1024, reserved = 1024;
  const int sms = num_sms();
  const int64_t need = (columns + sms - 1) / sms;  // columns per SM for a single wave
  int best_cols = 1, best_total = 0;
  for (int m = 4; m <= 32; m += 4) {
    const size_t avail = per_sm / m;
    if (avail <= reserved) break;
    int cols = (int)((avail - reserved) / bytes_per_col);
    if (cols > NC_MAX) cols = NC_MAX;
    if (cols == NC_MAX && cols * m >= need) return NC_MAX;  // full warps, one wave
    if (cols >= 1 && cols * m > best_total) {
      best_total = cols * m;
      best_cols = cols;
    }
  }
  return best_cols;
}

int launch_riem(const RiemArgs& a, cudaStream_t st) {
#ifdef FV3B_RIEM_REGRING
  const size_t per_col = (size_t)(a.nk + 1) * sizeof(double);
#else
  const size_t per_col = (size_t)(a.nk + 1 + 3 * RD) * sizeof(double);  // S0 + the operand ring
#endif
  const int forced = tune_get(FV3B_TUNE_RIEM_COLS);
  const int nc = forced > 0 ? (forced < NC_MAX ? forced : NC_MAX) : cols_per_cta(per_col, (int64_t)a.ni_ext * a.nj_ext);
#ifdef FV3B_RIEM_REGRING
  const size_t bytes = per_col * nc;
#else
  const size_t bytes = (size_t)(a.nk + 1) * sizeof(double) * nc + RING * sizeof(double);
#endif
  FV3B_TRY(set_smem((const void*)riem_kernel, bytes));
  const int cols = a.ni_ext * a.nj_ext;
  riem_kernel<<<cdiv(cols, nc), nc, bytes, st>>>(a);
  return check_launch("riem_solver_c");
}

}  // namespace fv3b

using namespace fv3b;

// fields: dm, pt, w (layers), gz (interfaces), ws (2-D), pef, gz_out
// (interfaces; must not alias the inputs: gz_out and pef stage intermediates).  scalars: ptop, rdgas, grav, gama,
// p_fac, dt.  Domain nk = interface levels (program domain, nk_layers + 1).
extern "C" int fv3b_riem_solver_c(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                  void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || nf != 8 || ns != 6)
    return fail(FV3B_EINVAL, "fv3b_riem_solver_c: expects 8 fields, 6 scalars (got %d, %d)", nf, ns);
  if (d->nk < 4) return fail(FV3B_EDOMAIN, "fv3b_riem_solver_c: program domain nk=%d below minimum 4", d->nk);
  RiemArgs a;
  const Halo h0 = {0, 0, 0, 0, 0, 0};
  FV3B_TRY(view_of(f[0], 3, *d, h0, "dm", &a.dm));
  FV3B_TRY(view_of(f[1], 3, *d, h0, "pt", &a.pt));
  FV3B_TRY(view_of(f[2], 3, *d, h0, "w", &a.w));
  FV3B_TRY(view_of(f[3], 3, *d, h0, "gz", &a.gz));
  FV3B_TRY(view_of(f[4], 2, *d, h0, "ws", &a.ws));
  FV3B_TRY(view_of(f[5], 3, *d, h0, "pef", &a.pef));
  FV3B_TRY(view_of(f[6], 3, *d, h0, "gz_out", &a.gzo));
  FV3B_TRY(view_of(f[7], 3, *d, h0, "scratch", &a.scr));
  for (int t = 5; t < 8; ++t)
    for (int u = 0; u < 4; ++u)
      if (f[t].data == f[u].data) return fail(FV3B_EINVAL, "fv3b_riem_solver_c: output %d aliases input %d", t, u);
  if (a.dm.sk != a.pt.sk || a.dm.sk != a.w.sk || a.dm.sk != a.gz.sk)
    return fail(FV3B_ELAYOUT, "fv3b_riem_solver_c: input K strides differ");
  a.has_wout = false;
  a.ilo = 0;
  a.jlo = 0;
  a.ni_ext = d->ni;
  a.nj_ext = d->nj;
  a.nk = d->nk - 1;
  a.ptop = s[0]; a.rdgas = s[1]; a.grav = s[2]; a.gama = s[3]; a.p_fac = s[4]; a.dt = s[5];
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  return launch_riem(a, (cudaStream_t)stream);
}

// fields: delp, then per tracer t: q_t, a2_t, a3_t, a4_t.  Domain nk =
// interface levels (program domain).  No scalars.  Outputs must not alias
// the inputs (a2 / a3 stage the backward sweep's operands).
extern "C" int fv3b_remap_profile(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                  void* stream) {
  // groups of fields sharing a layer thickness: ns == 0 -> one group
  // (delp, 4 fields per tracer); else s[g] = fields in group g and the field
  // list is, per group, its thickness then 4 fields per member
  int ng = ns == 0 ? 1 : ns, cnt[16], total = 0;
  if (f == nullptr || d == nullptr || ns < 0 || ns > 16 || (ns > 0 && s == nullptr))
    return fail(FV3B_EINVAL, "fv3b_remap_profile: bad arguments");
  if (ns == 0) {
    if (nf < 5 || (nf - 1) % 4 != 0) return fail(FV3B_EINVAL, "fv3b_remap_profile: expects 1 + 4*nq fields");
    cnt[0] = (nf - 1) / 4;
  } else {
    for (int g = 0; g < ng; ++g) {
      cnt[g] = (int)s[g];
      if (cnt[g] < 1 || (double)cnt[g] != s[g]) return fail(FV3B_EINVAL, "fv3b_remap_profile: bad group size %g", s[g]);
    }
  }
  for (int g = 0; g < ng; ++g) total += cnt[g];
  if (total > 16 || nf != ng + 4 * total)
    return fail(FV3B_EINVAL, "fv3b_remap_profile: expects per group its thickness + 4 per field (<= 16 fields)");
  if (d->nk < 3) return fail(FV3B_EDOMAIN, "fv3b_remap_profile: program domain nk=%d below minimum 3", d->nk);
  // outputs never alias an input (any thickness or any q)
  bool input[4 * 16 + 16] = {};
  for (int g = 0, x = 0; g < ng; ++g) {
    input[x++] = true;
    for (int m = 0; m < cnt[g]; ++m, x += 4) input[x] = true;
  }
  for (int x = 0; x < nf; ++x)
    if (!input[x])
      for (int y = 0; y < nf; ++y)
        if (y != x && f[y].data == f[x].data)
          return fail(FV3B_EINVAL, "fv3b_remap_profile: output %d aliases field %d", x, y);
  RemapArgs a;
  const Halo h0 = {0, 0, 0, 0, 0, 0};
  a.nq = total;
  a.npair = 0;
  for (int g = 0, x = 0, t = 0; g < ng; ++g) {
    View dp;
    const int xd = x++;
    FV3B_TRY(view_of(f[xd], 3, *d, h0, "thickness", &dp));
    if (g == 0) a.delp = dp;
    if (dp.sj != a.delp.sj || dp.sk != a.delp.sk) return fail(FV3B_ELAYOUT, "fv3b_remap_profile: strides differ");
    for (int m = 0; m < cnt[g]; ++m, ++t) {
      View v[4];
      for (int u = 0; u < 4; ++u) FV3B_TRY(view_of(f[x + u], 3, *d, h0, "remap field", &v[u]));
      for (int u = 0; u < 4; ++u)
        if (v[u].sj != a.delp.sj || v[u].sk != a.delp.sk) return fail(FV3B_ELAYOUT, "fv3b_remap_profile: strides differ");
      a.dp[t] = dp.o;
      a.q[t] = v[0].o;
      a.a2[t] = v[1].o;
      a.a3[t] = v[2].o;
      a.a4[t] = v[3].o;
      if (m % 2 == 0) {
        a.pair0[a.npair] = t;
        a.pairn[a.npair++] = m + 1 < cnt[g] ? 2 : 1;
      }
      x += 4;
    }
  }
  a.sj = a.delp.sj;
  a.sk = a.delp.sk;
  a.ni = d->ni;
  a.nj = d->nj;
  a.nk = d->nk - 1;
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  dim3 grid(cdiv(a.ni * a.nj, RM_COLS), cdiv(a.npair, RM_TQ));
  remap_kernel<<<grid, dim3(RM_COLS, RM_TQ), 0, (cudaStream_t)stream>>>(a);
  return check_launch("remap_profile");
}

// ---------------------------------------------------------------------------
// remap mapping (oracle/remap_map.py; FV3 map1_ppm, the Lagrangian-to-
// Eulerian step after remap_profile).  A CTA owns 32 columns and all tracers
// (threadIdx.y strides over them).  Every warp stages delp and ak / bk; one
// thread per column forms the Lagrangian interfaces pe1 (ptop + running sum
// of delp), then every thread the target interfaces pe2 = ak + bk * ps, in
// shared memory (the search over source layers is data dependent).  Each
// (column, tracer) thread then runs map1_ppm over its column.  delp is
// rewritten in place with the pe2 differences after the last barrier (all of
// the CTA's reads of it are done, and no other CTA reads these columns).
// Measured alternatives, all slower at C2 (0.35 ms): a per-column index
// pass + (tracer, level)-parallel evaluation (0.38-0.52 ms), a single
// streaming pass per (column, tracer) with a prefetch ring (0.76 ms).
// ---------------------------------------------------------------------------
namespace fv3b {

struct RemapMapArgs {
  View delp, ak, bk;           // delp: the first group's thickness (strides shared)
  double* thick[16];           // per group: its thickness (rewritten with the pe2 differences)
  int gfirst[17];              // group g maps fields gfirst[g] .. gfirst[g+1]-1
  bool glog[16];               // group g maps in log pressure: thick[g] = log(pe1), lnpe2[g] = log(pe2)
  const double* lnpe2[16];
  int ngroup;
  int ncb;                     // blocks of 32 columns per CTA
  const double* q[16];
  const double* a2[16];
  const double* a3[16];
  const double* a4[16];
  double* qo[16];
  int64_t sj, sk;
  int nq, ni, nj, nk;  // nk layers
};

// fields per thread (kernel template): 4 for wide groups, 2 for narrow ones
// (measured: 4-5 best for the 10 scalar fields, 2 for the single-field wind
// groups, whose threads then carry no second field)
constexpr int MP_COLS = 32, MP_TY = 16;  // blockDim.y = min(ceil(nq / MP_F), MP_TY)
constexpr double MP_R3 = 1.0 / 3.0, MP_R23 = 2.0 / 3.0;  // the oracle's R3, R23 (same roundings)

// map1_ppm in log pressure for one field per thread (a log group, FV3's pt
// with kord_tm < 0): the source and target interfaces are the precomputed
// log(pe1), log(pe2) (fv3b_log_thickness), read per level; the cursor walk
// and every expression are remap_map_kernel's (oracle/remap_map.py
// map_columns on log_edges).
__device__ __forceinline__ void map_log_column(const double* __restrict__ l1, const double* __restrict__ l2,
                                               const double* __restrict__ q, const double* __restrict__ a2,
                                               const double* __restrict__ a3, const double* __restrict__ a4,
                                               double* qo, int nk, int64_t sk) {
  // the next source interface, the next target interface and the next
  // layer's coefficients are loaded one step ahead, so the cursor walk never
  // waits on a load (the linear kernel's running-sum prefetch)
  int k1 = 0;
  double pk = __ldg(l1), pn = __ldg(l1 + sk), pnn = __ldg(l1 + min(2, nk) * sk);
  double top = __ldg(l2), bot = __ldg(l2 + sk);
  double b2 = __ldg(a2), b3 = __ldg(a3), b4 = __ldg(a4);
  const int k1n = nk > 1 ? 1 : 0;
  double n2 = __ldg(a2 + k1n * sk), n3 = __ldg(a3 + k1n * sk), n4 = __ldg(a4 + k1n * sk);
  auto advance_to = [&](int m, double pm, double pm1) {  // the cursor moves to source layer m
    k1 = m;
    pk = pm;
    pn = pm1;
    pnn = __ldg(l1 + min(m + 2, nk) * sk);
    b2 = __ldg(a2 + m * sk);
    b3 = __ldg(a3 + m * sk);
    b4 = __ldg(a4 + m * sk);
    const int mn = m + 1 < nk ? m + 1 : m;
    n2 = __ldg(a2 + mn * sk);
    n3 = __ldg(a3 + mn * sk);
    n4 = __ldg(a4 + mn * sk);
  };
  for (int k2 = 0; k2 < nk; ++k2) {
    const double botn = __ldg(l2 + min(k2 + 2, nk) * sk);
    while (top > pn && k1 < nk - 1) {
      ++k1;
      pk = pn;
      pn = pnn;
      pnn = __ldg(l1 + min(k1 + 2, nk) * sk);
      b2 = n2;
      b3 = n3;
      b4 = n4;
      const int mn = k1 + 1 < nk ? k1 + 1 : k1;
      n2 = __ldg(a2 + mn * sk);
      n3 = __ldg(a3 + mn * sk);
      n4 = __ldg(a4 + mn * sk);
    }
    const double d = pn - pk;
    const double pl = (top - pk) / d;
    if (bot <= pn) {
      const double pr = (bot - pk) / d;
      qo[k2 * sk] = b2 + 0.5 * (b4 + b3 - b2) * (pr + pl) - b4 * MP_R3 * (pr * (pr + pl) + pl * pl);
    } else {
      double qsum = (pn - top) * (b2 + 0.5 * (b4 + b3 - b2) * (1.0 + pl) - b4 * (MP_R3 * (1.0 + pl * (1.0 + pl))));
      double pm = pn;
      for (int m = k1 + 1; m < nk; ++m) {
        const double pm1 = m == k1 + 1 ? pnn : __ldg(l1 + (m + 1) * sk);
        const double dm = pm1 - pm;
        if (bot > pm1) {
          qsum = qsum + dm * __ldg(q + m * sk);
          pm = pm1;
        } else {
          const double dp = bot - pm;
          const double esl = dp / dm;
          const double c2 = __ldg(a2 + m * sk);
          qsum = qsum + dp * (c2 + 0.5 * esl * (__ldg(a3 + m * sk) - c2 + __ldg(a4 + m * sk) * (1.0 - MP_R23 * esl)));
          advance_to(m, pm, pm1);
          break;
        }
      }
      qo[k2 * sk] = qsum / (bot - top);
    }
    top = bot;
    bot = botn;
  }
}

// LG: the launch has log-pressure groups (their CTAs take map_log_column;
// kept out of the other instantiations, whose registers it would raise)
template <int MP_F, bool LG>
__global__ void __launch_bounds__(MP_COLS * MP_TY) remap_map_kernel(const RemapMapArgs a) {
  // map1_ppm's walk over the source layers only moves downwards, so the
  // Lagrangian interfaces pe1 are produced by a running sum as it advances
  // (the same additions in the same order as pe1[k+1] = pe1[k] + delp[k]):
  // no per-column level arrays in shared memory, occupancy bounded by
  // registers only.  ps = pe1[nk] comes from a first pass over the column.
  extern __shared__ double sm[];  // ak, bk [nk + 1]
  // threadIdx.y = (column block, field thread): a.ncb blocks of 32 columns,
  // blockDim.y / a.ncb field threads per column
  const int c = threadIdx.x, ny = blockDim.y / a.ncb, ty = threadIdx.y % ny, cb = threadIdx.y / ny;
  const int cidx = (blockIdx.x * a.ncb + cb) * MP_COLS + c;
  const bool live = cidx < a.ni * a.nj;
  const int nk = a.nk;
  const int i = live ? cidx % a.ni : 0, j = live ? cidx / a.ni : 0;
  const int64_t off = i + (int64_t)j * a.sj, sk = a.sk;
  const int grp = blockIdx.y;
  if (LG && a.glog[grp]) {  // a log-pressure group: its interface pair, one field per thread, nothing rewritten
    const double* l1 = a.thick[grp] + off;
    const double* l2 = a.lnpe2[grp] + off;
    if (live)
      for (int t = a.gfirst[grp] + threadIdx.y % (blockDim.y / a.ncb); t < a.gfirst[grp + 1]; t += blockDim.y / a.ncb)
        map_log_column(l1, l2, a.q[t] + off, a.a2[t] + off, a.a3[t] + off, a.a4[t] + off, a.qo[t] + off, a.nk, a.sk);
    return;
  }
  double* thick = a.thick[grp] + off;
  double* AK = sm;
  double* BK = sm + (nk + 1);
  for (int e = c + threadIdx.y * MP_COLS; e <= nk; e += MP_COLS * blockDim.y) {
    AK[e] = __ldg(a.ak.o + e * a.ak.sk);
    BK[e] = __ldg(a.bk.o + e * a.bk.sk);
  }
  __syncthreads();
  auto th = [&](int k) { return thick[k * sk]; };  // (rewritten at the end: plain loads)
  double ps = AK[0];
  if (live)
    for (int k = 0; k < nk; ++k) ps = ps + th(k);
  // pe2 = ak + bk * ps, the end interfaces from pe1 (pe1[0] = ak[0])
  auto p2 = [&](int k) { return k == 0 ? AK[0] : (k == nk ? ps : AK[k] + BK[k] * ps); };
  const int tb = a.gfirst[grp], te = a.gfirst[grp + 1];
  if (live)
    for (int t0 = tb + ty; t0 < te; t0 += ny * MP_F) {
      const double* Q[MP_F];
      const double* A2[MP_F];
      const double* A3[MP_F];
      const double* A4[MP_F];
      double* QO[MP_F];
      bool on[MP_F];
#pragma unroll
      for (int f = 0; f < MP_F; ++f) {
        const int t = t0 + f * ny;
        on[f] = t < te;
        const int tt = on[f] ? t : t0;
        Q[f] = a.q[tt] + off;
        A2[f] = a.a2[tt] + off;
        A3[f] = a.a3[tt] + off;
        A4[f] = a.a4[tt] + off;
        QO[f] = a.qo[tt] + off;
      }
      // cursor: source layer k1 with pk = pe1[k1], pn = pe1[k1 + 1]; tn =
      // th(k1 + 1) is loaded one advance ahead, so the search never waits on
      // the thickness load of the layer it steps into
      int k1 = 0;
      double pk = AK[0], pn = pk + th(0);
      double tn = th(nk > 1 ? 1 : 0);
      // narrow groups (MP_F <= 2): the profile coefficients of layer k1 (b*)
      // and k1 + 1 (n*, loaded one advance ahead) stay in registers while the
      // cursor stays put (winds 0.187 -> 0.162 ms); the wide groups reload
      // them per target layer (L1 hits), as their registers would spill
      constexpr bool CACHE = MP_F <= 2;
      double b2[MP_F], b3[MP_F], b4[MP_F], n2[CACHE ? MP_F : 1], n3[CACHE ? MP_F : 1], n4[CACHE ? MP_F : 1];
      auto coef = [&](int k, double* c2, double* c3, double* c4) {
#pragma unroll
        for (int f = 0; f < MP_F; ++f) {
          c2[f] = __ldg(A2[f] + k * sk);
          c3[f] = __ldg(A3[f] + k * sk);
          c4[f] = __ldg(A4[f] + k * sk);
        }
      };
      if constexpr (CACHE) {
        coef(0, b2, b3, b4);
        coef(nk > 1 ? 1 : 0, n2, n3, n4);
      }
      for (int k2 = 0; k2 < nk; ++k2) {
        const double top = p2(k2), bot = p2(k2 + 1);
        while (top > pn && k1 < nk - 1) {
          ++k1;
          pk = pn;
          pn = pk + tn;
          tn = th(k1 + 1 < nk ? k1 + 1 : k1);
          if constexpr (CACHE) {
#pragma unroll
            for (int f = 0; f < MP_F; ++f) {
              b2[f] = n2[f];
              b3[f] = n3[f];
              b4[f] = n4[f];
            }
            coef(k1 + 1 < nk ? k1 + 1 : k1, n2, n3, n4);
          }
        }
        if constexpr (!CACHE) coef(k1, b2, b3, b4);
        const double d = pn - pk;
        const double pl = (top - pk) / d;
        if (bot <= pn) {  // the whole target layer lies in source layer k1
          const double pr = (bot - pk) / d;
#pragma unroll
          for (int f = 0; f < MP_F; ++f)
            if (on[f])
              QO[f][k2 * sk] = b2[f] + 0.5 * (b4[f] + b3[f] - b2[f]) * (pr + pl) -
                               b4[f] * MP_R3 * (pr * (pr + pl) + pl * pl);
        } else {  // the rest of k1, whole source layers, then part of the last one
          double qsum[MP_F];
#pragma unroll
          for (int f = 0; f < MP_F; ++f)
            qsum[f] = (pn - top) * (b2[f] + 0.5 * (b4[f] + b3[f] - b2[f]) * (1.0 + pl) -
                                    b4[f] * (MP_R3 * (1.0 + pl * (1.0 + pl))));
          double pm = pn;  // pe1[m]
          for (int m = k1 + 1; m < nk; ++m) {
            const double pm1 = pm + (m == k1 + 1 ? tn : th(m));  // pe1[m + 1]
            const double dm = pm1 - pm;
            if (bot > pm1) {
#pragma unroll
              for (int f = 0; f < MP_F; ++f) qsum[f] = qsum[f] + dm * __ldg(Q[f] + m * sk);
              pm = pm1;
            } else {
              const double dp = bot - pm;
              const double esl = dp / dm;
#pragma unroll
              for (int f = 0; f < MP_F; ++f) {
                const double c2 = __ldg(A2[f] + m * sk);
                qsum[f] = qsum[f] + dp * (c2 + 0.5 * esl * (__ldg(A3[f] + m * sk) - c2 +
                                                           __ldg(A4[f] + m * sk) * (1.0 - MP_R23 * esl)));
              }
              k1 = m;  // the next target layer starts in this one
              pk = pm;
              pn = pm1;
              tn = th(m + 1 < nk ? m + 1 : m);
              if constexpr (CACHE) {
                coef(m, b2, b3, b4);
                coef(m + 1 < nk ? m + 1 : m, n2, n3, n4);
              }
              break;
            }
          }
#pragma unroll
          for (int f = 0; f < MP_F; ++f)
            if (on[f]) QO[f][k2 * sk] = qsum[f] / (bot - top);
        }
      }
    }
  __syncthreads();  // every walk of the CTA has read the thickness
  if (live && ty == 0)
    for (int k = 0; k < nk; ++k) thick[k * sk] = p2(k + 1) - p2(k);
}

}  // namespace fv3b

// fields: delp (3-D, rewritten in place), ak, bk (K, nk+1 target
// coefficients), then per tracer t: q_t, a4_2_t, a4_3_t, a4_4_t (remap_profile
// outputs), q_out_t.  Domain nk = interface levels.  Grouped form: s[g] =
// fields in group g, negative for a group mapped in log pressure, whose
// thickness slot holds log(pe1) followed by log(pe2) (interfaces,
// fv3b_log_thickness; nothing is rewritten).
extern "C" int fv3b_remap_map(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                              void* stream) {
  // ns == 0: delp, ak, bk, then 5 fields per tracer (one group).  ns >= 1:
  // groups of fields sharing a thickness, s[g] = fields in group g; the field
  // list is ak, bk, then per group its thickness and 5 per member.
  int ng = ns == 0 ? 1 : ns, cnt[16], total = 0;
  if (f == nullptr || d == nullptr || ns < 0 || ns > 16 || (ns > 0 && s == nullptr))
    return fail(FV3B_EINVAL, "fv3b_remap_map: bad arguments");
  if (ns == 0) {
    if (nf < 8 || (nf - 3) % 5 != 0) return fail(FV3B_EINVAL, "fv3b_remap_map: expects 3 + 5*nq fields");
    cnt[0] = (nf - 3) / 5;
  } else {
    for (int g = 0; g < ng; ++g) {
      cnt[g] = (int)(s[g] < 0 ? -s[g] : s[g]);  // negative: a log-pressure group
      if (cnt[g] < 1 || (double)cnt[g] != (s[g] < 0 ? -s[g] : s[g]))
        return fail(FV3B_EINVAL, "fv3b_remap_map: bad group size %g", s[g]);
    }
  }
  int nlog = 0;
  for (int g = 0; g < ng; ++g) {
    total += cnt[g];
    nlog += ns > 0 && s[g] < 0;
  }
  if (total > 16 || nf != 2 + ng + nlog + 5 * total)
    return fail(FV3B_EINVAL,
                "fv3b_remap_map: expects ak, bk, per group its thickness (log groups: log(pe1), log(pe2)) and 5 per "
                "field (<= 16 fields)");
  if (d->nk < 2 || d->nk > 4096)
    return fail(FV3B_EDOMAIN, "fv3b_remap_map: program domain nk=%d outside [2, 4096]", d->nk);
  // field-list positions: thickness of group g, ak, bk, field t's five
  int xthick[16], xfield[16];
  int xak, xbk;
  if (ns == 0) {
    xthick[0] = 0;
    xak = 1;
    xbk = 2;
    for (int t = 0; t < total; ++t) xfield[t] = 3 + 5 * t;
  } else {
    xak = 0;
    xbk = 1;
    for (int g = 0, x = 2, t = 0; g < ng; ++g) {
      xthick[g] = x++;
      if (s[g] < 0) ++x;  // log(pe2) follows log(pe1)
      for (int m = 0; m < cnt[g]; ++m, ++t, x += 5) xfield[t] = x;
    }
  }
  RemapMapArgs a;
  const Halo h0 = {0, 0, 0, 0, 0, 0};
  FV3B_TRY(view_of(f[xthick[0]], 3, *d, h0, "delp", &a.delp));
  FV3B_TRY(view_of(f[xak], 1, *d, h0, "ak", &a.ak));
  FV3B_TRY(view_of(f[xbk], 1, *d, h0, "bk", &a.bk));
  a.nq = total;
  a.ngroup = ng;
  for (int g = 0; g < ng; ++g) {
    a.glog[g] = ns > 0 && s[g] < 0;
    a.lnpe2[g] = nullptr;
    if (a.glog[g]) {
      View v;
      FV3B_TRY(view_of(f[xthick[g] + 1], 3, *d, h0, "log(pe2)", &v));
      if (v.sj != a.delp.sj || v.sk != a.delp.sk) return fail(FV3B_ELAYOUT, "fv3b_remap_map: strides differ");
      a.lnpe2[g] = v.o;
    }
  }
  for (int g = 0, t = 0; g < ng; ++g) {
    View v;
    FV3B_TRY(view_of(f[xthick[g]], 3, *d, h0, "thickness", &v));
    if (v.sj != a.delp.sj || v.sk != a.delp.sk) return fail(FV3B_ELAYOUT, "fv3b_remap_map: strides differ");
    a.thick[g] = v.o;
    a.gfirst[g] = t;
    t += cnt[g];
    a.gfirst[g + 1] = t;
  }
  for (int t = 0; t < total; ++t) {
    View v[5];
    for (int u = 0; u < 5; ++u) FV3B_TRY(view_of(f[xfield[t] + u], 3, *d, h0, "remap_map field", &v[u]));
    for (int u = 0; u < 5; ++u)
      if (v[u].sj != a.delp.sj || v[u].sk != a.delp.sk) return fail(FV3B_ELAYOUT, "fv3b_remap_map: strides differ");
    a.q[t] = v[0].o;
    a.a2[t] = v[1].o;
    a.a3[t] = v[2].o;
    a.a4[t] = v[3].o;
    a.qo[t] = v[4].o;
  }
  for (int t = 0; t < total; ++t) {  // q_out never aliases another field
    const int x = xfield[t] + 4;
    for (int g = 0; g < nf; ++g)
      if (g != x && f[g].data == f[x].data) return fail(FV3B_EINVAL, "fv3b_remap_map: q_out%d aliases field %d", t, g);
  }
  a.sj = a.delp.sj;
  a.sk = a.delp.sk;
  a.ni = d->ni;
  a.nj = d->nj;
  a.nk = d->nk - 1;
  if (d->ni <= 0 || d->nj <= 0) return FV3B_OK;
  int maxc = 1;
  for (int g = 0; g < ng; ++g) maxc = cnt[g] > maxc ? cnt[g] : maxc;
  const int F = maxc >= 4 ? 4 : 2;
  const int ty = cdiv(maxc, F) < MP_TY ? cdiv(maxc, F) : MP_TY;
  a.ncb = ty >= 4 ? 1 : 4 / ty;  // at least 4 warps per CTA
  const size_t bytes = (size_t)2 * (a.nk + 1) * sizeof(double);
  bool anylog = false;
  for (int g = 0; g < ng; ++g) anylog = anylog || a.glog[g];
  const void* kern = F == 4 ? (anylog ? (const void*)remap_map_kernel<4, true> : (const void*)remap_map_kernel<4, false>)
                            : (anylog ? (const void*)remap_map_kernel<2, true> : (const void*)remap_map_kernel<2, false>);
  if (bytes > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return check_launch("remap_map smem attribute");
  dim3 grid(cdiv(a.ni * a.nj, MP_COLS * a.ncb), ng), block(MP_COLS, ty * a.ncb);
  if (F == 4 && anylog)
    remap_map_kernel<4, true><<<grid, block, bytes, (cudaStream_t)stream>>>(a);
  else if (F == 4)
    remap_map_kernel<4, false><<<grid, block, bytes, (cudaStream_t)stream>>>(a);
  else if (anylog)
    remap_map_kernel<2, true><<<grid, block, bytes, (cudaStream_t)stream>>>(a);
  else
    remap_map_kernel<2, false><<<grid, block, bytes, (cudaStream_t)stream>>>(a);
  return check_launch("remap_map");
}
