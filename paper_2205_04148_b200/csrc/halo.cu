// K6 halo_update, on-device parts.
//
//  * fv3b_halo_periodic: fills the I/J halo of every field of a doubly
//    periodic single-rank domain in one launch (corners included);
//  * fv3b_halo_pack / fv3b_halo_unpack: copy the edge strips of a batch of
//    fields to / from one contiguous message buffer for the neighbour
//    exchange of a decomposed domain (NCCL P2P moves the buffers).  A strip
//    is a rectangle [i0, i0+w) x [j0, j0+h) x all levels of every field;
//    buffer layout is field-major, then level, row, column.
#include <string.h>

#include "common.cuh"

namespace fv3b {

constexpr int HALO_MAXF = 32;
#ifndef FV3B_HALO_KU  // levels per thread of the periodic fill (tools/build_variant.py sweeps)
#define FV3B_HALO_KU 8
#endif

struct HaloArgs {
  double* o[HALO_MAXF];  // interior origins
  int64_t sj, sk;
  int levels[HALO_MAXF];  // levels to process per field (1 for 2-D)
  int nf, ni, nj, h;
};

// One thread per halo cell of a level: e enumerates the ring [-h, n+h)^2
// minus the interior (the south and north bands of full width, then the west
// and east bands of the interior rows); source = periodic wrap.
__global__ void halo_periodic_kernel(const HaloArgs a) {
  // each thread copies one ring cell on HALO_KU consecutive levels: the
  // independent loads are issued together (the copy is latency-bound)
  constexpr int HALO_KU = FV3B_HALO_KU;
  const int W = a.ni + 2 * a.h, h = a.h;
  const int f = blockIdx.z, kb = blockIdx.y * HALO_KU;
  const int nl = min(HALO_KU, a.levels[f] - kb);
  if (nl <= 0) return;
  double* o = a.o[f] + (int64_t)kb * a.sk;
  const int nband = W * h;           // one south / north band
  const int nside = h * a.nj;        // one west / east band
  const int n = 2 * nband + 2 * nside;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    int i, j;
    if (e < 2 * nband) {
      const int b = e / nband, r = e % nband;
      i = r % W - h;
      j = (b == 0 ? -h : a.nj) + r / W;
    } else {
      const int r0 = e - 2 * nband, b = r0 / nside, r = r0 % nside;
      i = (b == 0 ? -h : a.ni) + r % h;
      j = r / h;
    }
    const int si = (i + a.ni) % a.ni, sj = (j + a.nj) % a.nj;
    const int64_t dst = i + (int64_t)j * a.sj, src = si + (int64_t)sj * a.sj;
    double v[HALO_KU];
#pragma unroll
    for (int k = 0; k < HALO_KU; ++k)
      if (k < nl) v[k] = o[src + k * a.sk];
#pragma unroll
    for (int k = 0; k < HALO_KU; ++k)
      if (k < nl) o[dst + k * a.sk] = v[k];
  }
}

struct StripArgs {
  double* o[HALO_MAXF];
  int64_t sj, sk;
  int levels[HALO_MAXF];
  int64_t off[HALO_MAXF];  // element offset of each field's strip in the buffer
  double* buf;
  int nf, i0, j0, w, h;
  bool unpack;
};

__global__ void strip_kernel(const StripArgs a) {
  const int f = blockIdx.z, k = blockIdx.y;
  if (k >= a.levels[f]) return;
  const int n = a.w * a.h;
  double* o = a.o[f] + (int64_t)k * a.sk;
  double* b = a.buf + a.off[f] + (int64_t)k * n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int i = a.i0 + e % a.w, j = a.j0 + e / a.w;
    double* p = o + i + (int64_t)j * a.sj;
    if (a.unpack)
      *p = b[e];
    else
      b[e] = *p;
  }
}

static int collect(const fv3b_field* f, int nf, const fv3b_domain* d, int h, double** o, int* levels, int64_t* sj,
                   int64_t* sk) {
  if (nf < 1 || nf > HALO_MAXF) return fail(FV3B_EINVAL, "halo: 1..%d fields per call (got %d)", HALO_MAXF, nf);
  *sj = 0;
  *sk = 0;
  for (int t = 0; t < nf; ++t) {
    View v;
    const Halo hh = {h, h, h, h, 0, 0};
    fv3b_domain dd = *d;
    dd.nk = 0;
    FV3B_TRY(view_of(f[t], f[t].rank, dd, hh, "halo field", &v));
    if (f[t].rank == 3) {
      if (*sk == 0) *sk = v.sk;
      if (v.sk != *sk) return fail(FV3B_ELAYOUT, "halo: 3-D fields must share strides");
    }
    if (*sj == 0) *sj = v.sj;
    if (v.sj != *sj) return fail(FV3B_ELAYOUT, "halo: fields must share the J stride");
    o[t] = v.o;
    levels[t] = f[t].rank == 3 ? f[t].shape[2] : 1;
  }
  return FV3B_OK;
}


// A device buffer passed as a rank-1 field: data = its address, shape[0] =
// its capacity in elements of its type (doubles for message buffers, int32
// for index lists, 64-bit words for barrier flags).
static int buffer_of(const fv3b_field& f, int64_t need, const char* what, void** out) {
  if (f.rank != 1 || f.data == nullptr)
    return fail(FV3B_EINVAL, "%s: expects a rank-1 buffer field with a non-null address", what);
  if ((int64_t)f.shape[0] < need)
    return fail(FV3B_EINVAL, "%s: buffer holds %d elements, the call needs %lld", what, f.shape[0], (long long)need);
  *out = f.data;
  return FV3B_OK;
}

// ---------------------------------------------------------------------------
// Multi-rectangle pack / unpack: every edge / corner strip of a halo update
// for a batch of fields in one launch (the decomposed-domain exchange,
// parallel.DecomposedHalo).  Rectangle r of field t at level k lives at
// buf[off_r + ((t * L) + k) * w_r * h_r + row * w_r + col], L = the fields'
// level count (all fields of a call share it).
// ---------------------------------------------------------------------------
constexpr int RECT_MAX = 8;

struct RectArgs {
  double* o[HALO_MAXF];
  int64_t sj, sk;
  double* buf;
  int i0[RECT_MAX], j0[RECT_MAX], w[RECT_MAX], h[RECT_MAX];
  int64_t off[RECT_MAX];
  int nrect, nf, levels;
  bool unpack;
};

__global__ void rects_kernel(const RectArgs a) {
  const int r = blockIdx.z % a.nrect, t = blockIdx.z / a.nrect, k = blockIdx.y;
  const int w = a.w[r], n = w * a.h[r];
  double* o = a.o[t] + (int64_t)k * a.sk;
  double* b = a.buf + a.off[r] + ((int64_t)t * a.levels + k) * n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double* p = o + (a.i0[r] + e % w) + (int64_t)(a.j0[r] + e / w) * a.sj;
    if (a.unpack)
      *p = b[e];
    else
      b[e] = *p;
  }
}

static int rects_call(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream,
                      bool unpack) {
  // fields: the halo fields, then the message buffer (a buffer field);
  // scalars: [nrect, (i0, j0, w, h, offset) x nrect]
  if (f == nullptr || d == nullptr || s == nullptr || ns < 1 || nf < 2)
    return fail(FV3B_EINVAL, "halo rects: bad arguments");
  RectArgs a;
  a.nrect = (int)s[0];
  if (a.nrect < 1 || a.nrect > RECT_MAX || ns != 1 + 5 * a.nrect)
    return fail(FV3B_EINVAL, "halo rects: 1..%d rectangles, 1 + 5*n scalars", RECT_MAX);
  --nf;
  int levels[HALO_MAXF];
  FV3B_TRY(collect(f, nf, d, 0, a.o, levels, &a.sj, &a.sk));
  for (int t = 1; t < nf; ++t)
    if (levels[t] != levels[0]) return fail(FV3B_EINVAL, "halo rects: fields must share their level count");
  a.levels = levels[0];
  a.nf = nf;
  a.unpack = unpack;
  int maxn = 1;
  int64_t need = 0;
  for (int r = 0; r < a.nrect; ++r) {
    const double* q = s + 1 + 5 * r;
    a.i0[r] = (int)q[0];
    a.j0[r] = (int)q[1];
    a.w[r] = (int)q[2];
    a.h[r] = (int)q[3];
    a.off[r] = (int64_t)q[4];
    if (a.w[r] <= 0 || a.h[r] <= 0 || a.off[r] < 0) return fail(FV3B_EINVAL, "halo rects: empty rectangle %d", r);
    maxn = a.w[r] * a.h[r] > maxn ? a.w[r] * a.h[r] : maxn;
    const int64_t end = a.off[r] + (int64_t)nf * a.levels * a.w[r] * a.h[r];
    need = end > need ? end : need;
  }
  void* buf;
  FV3B_TRY(buffer_of(f[nf], need, "halo rects", &buf));
  a.buf = static_cast<double*>(buf);
  dim3 grid(cdiv(maxn, 256) < 16 ? cdiv(maxn, 256) : 16, a.levels, a.nrect * nf);
  rects_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch(unpack ? "fv3b_halo_unpack_rects" : "fv3b_halo_pack_rects");
}

// ---------------------------------------------------------------------------
// Peer-memory strip copies: the decomposed-domain halo update without
// message buffers (parallel.PeerHalo).  Each rectangle of each field goes
// straight from the source field to a destination field that may live in
// another rank's allocation (a CUDA-IPC / peer mapping over NVLink, or
// another block on the same device): the sender's edge strip is stored
// into the neighbour's halo (posted stores over NVLink), replacing pack +
// ncclSend/ncclRecv + unpack with one launch per rank.
// ---------------------------------------------------------------------------
constexpr int PEER_MAXF = HALO_MAXF;

struct PeerArgs {
  const double* src[PEER_MAXF];
  double* dst[RECT_MAX][PEER_MAXF];
  int64_t sj, sk;
  int si0[RECT_MAX], sj0[RECT_MAX], di0[RECT_MAX], dj0[RECT_MAX], w[RECT_MAX], h[RECT_MAX];
  int nrect, nf;
};

__global__ void peer_kernel(const PeerArgs a) {
  const int r = blockIdx.z % a.nrect, t = blockIdx.z / a.nrect, k = blockIdx.y;
  const int w = a.w[r], n = w * a.h[r];
  const double* s = a.src[t] + (int64_t)k * a.sk + a.si0[r] + (int64_t)a.sj0[r] * a.sj;
  double* o = a.dst[r][t] + (int64_t)k * a.sk + a.di0[r] + (int64_t)a.dj0[r] * a.sj;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int64_t off = e % w + (int64_t)(e / w) * a.sj;
    o[off] = s[off];
  }
}

static int peer_call(const fv3b_field* f, int ntot, const double* s, int ns, const fv3b_domain* d, void* stream) {
  // scalars: [nf, nrect, (src i0, src j0, dst i0, dst j0, w, h) x nrect]
  // fields: nf sources, then rectangle r's destination of field t at nf + r*nf + t
  if (f == nullptr || d == nullptr || s == nullptr || ns < 2) return fail(FV3B_EINVAL, "halo peer: bad arguments");
  PeerArgs a;
  a.nf = (int)s[0];
  a.nrect = (int)s[1];
  if (a.nf < 1 || a.nf > PEER_MAXF || a.nrect < 1 || a.nrect > RECT_MAX || ns != 2 + 6 * a.nrect ||
      ntot != a.nf * (1 + a.nrect))
    return fail(FV3B_EINVAL, "halo peer: 1..%d fields, 1..%d rectangles, 2 + 6*nrect scalars, nf*(1+nrect) fields",
                PEER_MAXF, RECT_MAX);
  int levels[PEER_MAXF], lv[PEER_MAXF];
  double* o[PEER_MAXF];
  FV3B_TRY(collect(f, a.nf, d, 0, o, levels, &a.sj, &a.sk));
  for (int t = 0; t < a.nf; ++t) a.src[t] = o[t];
  for (int r = 0; r < a.nrect; ++r) {
    int64_t sj, sk;
    FV3B_TRY(collect(f + a.nf * (1 + r), a.nf, d, 0, a.dst[r], lv, &sj, &sk));
    if (sj != a.sj || sk != a.sk) return fail(FV3B_ELAYOUT, "halo peer: destinations must share the sources' strides");
    for (int t = 0; t < a.nf; ++t)
      if (lv[t] != levels[t] || levels[t] != levels[0])
        return fail(FV3B_EINVAL, "halo peer: fields must share their level count");
  }
  int maxn = 1;
  for (int r = 0; r < a.nrect; ++r) {
    const double* q = s + 2 + 6 * r;
    a.si0[r] = (int)q[0];
    a.sj0[r] = (int)q[1];
    a.di0[r] = (int)q[2];
    a.dj0[r] = (int)q[3];
    a.w[r] = (int)q[4];
    a.h[r] = (int)q[5];
    if (a.w[r] <= 0 || a.h[r] <= 0) return fail(FV3B_EINVAL, "halo peer: empty rectangle %d", r);
    maxn = a.w[r] * a.h[r] > maxn ? a.w[r] * a.h[r] : maxn;
  }
  dim3 grid(cdiv(maxn, 256) < 16 ? cdiv(maxn, 256) : 16, levels[0], a.nrect * a.nf);
  peer_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch("fv3b_halo_peer_rects");
}

// ---------------------------------------------------------------------------
// Peer-memory index-list stores: the cubed-sphere halo update without
// message buffers (cubesphere.CubePeerHalo).  Destination set d is one
// neighbour tile's fields (peer-mapped) or this tile's own (the corner
// fill); entry s of its list is (source slot, source offset, destination
// slot, destination offset, sign), offsets interior-relative, so each
// rotated / component-swapped / sign-flipped halo cell is one load from this
// tile and one store into the neighbour, all levels of up to 32 fields.
// ---------------------------------------------------------------------------
struct PeerIdxArgs {
  const double* src[PEER_MAXF];
  double* dst[RECT_MAX][PEER_MAXF];
  const int* idx[RECT_MAX];
  int n[RECT_MAX];
  int64_t sk;
  int nset;
};

__global__ void peer_idx_kernel(const PeerIdxArgs a) {
  const int d = blockIdx.z, k = blockIdx.y;
  const int* idx = a.idx[d];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < a.n[d]; e += gridDim.x * blockDim.x) {
    const int* x = idx + 5 * e;
    const double v = a.src[x[0]][x[1] + (int64_t)k * a.sk];
    a.dst[d][x[2]][x[3] + (int64_t)k * a.sk] = x[4] < 0 ? -v : v;
  }
}

static int peer_idx_call(const fv3b_field* f, int ntot, const double* s, int ns, const fv3b_domain* d,
                         void* stream) {
  // scalars: [nf, nset]; fields: nf sources, then set r's destination of
  // slot t at nf + r*nf + t, then set r's index list (an int32 buffer
  // field of 5 entries per cell) at nf*(1+nset) + r
  if (f == nullptr || d == nullptr || s == nullptr || ns != 2) return fail(FV3B_EINVAL, "halo peer idx: bad arguments");
  PeerIdxArgs a;
  const int nf = (int)s[0];
  a.nset = (int)s[1];
  if (nf < 1 || nf > PEER_MAXF || a.nset < 1 || a.nset > RECT_MAX || ntot != nf * (1 + a.nset) + a.nset)
    return fail(FV3B_EINVAL, "halo peer idx: 1..%d fields, 1..%d sets, nf*(1+nset) fields + nset lists",
                PEER_MAXF, RECT_MAX);
  int levels[PEER_MAXF], lv[PEER_MAXF];
  double* o[PEER_MAXF];
  int64_t sj, sk;
  FV3B_TRY(collect(f, nf, d, 0, o, levels, &sj, &sk));
  for (int t = 0; t < nf; ++t) {
    a.src[t] = o[t];
    if (levels[t] != levels[0]) return fail(FV3B_EINVAL, "halo peer idx: fields must share their level count");
  }
  a.sk = sk;
  int maxn = 0;
  for (int r = 0; r < a.nset; ++r) {
    int64_t sj2, sk2;
    FV3B_TRY(collect(f + nf * (1 + r), nf, d, 0, a.dst[r], lv, &sj2, &sk2));
    if (sj2 != sj || sk2 != sk) return fail(FV3B_ELAYOUT, "halo peer idx: destinations must share the sources' strides");
    const fv3b_field& lf = f[nf * (1 + a.nset) + r];
    a.n[r] = lf.rank == 1 ? lf.shape[0] / 5 : -1;
    a.idx[r] = nullptr;
    if (a.n[r] < 0 || lf.shape[0] % 5 != 0) return fail(FV3B_EINVAL, "halo peer idx: list %d is not 5 int32 per entry", r);
    if (a.n[r] > 0) {
      void* p;
      FV3B_TRY(buffer_of(lf, 5 * (int64_t)a.n[r], "halo peer idx list", &p));
      a.idx[r] = static_cast<const int*>(p);
    }
    maxn = a.n[r] > maxn ? a.n[r] : maxn;
  }
  if (maxn == 0) return FV3B_OK;
  dim3 grid(cdiv(maxn, 256) < 32 ? cdiv(maxn, 256) : 32, levels[0], a.nset);
  peer_idx_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch("fv3b_halo_peer_idx");
}

// ---------------------------------------------------------------------------
// Stream-ordered barrier among a rank and its neighbours over peer-mapped
// flag words (parallel.FlagSync): one thread bumps (or reads) this rank's
// update counter e, stores e with release semantics into the flag word it
// owns in every neighbour's flag array, then spins (acquire loads, nanosleep
// back-off) until every neighbour has stored >= e into this rank's array.
// No host synchronisation, so a PeerHalo update is three stream-ordered
// launches (arrive barrier, peer stores, stored barrier) and can be captured
// in a CUDA graph.  The spin is bounded (10 s of globaltimer): a neighbour
// that never arrives sets *err and traps (the context reports the failure)
// instead of hanging the device or continuing on a torn halo.
// ---------------------------------------------------------------------------
struct SigArgs {
  unsigned long long* epoch;
  unsigned long long* remote[RECT_MAX];  // my word in each neighbour's array
  unsigned long long* local[RECT_MAX];   // each neighbour's word in my array
  int* err;
  int npeer, bump;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void signal_wait_kernel(const SigArgs a) {
  if (threadIdx.x != 0) return;
  unsigned long long e = *a.epoch;
  if (a.bump) *a.epoch = ++e;
  __threadfence_system();  // this stream's earlier writes (peer stores included) before the flags
  for (int p = 0; p < a.npeer; ++p)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.remote[p]), "l"(e) : "memory");
  const unsigned long long t0 = global_ns();
  for (int p = 0; p < a.npeer; ++p) {
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.local[p]) : "memory");
      if (v >= e) break;
      if (global_ns() - t0 > 10000000000ull) {
        // fail loudly: a neighbour never arrived, so the stores that follow
        // this barrier could overwrite a halo it is still reading.  The
        // error word records why; the trap aborts the stream (the host sees
        // a launch failure at its next synchronisation) instead of letting
        // the step continue on a torn halo.
        atomicExch(a.err, 1);
        __threadfence_system();
        __trap();
      }
      __nanosleep(200);
    }
  }
  __threadfence_system();
}

static int signal_call(const fv3b_field* f, int nf, const double* s, int ns, void* stream) {
  // fields (buffer fields of one element each): the counter (u64), the
  // error word (int32), then (remote, local) flag words per neighbour;
  // scalars: [bump, npeer]
  if (f == nullptr || s == nullptr || ns != 2) return fail(FV3B_EINVAL, "peer barrier: bad arguments");
  SigArgs a;
  a.bump = s[0] != 0.0;
  a.npeer = (int)s[1];
  if (a.npeer < 0 || a.npeer > RECT_MAX || nf != 2 + 2 * a.npeer)
    return fail(FV3B_EINVAL, "peer barrier: 0..%d neighbours, 2 + 2*n buffer fields", RECT_MAX);
  void* p;
  FV3B_TRY(buffer_of(f[0], 1, "peer barrier counter", &p));
  a.epoch = static_cast<unsigned long long*>(p);
  FV3B_TRY(buffer_of(f[1], 1, "peer barrier error word", &p));
  a.err = static_cast<int*>(p);
  for (int q = 0; q < a.npeer; ++q) {
    FV3B_TRY(buffer_of(f[2 + 2 * q], 1, "peer barrier remote flag", &p));
    a.remote[q] = static_cast<unsigned long long*>(p);
    FV3B_TRY(buffer_of(f[3 + 2 * q], 1, "peer barrier local flag", &p));
    a.local[q] = static_cast<unsigned long long*>(p);
  }
  signal_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(a);
  return check_launch("fv3b_peer_barrier");
}

// ---------------------------------------------------------------------------
// Index-list gather / scatter: the cubed-sphere halo update (cubesphere.py),
// whose strips arrive rotated and component-swapped.  Entry s of a gather
// list is (field slot, interior-relative cell offset); of a scatter list
// (field slot, cell offset, sign).  The message holds level k of entry s at
// buf[k * n + s] (consecutive threads touch consecutive slots).
// ---------------------------------------------------------------------------
struct IdxArgs {
  double* o[HALO_MAXF];
  int64_t sk;
  double* buf;
  const int* idx;
  int n, levels;
  bool scatter;
};

__global__ void idx_kernel(const IdxArgs a) {
  const int k = blockIdx.y;
  double* b = a.buf + (int64_t)k * a.n;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < a.n; s += gridDim.x * blockDim.x) {
    if (a.scatter) {
      const int f = a.idx[3 * s], off = a.idx[3 * s + 1], sg = a.idx[3 * s + 2];
      const double v = b[s];
      a.o[f][off + (int64_t)k * a.sk] = sg < 0 ? -v : v;
    } else {
      const int f = a.idx[2 * s], off = a.idx[2 * s + 1];
      b[s] = a.o[f][off + (int64_t)k * a.sk];
    }
  }
}

static int idx_call(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream,
                    bool scatter) {
  // fields: the halo fields, then the message buffer (doubles) and the
  // index list (int32, 2 per entry to gather, 3 to scatter) as buffer
  // fields; scalars: [n entries]
  if (f == nullptr || d == nullptr || s == nullptr || ns != 1 || nf < 3)
    return fail(FV3B_EINVAL, "halo gather/scatter: fields + buffer + list, 1 scalar");
  IdxArgs a;
  a.n = (int)s[0];
  a.scatter = scatter;
  if (a.n < 0) return fail(FV3B_EINVAL, "halo gather/scatter: negative entry count");
  nf -= 2;
  int levels[HALO_MAXF];
  int64_t sj;
  FV3B_TRY(collect(f, nf, d, 0, a.o, levels, &sj, &a.sk));
  for (int t = 1; t < nf; ++t)
    if (levels[t] != levels[0]) return fail(FV3B_EINVAL, "halo gather/scatter: fields must share their level count");
  a.levels = levels[0];
  void* p;
  FV3B_TRY(buffer_of(f[nf], (int64_t)a.n * a.levels, "halo gather/scatter buffer", &p));
  a.buf = static_cast<double*>(p);
  FV3B_TRY(buffer_of(f[nf + 1], (int64_t)a.n * (scatter ? 3 : 2), "halo gather/scatter list", &p));
  a.idx = static_cast<const int*>(p);
  if (a.n == 0) return FV3B_OK;
  dim3 grid(cdiv(a.n, 256) < 32 ? cdiv(a.n, 256) : 32, a.levels);
  idx_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch(scatter ? "fv3b_halo_scatter" : "fv3b_halo_gather");
}

}  // namespace fv3b

using namespace fv3b;

// fields: any mix of 3-D / 2-D fields (<= 32) of one geometry.  scalars:
// [halo width].  Fills all allocated levels.
extern "C" int fv3b_halo_periodic(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                  void* stream) {
  if (f == nullptr || d == nullptr || s == nullptr || ns != 1) return fail(FV3B_EINVAL, "fv3b_halo_periodic: 1 scalar");
  HaloArgs a;
  a.h = (int)s[0];
  if (a.h < 0 || a.h > d->ni || a.h > d->nj) return fail(FV3B_EINVAL, "fv3b_halo_periodic: bad halo width %d", a.h);
  FV3B_TRY(collect(f, nf, d, a.h, a.o, a.levels, &a.sj, &a.sk));
  a.nf = nf;
  a.ni = d->ni;
  a.nj = d->nj;
  int maxl = 1;
  for (int t = 0; t < nf; ++t) maxl = a.levels[t] > maxl ? a.levels[t] : maxl;
  const int ring = 2 * (d->ni + 2 * a.h) * a.h + 2 * a.h * d->nj;
  dim3 grid(cdiv(ring, 256) < 16 ? cdiv(ring, 256) : 16, cdiv(maxl, FV3B_HALO_KU), nf);
  halo_periodic_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch("fv3b_halo_periodic");
}

static int strip_call(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d, void* stream,
                      bool unpack) {
  // fields: the halo fields, then the message buffer (a buffer field);
  // scalars: i0, j0, w, h (strip rectangle, interior-relative)
  if (f == nullptr || d == nullptr || s == nullptr || ns != 4 || nf < 2)
    return fail(FV3B_EINVAL, "halo strip: fields + buffer, 4 scalars");
  StripArgs a;
  a.i0 = (int)s[0];
  a.j0 = (int)s[1];
  a.w = (int)s[2];
  a.h = (int)s[3];
  if (a.w <= 0 || a.h <= 0) return fail(FV3B_EINVAL, "halo strip: empty strip");
  --nf;
  FV3B_TRY(collect(f, nf, d, 0, a.o, a.levels, &a.sj, &a.sk));
  a.nf = nf;
  a.unpack = unpack;
  int64_t off = 0;
  int maxl = 1;
  for (int t = 0; t < nf; ++t) {
    a.off[t] = off;
    off += (int64_t)a.levels[t] * a.w * a.h;
    maxl = a.levels[t] > maxl ? a.levels[t] : maxl;
  }
  void* buf;
  FV3B_TRY(buffer_of(f[nf], off, "halo strip", &buf));
  a.buf = static_cast<double*>(buf);
  dim3 grid(cdiv(a.w * a.h, 256) < 16 ? cdiv(a.w * a.h, 256) : 16, maxl, nf);
  strip_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch(unpack ? "fv3b_halo_unpack" : "fv3b_halo_pack");
}

extern "C" int fv3b_halo_pack(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                              void* stream) {
  return strip_call(f, nf, s, ns, d, stream, false);
}

extern "C" int fv3b_halo_unpack(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                void* stream) {
  return strip_call(f, nf, s, ns, d, stream, true);
}

extern "C" int fv3b_halo_pack_rects(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                    void* stream) {
  return rects_call(f, nf, s, ns, d, stream, false);
}

extern "C" int fv3b_halo_unpack_rects(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                      void* stream) {
  return rects_call(f, nf, s, ns, d, stream, true);
}

extern "C" int fv3b_halo_peer_rects(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                    void* stream) {
  return peer_call(f, nf, s, ns, d, stream);
}

extern "C" int fv3b_halo_peer_idx(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                  void* stream) {
  return peer_idx_call(f, nf, s, ns, d, stream);
}

extern "C" int fv3b_peer_barrier(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                 void* stream) {
  (void)d;
  return signal_call(f, nf, s, ns, stream);
}

extern "C" int fv3b_halo_gather(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                void* stream) {
  return idx_call(f, nf, s, ns, d, stream, false);
}

extern "C" int fv3b_halo_scatter(const fv3b_field* f, int nf, const double* s, int ns, const fv3b_domain* d,
                                 void* stream) {
  return idx_call(f, nf, s, ns, d, stream, true);
}
