// eval_kernels.cuh -- device-side building blocks shared by the evaluation
// translation units (eval.cu: host dispatch + ABI; eval_laplace.cu,
// eval_helmholtz.cu, eval_deriv.cu: the compile-time-order kernels, split so
// that they compile in parallel).
#pragma once

#include "common.cuh"

namespace tsqbx {

struct EvalParams {
  const double4* __restrict__ sp;    // {x, y, z, Re w}
  const double* __restrict__ swi;    // Im w
  const double4* __restrict__ snrm;  // {nx, ny, nz, 0} or null
  const double* __restrict__ ctr;    // processing order
  const int64_t* __restrict__ nptr;
  const int32_t* __restrict__ nidx;
  const int64_t* __restrict__ sell_ptr;  // sliced-ELL layout (null = CSR only)
  const int32_t* __restrict__ sell_idx;
  const double* __restrict__ tgt;
  const double* __restrict__ tnrm;
  const int64_t* __restrict__ tptr;  // rows in processing order
  const int64_t* __restrict__ tout;  // processing target -> output slot (null = identity)
  const double* __restrict__ ttab;   // Helmholtz per-target Bessel table
  double2* __restrict__ out;
  int64_t out_offset;
  int64_t tbase;                     // uniform runs: target index of the launch's row 0
  unsigned long long* err;
  int64_t n_ctr;
  int ttab_stride;
  int p;
  int variant;
  int G;
  int log2G;
  int validate;
  int real_w;                        // host assertion: all Im w == 0
  int tuni;                          // k > 0: row g owns targets [k g, k g + k) (no tptr load)
  const unsigned* __restrict__ imag_flag;   // device: pack_kernel saw Im w != 0
  double k;
  SincCosCoeffs sc;                  // sin/cos series (kSincCos), constant-bank operands
  int series;                        // 0: per-warp vote; 1: narrow only; 2: wide (library past pi/2)
  int long_rows;                     // TSQBX_FLAG_LONG_ROWS: kernels tuned for long near lists
  int two_rows;                      // TSQBX_FLAG_TWO_ROWS: Laplace S, two rows per thread
  const int32_t* __restrict__ win_src;   // TSQBX_FLAG_WINDOW: per slice its distinct sources
  const int32_t* __restrict__ win_len;
};

int64_t packed_doubles(int64_t n, int with_normals);
int64_t packed_meta_offset(int64_t n, int with_normals);

__device__ __forceinline__ int64_t out_slot(const EvalParams& a, int64_t t) {
  return (a.tout ? a.tout[t] : t) - a.out_offset;
}

__device__ __forceinline__ void flag_suspect(unsigned long long* err) {
  atomicMin(err, (unsigned long long)TSQBX_ERR_KEY_SUSPECT);
}

// ---------------------------------------------------------------------------
// Source stream of one CSR row for one lane: the row's entries j = lane,
// lane + G, ... are read through a two-deep software pipeline (index two
// iterations ahead, source record one iteration ahead) so the gather latency
// overlaps the previous source's arithmetic.
// ---------------------------------------------------------------------------
struct SourceStream {
  const int32_t* __restrict__ idx;   // this lane's first index entry
  const double4* __restrict__ sp;
  const double* __restrict__ swi;
  int stride, count, i;
  int s_next2;
  double4 q_next;
  double w_next;
  bool real_w;

  __device__ __forceinline__ SourceStream(const int32_t* first, int str, int n, const double4* p,
                                          const double* wi, bool realw)
      : idx(first), sp(p), swi(wi), stride(str), count(n), i(0), s_next2(0), w_next(0.0),
        real_w(realw) {
    q_next = make_double4(0.0, 0.0, 0.0, 0.0);
    int s0 = 0;
    if (count > 0) s0 = __ldg(idx);
    if (count > 1) s_next2 = __ldg(idx + stride);
    if (count > 0) {
      q_next = ld256(sp + s0);
      if (!real_w) w_next = __ldg(swi + s0);
    }
  }
  __device__ __forceinline__ bool more() const { return i < count; }
  // returns the current source and advances the pipeline
  __device__ __forceinline__ void next(double4& q, double& wi) {
    q = q_next;
    wi = w_next;
    if (i + 1 < count) {
      q_next = ld256(sp + s_next2);
      if (!real_w) w_next = __ldg(swi + s_next2);
    }
    if (i + 2 < count) s_next2 = __ldg(idx + (i + 2) * stride);
    ++i;
  }
};

// entries j = lane, lane + G, ... of a CSR row of length len
__device__ __forceinline__ SourceStream csr_stream(const EvalParams& a, int64_t b, int len,
                                                   int lane, int G) {
  const int n = len > lane ? (len - lane + G - 1) / G : 0;
  return SourceStream(a.nidx + b + lane, G, n, a.sp, a.swi, false);
}

struct GroupCoord {
  int64_t g;
  int lane, G;
  unsigned mask;
};

__device__ __forceinline__ bool group_coord(const EvalParams& a, GroupCoord& c) {
  const int lg = a.log2G;
  c.G = 1 << lg;
  c.g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> lg;
  c.lane = (int)(threadIdx.x & (unsigned)(c.G - 1));
  c.mask = group_mask(c.G);
  return c.g < a.n_ctr;
}

// ---------------------------------------------------------------------------
// Thread-per-center kernels on the sliced-ELL layout (SELL-32x4): rows are cut
// into slices of 32 consecutive (Morton-adjacent) centers, and a slice's near
// indices are stored in column blocks of 4, so lane l of a warp owns row 32s + l
// and one 16-byte load per lane (512 coalesced bytes per warp) brings the next
// 4 indices.  No shuffles, no reductions: each thread accumulates its own
// center's targets.
// ---------------------------------------------------------------------------
// Source stream over one SELL-32x4 row.  The index stream (compulsory HBM
// traffic) is staged through a per-thread shared-memory ring with cp.async:
// kRing index blocks (4 entries each) are in flight ahead of use, so the
// DRAM latency of the CSR stream never reaches the arithmetic.  The source
// record (an L1/L2 gather) is fetched one entry ahead into registers.
#ifndef TSQBX_SELL_BLOCK
#define TSQBX_SELL_BLOCK 256
#endif
#ifndef TSQBX_RING
#define TSQBX_RING 3
#endif
constexpr int kSellBlock = TSQBX_SELL_BLOCK;   // threads per CTA of the SELL kernels
// minimum resident CTAs per SM requested from ptxas (caps registers per thread)
#ifndef TSQBX_LAP_MINB
#define TSQBX_LAP_MINB 3
#endif
// two targets per center with uniform target runs (no tgt_ptr registers): one
// more CTA per SM despite a few spilled loop invariants (C2 dense +2.9 %,
// C2 literal +6 %; the general-tgt_ptr kernel spills twice as much and keeps 3)
#ifndef TSQBX_LAP_MINB_UNI
#define TSQBX_LAP_MINB_UNI 4
#endif
// one target per center (C1, C4, C5): one more CTA per SM (measured: C4
// literal +9 %, C5 literal +12 %, dense -1 %; with two targets it costs 2-40 %)
#ifndef TSQBX_LAP_MINB1
#define TSQBX_LAP_MINB1 4
#endif
#ifndef TSQBX_HELM_MINB1
#define TSQBX_HELM_MINB1 3
#endif
#ifndef TSQBX_HELM_MINB
#define TSQBX_HELM_MINB 2
#endif
constexpr int kRing = TSQBX_RING;  // index blocks in flight (4 kRing entries of lookahead)
constexpr int kSlots = kRing + 1;  // ring slots per thread (a power of two keeps b % kSlots a mask)

#ifndef TSQBX_GATHER_DEPTH
#define TSQBX_GATHER_DEPTH 1
#endif
// SELL streams: L1-prefetch the next index block's source records on entering
// a block (their gathers then hit L1).  Off: measured 2-6 % slower on every
// preset (C2 literal 29.2 vs 27.3 us, C5 dense 12.94 vs 12.30 ms)
#ifndef TSQBX_REC_PREFETCH
#define TSQBX_REC_PREFETCH 0
#endif
constexpr bool kRecPrefetch = TSQBX_REC_PREFETCH != 0;
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// D = source records gathered ahead of use (1: the next one; 2: two deep)
// WIN: the rows' sources were staged in a shared-memory window (windowed SELL,
// tsqbx_sell_window): the entries are window indices and sp / swi point into
// the window (shared-memory loads instead of global gathers)
template <bool NRM = false, int D = TSQBX_GATHER_DEPTH, bool WIN = false>
struct SellStream {
  const int4* __restrict__ blk;   // this lane's block 0; block b at blk + 32 b
  const double4* __restrict__ sp;
  const double* __restrict__ swi;
  int4* ring;                     // [kRing + 1][kSellBlock] int4, this thread's column
  int blk_stride = 32;            // int4s between this thread's consecutive blocks
  int count, nblk, i;
  int4 cur;                       // indices of the block being consumed / 4
  double4 q_next[D];
  double w_next[D];
  bool real_w;
  const double4* __restrict__ snrm;   // NRM: source normals, fetched with the record
  double4 n_next[D];

  __device__ __forceinline__ void issue(int b) {
    // block b goes to slot b % kSlots; always commit so group counts stay uniform
    if (b < nblk) cp_async16(ring + (b % kSlots) * kSellBlock, blk + blk_stride * b);
    cp_async_commit();
  }
  __device__ __forceinline__ SellStream(const EvalParams& a, int64_t g, int n, bool realw,
                                        int4* ring_base)
      : SellStream(a, a.sell_ptr[g >> 5], g, n, realw, ring_base, true) {}
  // `soff` = sell_ptr[g / 32], loaded by the caller; go = false only issues the
  // first kRing index blocks (start() later waits for block 0 and gathers).
  // b0 / bs: this thread takes the row's blocks b0, b0 + bs, ... (a row split
  // over bs threads); `count` becomes the number of entries in those blocks.
  // issued: the first kRing blocks were already issued (by an earlier
  // SellStream over the same row and ring); foreign: kRing cp.async groups of
  // another row were committed right after them (laplace_sell2_kernel), so
  // waiting for one of the first kRing blocks leaves 2 kRing - 1 groups pending
  bool foreign = false;
  __device__ __forceinline__ SellStream(const EvalParams& a, int64_t soff, int64_t g, int n,
                                        bool realw, int4* ring_base, bool go, int b0 = 0,
                                        int bs = 1, bool issued = false, bool foreign_ = false,
                                        const double4* win_q = nullptr,
                                        const double* win_w = nullptr)
      : sp(WIN ? win_q : a.sp), swi(WIN ? win_w : a.swi), count(n), i(0), real_w(realw),
        snrm(a.snrm) {
    const int nb = (n + 3) >> 2;                       // blocks of the whole row
    blk = reinterpret_cast<const int4*>(a.sell_idx + soff) + (g & 31) + 32 * b0;
    blk_stride = 32 * bs;
    ring = ring_base + threadIdx.x;
    nblk = nb > b0 ? (nb - b0 + bs - 1) / bs : 0;
    count = nblk == 0 ? 0 : 4 * (nblk - 1) + min(4, n - 4 * (b0 + bs * (nblk - 1)));
    foreign = foreign_;
    if (!issued) issue_first();
    if (go) start();
  }
  __device__ __forceinline__ void issue_first() {
#pragma unroll
    for (int b = 0; b < kRing; ++b) issue(b);
  }
  __device__ __forceinline__ void start() {
    i = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      q_next[d] = make_double4(0.0, 0.0, 0.0, 0.0);
      w_next[d] = 0.0;
    }
    cur = make_int4(0, 0, 0, 0);
    if (count > 0) enter_block(0);
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < count) fetch(d, d == 0 ? cur.x : d == 1 ? cur.y : d == 2 ? cur.z : cur.w);
  }
  __device__ __forceinline__ void restart() {
    issue_first();
    start();
  }
  __device__ __forceinline__ void enter_block(int b) {
    if (foreign) {
      if (b < kRing) cp_async_wait<2 * kRing - 1>();
      else cp_async_wait<kRing - 1>();          // block b has landed
    } else if (kRecPrefetch && kRing >= 2) {
      // blocks b and b + 1 have landed: the source records of block b + 1 go
      // into L1 now, 4-8 entries ahead of their gathers
      cp_async_wait<kRing - 2>();
      if (b + 1 < nblk) {
        const int4 nx = ring[((b + 1) % kSlots) * kSellBlock];
        const int e = 4 * (b + 1);
        prefetch_l1(sp + nx.x);
        if (e + 1 < count) prefetch_l1(sp + nx.y);
        if (e + 2 < count) prefetch_l1(sp + nx.z);
        if (e + 3 < count) prefetch_l1(sp + nx.w);
      }
    } else {
      cp_async_wait<kRing - 1>();               // block b has landed
    }
    cur = ring[(b % kSlots) * kSellBlock];
    issue(b + kRing);                           // reuses the slot of block b - 1
  }
  __device__ __forceinline__ void fetch(int d, int s) {
    if (WIN) {
      const unsigned at = (unsigned)__cvta_generic_to_shared(sp + s);
      double4 v;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(at));
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.z), "=d"(v.w) : "r"(at + 16));
      q_next[d] = v;
      if (!real_w) w_next[d] = swi[s];
    } else {
      q_next[d] = ld256(sp + s);
      if (!real_w) w_next[d] = __ldg(swi + s);
    }
    if (NRM) n_next[d] = ld256(snrm + s);
  }
  __device__ __forceinline__ bool more() const { return i < count; }
  __device__ __forceinline__ void next(double4& q, double& wi) {
    double4 nrm;
    next(q, wi, nrm);
  }
  __device__ __forceinline__ void next(double4& q, double& wi, double4& nrm) {
    q = q_next[0];
    wi = w_next[0];
    if (NRM) nrm = n_next[0];
#pragma unroll
    for (int d = 0; d + 1 < D; ++d) {
      q_next[d] = q_next[d + 1];
      w_next[d] = w_next[d + 1];
      if (NRM) n_next[d] = n_next[d + 1];
    }
    ++i;
    const int j = i + D - 1;                    // the entry to gather now
    if (j < count) {
      const int e = j & 3;
      if (e == 0) enter_block(j >> 2);
      fetch(D - 1, e == 0 ? cur.x : e == 1 ? cur.y : e == 2 ? cur.z : cur.w);
    }
  }
};

// Row metadata every SELL kernel needs first.  Loaded before anything that
// depends on a load (the real-weight flag, the target range), so the four
// independent first-level loads overlap instead of forming a chain.
struct RowHead {
  int64_t soff, t0, t1;
  double cx, cy, cz;
  int len;
};
// UNI: row g owns targets [UNI g, UNI g + UNI) (TSQBX_FLAG_UNIFORM_TARGETS), no tptr load
template <int UNI = 0>
__device__ __forceinline__ RowHead load_head(const EvalParams& a, int64_t g) {
  RowHead h;
  h.soff = a.sell_ptr[g >> 5];
  h.len = (int)(a.nptr[g + 1] - a.nptr[g]);
  if (UNI > 0) {       // uniform target runs: the target range needs no load
    h.t0 = a.tbase + g * UNI;
    h.t1 = h.t0 + UNI;
  } else {
    h.t0 = a.tptr[g];
    h.t1 = a.tptr[g + 1];
  }
  h.cx = a.ctr[3 * g];
  h.cy = a.ctr[3 * g + 1];
  h.cz = a.ctr[3 * g + 2];
  return h;
}

// compile-time-order launchers (one per translation unit); false = p not
// instantiated (p > 16)
bool launch_laplace_fast(int p, bool sell, int nt, bool val, const EvalParams& a, int64_t n_ctr,
                         cudaStream_t st);
bool launch_helmholtz_fast(int p, bool sell, int nt, bool val, const EvalParams& a,
                           int64_t n_ctr, cudaStream_t st);
bool launch_laplace_flat(int p, int nt, bool val, const EvalParams& a, int64_t n_ctr,
                         cudaStream_t st);
bool launch_deriv_fast(int p, int equation, int variant, int nt, const EvalParams& a,
                       int64_t n_ctr, cudaStream_t st);

}  // namespace tsqbx
