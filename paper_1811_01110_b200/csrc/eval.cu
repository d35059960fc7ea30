// eval.cu -- sm_100a fp64 TSQBX evaluation kernels + their C ABI entry points.
//
// Hot path: for every center c and each of its targets t,
//   Laplace   u(t) = 1/(4 pi)  sum_{s in near(c)} w_s sum_{n<=p} |t-c|^n/|s-c|^{n+1} P_n(cos g)
//   Helmholtz u(t) = ik/(4 pi) sum_{s in near(c)} w_s sum_{n<=p} (2n+1) j_n(k|t-c|) h_n(k|s-c|) P_n(cos g)
// (reference: _core.pyx:205-307 and :310-419).
//
// Work decomposition: a group of G lanes (G in {1,2,4,8,16,32}) owns one
// center; its lanes stride over the center's CSR row, every lane evaluating
// one source against ALL of the center's targets (the source-side work -- s-c,
// 1/R, h_n(kR) -- is shared by the targets), then the group reduces with
// warp shuffles.  Centers arrive in Morton order from the CSR builder, so the
// groups of one CTA read overlapping source neighbourhoods out of L1.
#include <cuda_runtime.h>

#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>

#include "common.cuh"

namespace tsqbx {

namespace {
thread_local char g_err[512] = "";
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return TSQBX_OK;
  return set_error(TSQBX_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

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
  unsigned long long* err;
  int64_t n_ctr;
  int ttab_stride;
  int p;
  int variant;
  int G;
  int log2G;
  int validate;
  int real_w;                        // host assertion: all Im w == 0
  const unsigned* __restrict__ imag_flag;   // device: pack_kernel saw Im w != 0
  double k;
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
// Laplace S, compile-time order P, NT targets per pass.
// Per pair: s-c, R^2, 1/R shared by the targets; per target A = (s-c).(t-c)/R^2,
// B = |t-c|^2/R^2 and the 3-op/order Clenshaw series (common.cuh).
// ---------------------------------------------------------------------------
template <int P, int NT, bool VAL>
__global__ void __launch_bounds__(256) laplace_s_kernel(const EvalParams a) {
  GroupCoord gc;
  if (!group_coord(a, gc)) return;
  const int64_t g = gc.g;
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int64_t b = a.nptr[g];
  const int len = (int)(a.nptr[g + 1] - b);
  const int64_t t0 = a.tptr[g], t1 = a.tptr[g + 1];

  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], ar[NT], ai[NT], bm[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = tb + q < t1;
      tx[q] = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      ty[q] = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      tz[q] = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(tz[q], tz[q], fma(ty[q], ty[q], tx[q] * tx[q]));
      ar[q] = ai[q] = bm[q] = 0.0;
    }
    SourceStream ss = csr_stream(a, b, len, gc.lane, gc.G);
    while (ss.more()) {
      double4 q4;
      double wim;
      ss.next(q4, wim);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double iR2 = iR * iR;
      const double wr = q4.w * iR, wi = wim * iR;
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const double A = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR2;
        const double B = r2[q] * iR2;
        const double S = laplace_series<P>(A, B);
        ar[q] = fma(S, wr, ar[q]);
        ai[q] = fma(S, wi, ai[q]);
        if (VAL) bm[q] = fmax(bm[q], B);
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      ar[q] = group_sum(ar[q], gc.G, gc.mask);
      ai[q] = group_sum(ai[q], gc.G, gc.mask);
      if (VAL) bm[q] = group_max(bm[q], gc.G, gc.mask);
    }
    if (gc.lane == 0) {
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        if (tb + q < t1) {
          a.out[out_slot(a, tb + q)] = make_double2(ar[q] * kInvFourPi, ai[q] * kInvFourPi);
          if (VAL && (!isfinite(ar[q]) || !isfinite(ai[q]) || bm[q] > kSepScreen))
            flag_suspect(a.err);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Helmholtz S, compile-time order P.  h_n(kR) is built once per source by the
// upward recurrence (_core.pyx:190-193) and shared by the targets; each target
// carries c_n = (2n+1) j_n(k|t-c|) kappa_n from the prologue table.
// ---------------------------------------------------------------------------
template <int P, int NT, bool VAL>
__global__ void __launch_bounds__(256) helmholtz_s_kernel(const EvalParams a) {
  GroupCoord gc;
  if (!group_coord(a, gc)) return;
  const int64_t g = gc.g;
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int64_t b = a.nptr[g];
  const int len = (int)(a.nptr[g + 1] - b);
  const int64_t t0 = a.tptr[g], t1 = a.tptr[g + 1];
  const double k = a.k, k2 = a.k * a.k, invk = 1.0 / a.k;

  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], ar[NT], ai[NT], bm[NT], cf[NT][P + 1];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = tb + q < t1;
      const double ux = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      const double uy = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      const double uz = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(uz, uz, fma(uy, uy, ux * ux));
      const double ir = r2[q] > 0.0 ? rsqrt(r2[q]) : 0.0;  // r = 0: cos g irrelevant
      tx[q] = ux * ir;
      ty[q] = uy * ir;
      tz[q] = uz * ir;
#pragma unroll
      for (int n = 0; n <= P; ++n)
        cf[q][n] = ok ? a.ttab[(tb + q) * a.ttab_stride + n] : 0.0;
      ar[q] = ai[q] = bm[q] = 0.0;
    }
    SourceStream ss = csr_stream(a, b, len, gc.lane, gc.G);
    while (ss.more()) {
      double4 q4;
      double wim;
      ss.next(q4, wim);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double x = k * (R2 * iR);
      const double invx = iR * invk;
      double hr[P + 1], hi[P + 1];
      {
        double h1r, h1i;
        hankel01(k2 * R2, x, invx, hr[0], hi[0], h1r, h1i);
        if constexpr (P >= 1) {
          hr[1] = h1r;
          hi[1] = h1i;
        }
      }
#pragma unroll
      for (int n = 1; n < P; ++n) {
        const double f = (2.0 * n + 1.0) * invx;
        hr[n + 1] = fma(f, hr[n], -hr[n - 1]);
        hi[n + 1] = fma(f, hi[n], -hi[n - 1]);
      }
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const double cg = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR;
        double sr = cf[q][0] * hr[0], si = cf[q][0] * hi[0];
        if constexpr (P >= 1) {
          double pm = 1.0, pc = cg;
          double c1 = cf[q][1] * pc;
          sr = fma(c1, hr[1], sr);
          si = fma(c1, hi[1], si);
#pragma unroll
          for (int n = 1; n < P; ++n) {
            const double pn = fma(c_leg.alpha[n] * cg, pc, -pm);
            pm = pc;
            pc = pn;
            const double cn = cf[q][n + 1] * pc;
            sr = fma(cn, hr[n + 1], sr);
            si = fma(cn, hi[n + 1], si);
          }
        }
        ar[q] = fma(q4.w, sr, fma(-wim, si, ar[q]));
        ai[q] = fma(q4.w, si, fma(wim, sr, ai[q]));
        if (VAL) bm[q] = fmax(bm[q], r2[q] * (iR * iR));
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      ar[q] = group_sum(ar[q], gc.G, gc.mask);
      ai[q] = group_sum(ai[q], gc.G, gc.mask);
      if (VAL) bm[q] = group_max(bm[q], gc.G, gc.mask);
    }
    if (gc.lane == 0) {
      const double pk = k * kInvFourPi;
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        if (tb + q < t1) {
          a.out[out_slot(a, tb + q)] = make_double2(-ai[q] * pk, ar[q] * pk);  // (ik/4pi) acc
          if (VAL && (!isfinite(ar[q]) || !isfinite(ai[q]) || bm[q] > kSepScreen))
            flag_suspect(a.err);
        }
      }
    }
  }
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

// D = source records gathered ahead of use (1: the next one; 2: two deep)
template <bool NRM = false, int D = TSQBX_GATHER_DEPTH>
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
  __device__ __forceinline__ SellStream(const EvalParams& a, int64_t soff, int64_t g, int n,
                                        bool realw, int4* ring_base, bool go, int b0 = 0,
                                        int bs = 1)
      : sp(a.sp), swi(a.swi), count(n), i(0), real_w(realw), snrm(a.snrm) {
    const int nb = (n + 3) >> 2;                       // blocks of the whole row
    blk = reinterpret_cast<const int4*>(a.sell_idx + soff) + (g & 31) + 32 * b0;
    blk_stride = 32 * bs;
    ring = ring_base + threadIdx.x;
    nblk = nb > b0 ? (nb - b0 + bs - 1) / bs : 0;
    count = nblk == 0 ? 0 : 4 * (nblk - 1) + min(4, n - 4 * (b0 + bs * (nblk - 1)));
    issue_first();
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
    cp_async_wait<kRing - 1>();                 // block b has landed
    cur = ring[(b % kSlots) * kSellBlock];
    issue(b + kRing);                           // reuses the slot of block b - 1
  }
  __device__ __forceinline__ void fetch(int d, int s) {
    q_next[d] = ld256(sp + s);
    if (!real_w) w_next[d] = __ldg(swi + s);
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
__device__ __forceinline__ RowHead load_head(const EvalParams& a, int64_t g) {
  RowHead h;
  h.soff = a.sell_ptr[g >> 5];
  h.len = (int)(a.nptr[g + 1] - a.nptr[g]);
  h.t0 = a.tptr[g];
  h.t1 = a.tptr[g + 1];
  h.cx = a.ctr[3 * g];
  h.cy = a.ctr[3 * g + 1];
  h.cz = a.ctr[3 * g + 2];
  return h;
}

template <int P, int NT, bool VAL, bool REALW, int S = 1>
__device__ __forceinline__ void laplace_sell_body(const EvalParams& a, int64_t g,
                                                  const RowHead& h, int4* ring, int part = 0,
                                                  unsigned gmask = 0xffffffffu) {
  const double cx = h.cx, cy = h.cy, cz = h.cz;
  const int len = h.len;
  const int64_t t0 = h.t0, t1 = h.t1;
  // high orders have more arithmetic per source to cover a second gather in
  // flight (measured: C4 dense p = 12 +7 %; p = 8 -2 %)
  using Stream = SellStream<false, (P >= 12 ? 2 : TSQBX_GATHER_DEPTH)>;
  // the index ring starts filling before the target range is known
  Stream ss(a, h.soff, g, len, REALW, ring, false, part, S);
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], ar[NT], ai[NT], bm[NT];
    int64_t slot[NT];   // output slots, loaded up front so the epilogue does not wait
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = tb + q < t1;
      slot[q] = ok ? out_slot(a, tb + q) : 0;
      tx[q] = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      ty[q] = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      tz[q] = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(tz[q], tz[q], fma(ty[q], ty[q], tx[q] * tx[q]));
      ar[q] = ai[q] = bm[q] = 0.0;
    }
    if (tb == t0) ss.start();
    else ss.restart();
    // one source against the NT targets
    auto source = [&](const double4& q4, double wim) {
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double iR2 = iR * iR;
      const double wr = q4.w * iR;
      const double wi = REALW ? 0.0 : wim * iR;
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const double A = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR2;
        const double B = r2[q] * iR2;
        const double S = laplace_series<P>(A, B);
        ar[q] = fma(S, wr, ar[q]);
        if (!REALW) ai[q] = fma(S, wi, ai[q]);
        if (VAL) bm[q] = fmax(bm[q], B);
      }
    };
    while (ss.more()) {
      double4 q4;
      double wim;
      ss.next(q4, wim);
      source(q4, wim);
    }
    if (S > 1) {
      // the S threads of this row hold partial sums over interleaved blocks:
      // a fixed xor tree over the part bits (lanes 32/S apart) adds them
#pragma unroll
      for (int off = 32 / S; off < 32; off <<= 1) {
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          ar[q] += __shfl_xor_sync(gmask, ar[q], off);
          if (!REALW) ai[q] += __shfl_xor_sync(gmask, ai[q], off);
          if (VAL) bm[q] = fmax(bm[q], __shfl_xor_sync(gmask, bm[q], off));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1 && part == 0) {
        a.out[slot[q]] = make_double2(ar[q] * kInvFourPi, ai[q] * kInvFourPi);
        if (VAL && (!isfinite(ar[q]) || !isfinite(ai[q]) || bm[q] > kSepScreen))
          flag_suspect(a.err);
      }
    }
  }
  if (t0 >= t1) cp_async_wait<0>();   // no pass consumed the ring: drain it before exit
}

// real weights (the usual Laplace density) skip every Im w load and FMA; the
// pack kernel records whether any Im w is nonzero, so no host round trip decides
//
// S > 1 splits every row over S threads of one warp (lanes 32/S apart take
// the row's SELL blocks round-robin; a CTA covers kSellBlock/S rows).  A
// thread's row takes ~100 µs on the dense presets whatever else runs on its
// SM (latency-bound per thread), so with whole rows the last partial wave of
// rows leaves most slots idle; S rows-parts per row make the work units S
// times shorter and the tail S times cheaper.
template <int P, int NT, bool VAL, int S>
__global__ void __launch_bounds__(kSellBlock, NT == 1 ? TSQBX_LAP_MINB1 : TSQBX_LAP_MINB) laplace_sell_kernel(const EvalParams a) {
  __shared__ int4 ring[kSlots * kSellBlock];
  constexpr int kRowsPerWarp = 32 / S;
  const int lane = threadIdx.x & 31;
  const int part = lane / kRowsPerWarp, rig = lane % kRowsPerWarp;
  const int64_t g = (int64_t)blockIdx.x * (kSellBlock / S) + (threadIdx.x >> 5) * kRowsPerWarp + rig;
  unsigned gmask = 0u;
#pragma unroll
  for (int k = 0; k < S; ++k) gmask |= 1u << (rig + k * kRowsPerWarp);
  if (g < a.n_ctr) {
    const RowHead h = load_head(a, g);
    const bool realw = a.real_w || *a.imag_flag == 0u;
    if (realw)
      laplace_sell_body<P, NT, VAL, true, S>(a, g, h, ring, part, gmask);
    else
      laplace_sell_body<P, NT, VAL, false, S>(a, g, h, ring, part, gmask);
  }
}

template <int P, int NT, bool VAL>
__global__ void __launch_bounds__(kSellBlock, NT == 1 ? TSQBX_HELM_MINB1 : TSQBX_HELM_MINB) helmholtz_sell_kernel(const EvalParams a) {
  // per-thread target coefficients c_n = (2n+1) j_n(k r) kappa_n, in registers
  // (a shared-memory copy measured slower)
  double cfr[NT][P + 1];
#define CF(n, q) cfr[q][n]
  __shared__ int4 ring[kSlots * kSellBlock];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < a.n_ctr) {
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int len = (int)(a.nptr[g + 1] - a.nptr[g]);
  const int64_t t0 = a.tptr[g], t1 = a.tptr[g + 1];
  const double k = a.k, k2 = a.k * a.k, invk = 1.0 / a.k;
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], ar[NT], ai[NT], bm[NT];
    int64_t slot[NT];   // output slots, loaded up front so the epilogue does not wait
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = tb + q < t1;
      slot[q] = ok ? out_slot(a, tb + q) : 0;
      const double ux = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      const double uy = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      const double uz = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(uz, uz, fma(uy, uy, ux * ux));
      const double ir = r2[q] > 0.0 ? rsqrt(r2[q]) : 0.0;  // r = 0: cos g irrelevant
      tx[q] = ux * ir;
      ty[q] = uy * ir;
      tz[q] = uz * ir;
      // c_n = (2n+1) j_n(k r) kappa_n computed here, in registers (no table pass);
      // j_n(0) = delta_n0 (_core.pyx:357)
      {
        double jn[P + 1];
        const double rr = r2[q] * ir;                 // |t - c|
        if (ok && rr > 0.0) {
          miller_j_reg<P + 1>(k * rr, jn);
        } else {
#pragma unroll
          for (int n = 0; n <= P; ++n) jn[n] = n == 0 && ok ? 1.0 : 0.0;
        }
#pragma unroll
        for (int n = 0; n <= P; ++n) CF(n, q) = (2.0 * n + 1.0) * jn[n] * c_leg.kappa[n];
      }
      ar[q] = ai[q] = bm[q] = 0.0;
    }
    SellStream<> ss(a, g, len, false, ring);
    while (ss.more()) {
      double4 q4;
      double wim;
      ss.next(q4, wim);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double invx = iR * invk;
      double hmr, hmi, hcr, hci;                 // h_{n-1}, h_n
      hankel01(k2 * R2, k * (R2 * iR), invx, hmr, hmi, hcr, hci);
      double cg[NT], pm[NT], pc[NT], sr[NT], si[NT];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        cg[q] = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR;
        const double c0 = CF(0, q);
        sr[q] = c0 * hmr;
        si[q] = c0 * hmi;
        if constexpr (P >= 1) {
          const double c1 = CF(1, q) * cg[q];
          sr[q] = fma(c1, hcr, sr[q]);
          si[q] = fma(c1, hci, si[q]);
        }
        pm[q] = 1.0;
        pc[q] = cg[q];
      }
#pragma unroll
      for (int n = 1; n < P; ++n) {
        // h_{n+1} = (2n+1)/x h_n - h_{n-1}   (_core.pyx:192-193)
        const double f = (2.0 * n + 1.0) * invx;
        const double hnr = fma(f, hcr, -hmr), hni = fma(f, hci, -hmi);
        hmr = hcr;
        hmi = hci;
        hcr = hnr;
        hci = hni;
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          const double pn = fma(c_leg.alpha[n] * cg[q], pc[q], -pm[q]);
          pm[q] = pc[q];
          pc[q] = pn;
          const double c = CF(n + 1, q) * pn;
          sr[q] = fma(c, hnr, sr[q]);
          si[q] = fma(c, hni, si[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        ar[q] = fma(q4.w, sr[q], fma(-wim, si[q], ar[q]));
        ai[q] = fma(q4.w, si[q], fma(wim, sr[q], ai[q]));
        if (VAL) bm[q] = fmax(bm[q], r2[q] * (iR * iR));
      }
    }
    const double pk = k * kInvFourPi;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1) {
        a.out[slot[q]] = make_double2(-ai[q] * pk, ar[q] * pk);  // (ik/4pi) acc
        if (VAL && (!isfinite(ar[q]) || !isfinite(ai[q]) || bm[q] > kSepScreen))
          flag_suspect(a.err);
      }
    }
  }
}  // rows
}
#undef CF

// ---------------------------------------------------------------------------
// S' (target-normal derivative) and D (double layer) on the SELL layout
// (_core.pyx:260-306, 399-417).  Same streaming as the S kernels; the series:
//   Laplace S':  G_n = rho^{n-1} P_n, F_n = rho^{n-1} P'_n  (n >= 1)
//                s = [nt.t^ sum n G_n + (nt.s^ - nt.t^ cg) sum F_n] / R^2
//   Laplace D :  T_n = rho^n P_n,     E_n = rho^n P'_n      (n >= 0)
//                s = [-ns.s^ sum (n+1) T_n + (ns.t^ - ns.s^ cg) sum E_n] / R^2
//   with G/T following T_{n+1} = a_n A T_n - b_n B T_{n-1} (A = rho cg, B = rho^2)
//   and E_{n+1} = B E_{n-1} + (2n+1) rho T_n (the P' ladder scaled by rho^n).
//   Helmholtz S': s = nt.t^ sum (2n+1) k j'_n P_n h_n
//                     + (nt.s^ - nt.t^ cg) sum (2n+1) j_n/r P'_n h_n
//   Helmholtz D : s = k ns.s^ sum (2n+1) j_n P_n h'_n
//                     + (ns.t^ - ns.s^ cg)/R sum (2n+1) j_n P'_n h_n
//   r = 0 conventions as the reference: cos g := 1, t^ := s^ (_core.pyx:241-242,
//   262-264, 285-288, 400-408).
// ---------------------------------------------------------------------------
struct Bonnet {
  double a[TSQBX_MAX_ORDER + 2], b[TSQBX_MAX_ORDER + 2];
  constexpr Bonnet() : a(), b() {
    for (int n = 0; n < TSQBX_MAX_ORDER + 2; ++n) {
      a[n] = double(2 * n + 1) / double(n + 1);
      b[n] = double(n) / double(n + 1);
    }
  }
};
static __constant__ Bonnet c_bon = Bonnet();

template <int P, int NT, int VARIANT>
__global__ void __launch_bounds__(kSellBlock, 512 / kSellBlock) laplace_deriv_sell_kernel(const EvalParams a) {
  __shared__ int4 ring[kSlots * kSellBlock];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.n_ctr) return;
  const bool val = a.validate != 0;
  const bool realw = a.real_w || *a.imag_flag == 0u;
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int len = (int)(a.nptr[g + 1] - a.nptr[g]);
  const int64_t t0 = a.tptr[g], t1 = a.tptr[g + 1];
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], rr[NT], ir[NT], nx[NT], ny[NT], nz[NT], ntt[NT];
    double ar[NT], ai[NT], bm[NT];
    int64_t slot[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = tb + q < t1;
      slot[q] = ok ? out_slot(a, tb + q) : 0;
      tx[q] = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      ty[q] = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      tz[q] = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(tz[q], tz[q], fma(ty[q], ty[q], tx[q] * tx[q]));
      rr[q] = sqrt(r2[q]);
      ir[q] = r2[q] > 0.0 ? 1.0 / rr[q] : 0.0;
      nx[q] = ny[q] = nz[q] = ntt[q] = 0.0;
      if (VARIANT == 1 && ok) {
        nx[q] = a.tnrm[3 * (tb + q)];
        ny[q] = a.tnrm[3 * (tb + q) + 1];
        nz[q] = a.tnrm[3 * (tb + q) + 2];
        ntt[q] = fma(nz[q], tz[q], fma(ny[q], ty[q], nx[q] * tx[q])) * ir[q];  // nt . t^
      }
      ar[q] = ai[q] = bm[q] = 0.0;
    }
    SellStream<VARIANT == 2> ss(a, g, len, realw, ring);
    while (ss.more()) {
      double4 q4, n4;
      double wim;
      ss.next(q4, wim, n4);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double iR2 = iR * iR;
      const double wr = q4.w * iR2;
      const double wi = realw ? 0.0 : wim * iR2;
      double nss = 0.0;
      if (VARIANT == 2) nss = fma(n4.z, dz, fma(n4.y, dy, n4.x * dx)) * iR;    // ns . s^
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const double dt = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q]));
        const double A = dt * iR2, B = r2[q] * iR2, rho = rr[q] * iR;
        const bool r0 = !(r2[q] > 0.0);
        const double cg = r0 ? 1.0 : dt * iR * ir[q];
        double sval;
        if (VARIANT == 1) {
          const double nts = fma(nz[q], dz, fma(ny[q], dy, nx[q] * dx)) * iR;   // nt . s^
          const double nth = r0 ? nts : ntt[q];
          double S1 = 0.0, S2 = 0.0;
          if constexpr (P >= 1) {
            double Gm = cg, Fm = 1.0;                          // G_1, F_1
            S1 = Gm;
            S2 = Fm;
            if constexpr (P >= 2) {
              double Gc = 0.5 * fma(3.0 * cg, A, -rho), Fc = 3.0 * A;   // G_2, F_2
              S1 = fma(2.0, Gc, S1);
              S2 += Fc;
#pragma unroll
              for (int n = 2; n < P; ++n) {
                const double Gn = fma(c_bon.a[n] * A, Gc, -(c_bon.b[n] * B) * Gm);
                const double Fn = fma(B, Fm, (2.0 * n + 1.0) * rho * Gc);
                Gm = Gc;
                Gc = Gn;
                Fm = Fc;
                Fc = Fn;
                S1 = fma(double(n + 1), Gn, S1);
                S2 += Fn;
              }
            }
          }
          sval = fma(nth, S1, (nts - nth * cg) * S2);
        } else {
          const double nst = r0 ? nss
                                : fma(n4.z, tz[q], fma(n4.y, ty[q], n4.x * tx[q])) * ir[q];
          double Tm = 1.0, Em = 0.0;                           // T_0, E_0
          double S1 = 1.0, S2 = 0.0;
          if constexpr (P >= 1) {
            double Tc = A, Ec = rho;                           // T_1, E_1
            S1 = fma(2.0, Tc, S1);
            S2 += Ec;
#pragma unroll
            for (int n = 1; n < P; ++n) {
              const double Tn = fma(c_bon.a[n] * A, Tc, -(c_bon.b[n] * B) * Tm);
              const double En = fma(B, Em, (2.0 * n + 1.0) * rho * Tc);
              Tm = Tc;
              Tc = Tn;
              Em = Ec;
              Ec = En;
              S1 = fma(double(n + 2), Tn, S1);
              S2 += En;
            }
          }
          sval = fma(-nss, S1, (nst - nss * cg) * S2);
        }
        ar[q] = fma(sval, wr, ar[q]);
        ai[q] = fma(sval, wi, ai[q]);
        if (val) bm[q] = fmax(bm[q], B);
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1) {
        a.out[slot[q]] = make_double2(ar[q] * kInvFourPi, ai[q] * kInvFourPi);
        if (val && (!isfinite(ar[q]) || !isfinite(ai[q]) || bm[q] > kSepScreen))
          flag_suspect(a.err);
      }
    }
  }
}

template <int P, int NT, int VARIANT>
__global__ void __launch_bounds__(kSellBlock, (384 / kSellBlock > 0 ? 384 / kSellBlock : 1)) helmholtz_deriv_sell_kernel(const EvalParams a) {
  // per-thread target coefficients in (dynamic) shared memory, [term][n][q][thread]
  extern __shared__ double cfs[];
  __shared__ int4 ring[kSlots * kSellBlock];
#define CFA(n, q) cfs[((n) * NT + (q)) * kSellBlock + tid]
#define CFB(n, q) cfs[(((P + 1) + (n)) * NT + (q)) * kSellBlock + tid]
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.n_ctr) return;
  const int tid = threadIdx.x;
  const bool val = a.validate != 0;
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int len = (int)(a.nptr[g + 1] - a.nptr[g]);
  const int64_t t0 = a.tptr[g], t1 = a.tptr[g + 1];
  const double k = a.k, k2 = a.k * a.k, invk = 1.0 / a.k;
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], nx[NT], ny[NT], nz[NT], ntt[NT];
    double ar[NT], ai[NT], bm[NT];
    int64_t slot[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const bool ok = tb + q < t1;
      slot[q] = ok ? out_slot(a, tb + q) : 0;
      const double ux = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      const double uy = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      const double uz = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(uz, uz, fma(uy, uy, ux * ux));
      const double rr = sqrt(r2[q]);
      const double ir = r2[q] > 0.0 ? 1.0 / rr : 0.0;
      tx[q] = ux * ir;                                  // t^ (0 at r = 0)
      ty[q] = uy * ir;
      tz[q] = uz * ir;
      nx[q] = ny[q] = nz[q] = ntt[q] = 0.0;
      if (VARIANT == 1 && ok) {
        nx[q] = a.tnrm[3 * (tb + q)];
        ny[q] = a.tnrm[3 * (tb + q) + 1];
        nz[q] = a.tnrm[3 * (tb + q) + 2];
        ntt[q] = fma(nz[q], tz[q], fma(ny[q], ty[q], nx[q] * tx[q]));
      }
      // j_0..j_{P+1}(k r) -> term coefficients (j_n(0) = delta_n0, j'_1(0) = 1/3)
      double jn[P + 2];
      if (ok && rr > 0.0) {
        miller_j_reg<P + 2>(k * rr, jn);
      } else {
#pragma unroll
        for (int n = 0; n <= P + 1; ++n) jn[n] = (n == 0 && ok) ? 1.0 : 0.0;
      }
      const double invx = rr > 0.0 ? 1.0 / (k * rr) : 0.0;
#pragma unroll
      for (int n = 0; n <= P; ++n) {
        const double tw = 2.0 * n + 1.0;
        if (VARIANT == 1) {
          double jp = n == 0 ? -jn[1] : jn[n - 1] - (n + 1.0) * invx * jn[n];
          if (!(rr > 0.0)) jp = (n == 1 && ok) ? 1.0 / 3.0 : 0.0;
          CFA(n, q) = tw * k * jp;                        // multiplies nt.t^ P_n h_n
          CFB(n, q) = rr > 0.0 ? tw * jn[n] * ir : 0.0;   // multiplies (...) P'_n h_n
        } else {
          CFA(n, q) = tw * jn[n];               // (D allocates only the first term)
        }
      }
      ar[q] = ai[q] = bm[q] = 0.0;
    }
    SellStream<VARIANT == 2> ss(a, g, len, false, ring);
    while (ss.more()) {
      double4 q4, n4;
      double wim;
      ss.next(q4, wim, n4);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double invx = iR * invk;
      double hmr, hmi, hcr, hci;                       // h_{n-1}, h_n, starting at n = 1
      hankel01(k2 * R2, k * (R2 * iR), invx, hmr, hmi, hcr, hci);
      double nss = 0.0;
      if (VARIANT == 2) nss = fma(n4.z, dz, fma(n4.y, dy, n4.x * dx)) * iR;
      double cg[NT], pm[NT], pc[NT], dm[NT], dc[NT], ar_[NT], ai_[NT], br_[NT], bi_[NT];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const bool r0 = !(r2[q] > 0.0);
        cg[q] = r0 ? 1.0 : fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR;
        // n = 0: P_0 = 1, P'_0 = 0
        if (VARIANT == 1) {
          ar_[q] = CFA(0, q) * hmr;                   // sum c_n P_n h_n
          ai_[q] = CFA(0, q) * hmi;
        } else {
          ar_[q] = -CFA(0, q) * hcr;                  // sum c_n P_n h'_n, h'_0 = -h_1
          ai_[q] = -CFA(0, q) * hci;
        }
        br_[q] = bi_[q] = 0.0;
        pm[q] = 1.0;
        pc[q] = cg[q];
        dm[q] = 0.0;
        dc[q] = 1.0;
      }
#pragma unroll
      for (int n = 1; n <= P; ++n) {
        // here (hm, hc) = (h_{n-1}, h_n); P_n = pc, P'_n = dc
        double hpr = 0.0, hpi = 0.0;
        if (VARIANT == 2) {
          const double f = (n + 1.0) * invx;
          hpr = fma(-f, hcr, hmr);                    // h'_n = h_{n-1} - (n+1)/x h_n
          hpi = fma(-f, hci, hmi);
        }
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          const double ca = CFA(n, q) * pc[q];
          if (VARIANT == 1) {
            ar_[q] = fma(ca, hcr, ar_[q]);
            ai_[q] = fma(ca, hci, ai_[q]);
            const double cb = CFB(n, q) * dc[q];
            br_[q] = fma(cb, hcr, br_[q]);
            bi_[q] = fma(cb, hci, bi_[q]);
          } else {
            ar_[q] = fma(ca, hpr, ar_[q]);
            ai_[q] = fma(ca, hpi, ai_[q]);
            const double cb = CFA(n, q) * dc[q];
            br_[q] = fma(cb, hcr, br_[q]);
            bi_[q] = fma(cb, hci, bi_[q]);
          }
          if (n < P) {
            const double pn = fma(c_bon.a[n] * cg[q], pc[q], -c_bon.b[n] * pm[q]);
            const double dn = fma(2.0 * n + 1.0, pc[q], dm[q]);
            pm[q] = pc[q];
            pc[q] = pn;
            dm[q] = dc[q];
            dc[q] = dn;
          }
        }
        if (n < P || VARIANT == 2) {
          const double f = (2.0 * n + 1.0) * invx;
          const double hnr = fma(f, hcr, -hmr), hni = fma(f, hci, -hmi);
          hmr = hcr;
          hmi = hci;
          hcr = hnr;
          hci = hni;
        }
      }
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        double sr, si;
        if (VARIANT == 1) {
          const double nts = fma(nz[q], dz, fma(ny[q], dy, nx[q] * dx)) * iR;
          const double nth = r2[q] > 0.0 ? ntt[q] : nts;
          const double m2 = nts - nth * cg[q];
          sr = fma(nth, ar_[q], m2 * br_[q]);
          si = fma(nth, ai_[q], m2 * bi_[q]);
        } else {
          const double nst = r2[q] > 0.0
                                 ? fma(n4.z, tz[q], fma(n4.y, ty[q], n4.x * tx[q]))
                                 : nss;
          const double m1 = k * nss, m2 = (nst - nss * cg[q]) * iR;
          sr = fma(m1, ar_[q], m2 * br_[q]);
          si = fma(m1, ai_[q], m2 * bi_[q]);
        }
        ar[q] = fma(q4.w, sr, fma(-wim, si, ar[q]));
        ai[q] = fma(q4.w, si, fma(wim, sr, ai[q]));
        if (val) bm[q] = fmax(bm[q], r2[q] * (iR * iR));
      }
    }
    const double pk = k * kInvFourPi;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1) {
        a.out[slot[q]] = make_double2(-ai[q] * pk, ar[q] * pk);
        if (val && (!isfinite(ar[q]) || !isfinite(ai[q]) || bm[q] > kSepScreen))
          flag_suspect(a.err);
      }
    }
  }
#undef CFA
#undef CFB
}

// ---------------------------------------------------------------------------
// Generic per-pair arithmetic: runtime order, every variant, reference
// operation order (_core.pyx:229-306 and :365-418).  Shared by the generic
// batch kernel and the single-call kernel.
// ---------------------------------------------------------------------------
struct GenericTarget {
  double c[3];      // center
  double r;         // |t - c|
  double th[3];     // (t - c)/r, 0 at r = 0
  double nt[3];     // target normal (S')
  const double* jt;   // Helmholtz: j_n(k r), n <= p
  const double* jtp;  // Helmholtz: j'_n(k r)
};

// (sre, sim) = the kernel sum of one source (before the weight and the
// 1/(4 pi) or ik/(4 pi) factor); rho = r / R for the separation screen
__device__ __forceinline__ void generic_pair(int equation, int variant, int p, double k,
                                             const GenericTarget& T, const double4& q4,
                                             const double4* n4p, double& sre, double& sim,
                                             double& rho_out) {
  const double* c = T.c;
  const double r = T.r;
  const double* th = T.th;
  const double* nt = T.nt;
  const double* jt = T.jt;
  const double* jtp = T.jtp;
  const double sc[3] = {q4.x - c[0], q4.y - c[1], q4.z - c[2]};
  const double R = sqrt(sc[0] * sc[0] + sc[1] * sc[1] + sc[2] * sc[2]);
  const double sh[3] = {sc[0] / R, sc[1] / R, sc[2] / R};
  double cg = 1.0;
  if (r > 0.0) cg = fmin(1.0, fmax(-1.0, sh[0] * th[0] + sh[1] * th[1] + sh[2] * th[2]));
  const double rho = r / R;
  rho_out = rho;
  double ns[3] = {0.0, 0.0, 0.0};
  if (variant == 2) {
    ns[0] = n4p->x;
    ns[1] = n4p->y;
    ns[2] = n4p->z;
  }
  sre = 0.0;
  sim = 0.0;
  if (equation == 0) {
    double sum = 0.0;
    if (variant == 0) {
      double rad = 1.0 / R, pm1 = 1.0, pc = cg;
      sum = rad;
      if (p >= 1) {
        rad *= rho;
        sum += rad * pc;
      }
      for (int n = 1; n < p; ++n) {
        const double pn = ((2 * n + 1) * cg * pc - n * pm1) / (n + 1.0);
        pm1 = pc;
        pc = pn;
        rad *= rho;
        sum += rad * pc;
      }
    } else if (variant == 1) {
      const double nt_sh = nt[0] * sh[0] + nt[1] * sh[1] + nt[2] * sh[2];
      const double nt_th = r > 0.0 ? nt[0] * th[0] + nt[1] * th[1] + nt[2] * th[2] : nt_sh;
      double rad = 1.0 / (R * R), pm1 = 1.0, pc = cg, dm1 = 0.0, dc = 1.0;
      for (int n = 1; n <= p; ++n) {
        sum += rad * (n * nt_th * pc + (nt_sh - nt_th * cg) * dc);
        if (n < p) {
          const double pn = ((2 * n + 1) * cg * pc - n * pm1) / (n + 1.0);
          const double dn = dm1 + (2 * n + 1) * pc;
          pm1 = pc;
          pc = pn;
          dm1 = dc;
          dc = dn;
          rad *= rho;
        }
      }
    } else {
      const double ns_sh = ns[0] * sh[0] + ns[1] * sh[1] + ns[2] * sh[2];
      const double ns_th = r > 0.0 ? ns[0] * th[0] + ns[1] * th[1] + ns[2] * th[2] : ns_sh;
      double rad = 1.0 / (R * R), pm1 = 1.0, pc = cg, dm1 = 0.0, dc = 1.0;
      sum = rad * (-1.0 * ns_sh);
      for (int n = 1; n <= p; ++n) {
        rad *= rho;
        sum += rad * (-(n + 1.0) * ns_sh * pc + (ns_th - ns_sh * cg) * dc);
        if (n < p) {
          const double pn = ((2 * n + 1) * cg * pc - n * pm1) / (n + 1.0);
          const double dn = dm1 + (2 * n + 1) * pc;
          pm1 = pc;
          pc = pn;
          dm1 = dc;
          dc = dn;
        }
      }
    }
    sre = sum;
  } else {
    // h_0..h_{p+1}(kR) upward (_core.pyx:190-193), h'_n (:195-198)
    double hr[TSQBX_MAX_ORDER + 2], hi[TSQBX_MAX_ORDER + 2];
    const double x = k * R;
    double sn, cs;
    sincos(x, &sn, &cs);
    hr[0] = sn / x;
    hi[0] = -cs / x;
    hr[1] = hr[0] / x + hi[0];   // h0 (1/x - i)
    hi[1] = hi[0] / x - hr[0];
    for (int n = 1; n <= p; ++n) {
      const double f = (2.0 * n + 1.0) / x;
      hr[n + 1] = f * hr[n] - hr[n - 1];
      hi[n + 1] = f * hi[n] - hi[n - 1];
    }
    double pm1 = 1.0, pc = cg, dm1 = 0.0, dc = 1.0;
    const double nt_sh = nt[0] * sh[0] + nt[1] * sh[1] + nt[2] * sh[2];
    const double nt_th = nt[0] * th[0] + nt[1] * th[1] + nt[2] * th[2];
    const double ns_sh = ns[0] * sh[0] + ns[1] * sh[1] + ns[2] * sh[2];
    const double ns_th = r > 0.0 ? ns[0] * th[0] + ns[1] * th[1] + ns[2] * th[2] : ns_sh;
    for (int n = 0; n <= p; ++n) {
      const double pn = n == 0 ? 1.0 : pc;
      const double dn = n == 0 ? 0.0 : dc;
      if (n >= 1 && n < p) {
        const double pnx = ((2 * n + 1) * cg * pc - n * pm1) / (n + 1.0);
        const double dnx = dm1 + (2 * n + 1) * pc;
        pm1 = pc;
        pc = pnx;
        dm1 = dc;
        dc = dnx;
      }
      const double tw = 2.0 * n + 1.0;
      if (variant == 0) {
        const double f = tw * jt[n] * pn;
        sre += f * hr[n];
        sim += f * hi[n];
      } else if (variant == 1) {
        double f;
        if (r > 0.0)
          f = tw * (k * nt_th * jtp[n] * pn + (nt_sh - nt_th * cg) * jt[n] * dn / r);
        else
          f = tw * k * nt_sh * jtp[n] * pn;
        sre += f * hr[n];
        sim += f * hi[n];
      } else {
        double hpr, hpi;
        if (n == 0) {
          hpr = -hr[1];
          hpi = -hi[1];
        } else {
          hpr = hr[n - 1] - (n + 1.0) / x * hr[n];
          hpi = hi[n - 1] - (n + 1.0) / x * hi[n];
        }
        const double f1 = tw * jt[n] * k * ns_sh * pn;
        const double f2 = tw * jt[n] * (ns_th - ns_sh * cg) * dn / R;
        sre += f1 * hpr + f2 * hr[n];
        sim += f1 * hpi + f2 * hi[n];
      }
    }
  }
}

// Generic kernel: groups of G lanes per center, one target per pass.
__global__ void __launch_bounds__(128) generic_kernel(const EvalParams a, int equation) {
  const int G = a.G;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = gt / G;
  if (g >= a.n_ctr) return;
  const int lane = (int)(threadIdx.x & (unsigned)(G - 1));
  const unsigned mask = group_mask(G);
  const double c[3] = {a.ctr[3 * g], a.ctr[3 * g + 1], a.ctr[3 * g + 2]};
  const int64_t b = a.nptr[g], e = a.nptr[g + 1];
  const int64_t t0 = a.tptr[g], t1 = a.tptr[g + 1];
  const int p = a.p, variant = a.variant;
  const double k = a.k;

  for (int64_t it = t0; it < t1; ++it) {
    const double tc[3] = {a.tgt[3 * it] - c[0], a.tgt[3 * it + 1] - c[1],
                          a.tgt[3 * it + 2] - c[2]};
    const double r = sqrt(tc[0] * tc[0] + tc[1] * tc[1] + tc[2] * tc[2]);
    double th[3] = {0.0, 0.0, 0.0};
    if (r > 0.0) {
      th[0] = tc[0] / r;
      th[1] = tc[1] / r;
      th[2] = tc[2] / r;
    }
    double nt[3] = {0.0, 0.0, 0.0};
    if (a.tnrm) {
      nt[0] = a.tnrm[3 * it];
      nt[1] = a.tnrm[3 * it + 1];
      nt[2] = a.tnrm[3 * it + 2];
    }
    const double* jt = equation ? a.ttab + it * a.ttab_stride : nullptr;
    const double* jtp = equation ? jt + (p + 1) : nullptr;
    double accr = 0.0, acci = 0.0, bmax = 0.0;
    GenericTarget T;
    for (int d = 0; d < 3; ++d) {
      T.c[d] = c[d];
      T.th[d] = th[d];
      T.nt[d] = nt[d];
    }
    T.r = r;
    T.jt = jt;
    T.jtp = jtp;
    for (int64_t j = b + lane; j < e; j += G) {
      const int s = a.nidx[j];
      const double4 q4 = a.sp[s];
      const double wim = a.swi[s];
      double sre, sim, rho;
      generic_pair(equation, variant, p, k, T, q4, variant == 2 ? a.snrm + s : nullptr, sre, sim,
                   rho);
      if (a.validate) bmax = fmax(bmax, rho * rho);
      accr += q4.w * sre - wim * sim;
      acci += q4.w * sim + wim * sre;
    }
    accr = group_sum(accr, G, mask);
    acci = group_sum(acci, G, mask);
    if (a.validate) bmax = group_max(bmax, G, mask);
    if (lane == 0) {
      double2 o;
      if (equation == 0) {
        o = make_double2(accr / kFourPi, acci / kFourPi);
      } else {
        const double pk = k / kFourPi;
        o = make_double2(-acci * pk, accr * pk);
      }
      a.out[out_slot(a, it)] = o;
      if (a.validate && (!isfinite(accr) || !isfinite(acci) || bmax > kSepScreen))
        flag_suspect(a.err);
    }
  }
}

// ---------------------------------------------------------------------------
// Helmholtz per-target prologue: one thread per center, loops over its targets.
// mode 0 (fast S):   tab[n] = (2n+1) j_n(k r) kappa_n,        n <= p
// mode 1 (generic):  tab[n] = j_n(k r), tab[p+1+n] = j'_n(k r)  (_core.pyx:354-359)
// ---------------------------------------------------------------------------
// generic-mode row: j_n, then j'_n (_core.pyx:194-198) from Miller's j (p + 2 values)
__device__ __forceinline__ void jrow_generic(int p, double x, const double* j, double* row) {
  for (int n = 0; n <= p; ++n) row[n] = j[n];
  row[p + 1] = -j[1];
  for (int n = 1; n <= p; ++n) row[p + 1 + n] = j[n - 1] - (n + 1.0) / x * j[n];
}

__global__ void helmholtz_target_table(const double* __restrict__ ctr, int64_t n_ctr,
                                       const double* __restrict__ tgt,
                                       const int64_t* __restrict__ tptr, int p, double k,
                                       int mode, double* __restrict__ tab, int stride) {
  const int64_t ic = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ic >= n_ctr) return;
  double j[TSQBX_MAX_ORDER + 2];
  for (int64_t it = tptr[ic]; it < tptr[ic + 1]; ++it) {
    const double dx = tgt[3 * it] - ctr[3 * ic], dy = tgt[3 * it + 1] - ctr[3 * ic + 1],
                 dz = tgt[3 * it + 2] - ctr[3 * ic + 2];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    double* row = tab + it * stride;
    if (r > 0.0) {
      const double x = k * r;
      miller_j(p + 2, x, j);
      if (mode == 0) {
        double km1 = 1.0, kc = 1.0;  // kappa_{n-1}, kappa_n
        for (int n = 0; n <= p; ++n) {
          const double kap = n == 0 ? 1.0 : kc;
          row[n] = (2.0 * n + 1.0) * j[n] * kap;
          if (n >= 1) {
            const double kn = (double(n) / double(n + 1)) * km1;
            km1 = kc;
            kc = kn;
          }
        }
      } else {
        jrow_generic(p, x, j, row);
      }
    } else {
      for (int n = 0; n < stride; ++n) row[n] = 0.0;
      row[0] = 1.0;
      if (mode == 1 && p >= 1) row[p + 2] = 1.0 / 3.0;  // j'_1(0) = 1/3
    }
  }
}

__global__ void fp64_probe_kernel(double* out, int64_t iters) {
  const double a = 1.0 + 1e-9 * threadIdx.x, b = -1e-12;
  double x0 = 1.0, x1 = 2.0, x2 = 3.0, x3 = 4.0, x4 = 5.0, x5 = 6.0, x6 = 7.0, x7 = 8.0;
  for (int64_t i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void set_key(unsigned long long* key, unsigned long long v) { *key = v; }

// ---------------------------------------------------------------------------
// exact validation in the reference arithmetic (tsqbx.py:43-53): no FMA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double norm_ref(double x, double y, double z) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

__global__ void validate_kernel(const double4* __restrict__ sp, const double* __restrict__ ctr,
                                int64_t n_ctr, const int64_t* __restrict__ nptr,
                                const int32_t* __restrict__ nidx,
                                const double* __restrict__ tgt,
                                const int64_t* __restrict__ tptr,
                                unsigned long long* err) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= n_ctr) return;
  const double cx = ctr[3 * g], cy = ctr[3 * g + 1], cz = ctr[3 * g + 2];
  const int64_t b = nptr[g], e = nptr[g + 1];
  for (int64_t it = tptr[g]; it < tptr[g + 1]; ++it) {
    const double r = norm_ref(__dadd_rn(tgt[3 * it], -cx), __dadd_rn(tgt[3 * it + 1], -cy),
                              __dadd_rn(tgt[3 * it + 2], -cz));
    for (int64_t j = b + lane; j < e; j += 32) {
      const double4 q = sp[nidx[j]];
      const double R = norm_ref(__dadd_rn(q.x, -cx), __dadd_rn(q.y, -cy), __dadd_rn(q.z, -cz));
      const unsigned long long pos = (unsigned long long)(j - b);
      const unsigned long long base = (unsigned long long)it << 32;
      if (R == 0.0) atomicMin(err, base | pos);
      else if (__dmul_rn(R, 1.0 + 1e-12) < r) atomicMin(err, base | (1ull << 31) | pos);
    }
  }
}

// ---------------------------------------------------------------------------
// Single call (the reference's per-(center, target) protocol, _core.pyx:205,
// :310; tsqbx.ts_accumulate): one CTA over one staged buffer
//   [center(3) target(3) tnormal(3) |t-c|(1) pad(6)] [sp: n x double4] [Im w: n] [pad]
//   [snrm: n x double4 (D only)]
// res = {Re, Im, err_key}: the sum with the reference's scaling and, when
// validating, the exact _prep key ((kind << 31) | position, tsqbx.py:44-53).
// ---------------------------------------------------------------------------
constexpr int kOneBlock = 128;
constexpr int64_t kOneZeroCopyDoubles = 32768;   // 256 KB: below this, read the host buffer in place

__global__ void __launch_bounds__(kOneBlock) one_kernel(int equation, int variant, double k,
                                                        int p, const double* __restrict__ st,
                                                        int n, double* __restrict__ res,
                                                        int validate) {
  __shared__ double jtab[2 * (TSQBX_MAX_ORDER + 1)];
  __shared__ double red_r[kOneBlock / 32], red_i[kOneBlock / 32];
  __shared__ unsigned long long red_k[kOneBlock / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double4* sp = reinterpret_cast<const double4*>(st + 16);
  const double* swi = st + 16 + 4 * (int64_t)n;
  const double4* snrm = reinterpret_cast<const double4*>(st + 16 + 4 * (int64_t)n +
                                                         (((int64_t)n + 3) & ~(int64_t)3));
  GenericTarget T;
  const double tc[3] = {st[3] - st[0], st[4] - st[1], st[5] - st[2]};
  T.r = sqrt(tc[0] * tc[0] + tc[1] * tc[1] + tc[2] * tc[2]);
  for (int d = 0; d < 3; ++d) {
    T.c[d] = st[d];
    T.th[d] = T.r > 0.0 ? tc[d] / T.r : 0.0;
    T.nt[d] = st[6 + d];
  }
  if (equation && tid == 0) {
    const int stride = 2 * (p + 1);
    if (T.r > 0.0) {
      double j[TSQBX_MAX_ORDER + 2];
      const double x = k * T.r;
      miller_j(p + 2, x, j);
      jrow_generic(p, x, j, jtab);
    } else {
      for (int m = 0; m < stride; ++m) jtab[m] = 0.0;
      jtab[0] = 1.0;
      if (p >= 1) jtab[p + 2] = 1.0 / 3.0;     // j'_1(0) = 1/3 (_core.pyx:357-359)
    }
  }
  T.jt = jtab;
  T.jtp = jtab + (p + 1);
  __syncthreads();
  // |t - c| exactly as the caller's _prep formed it (numpy's 1-D norm is a dot
  // product whose rounding is the host's business), staged in slot 9
  const double rref = st[9];
  double accr = 0.0, acci = 0.0;
  unsigned long long key = (unsigned long long)TSQBX_ERR_KEY_NONE;
  for (int j = tid; j < n; j += kOneBlock) {
    const double4 q4 = sp[j];
    const double wim = swi[j];
    double sre, sim, rho;
    generic_pair(equation, variant, p, k, T, q4, variant == 2 ? snrm + j : nullptr, sre, sim, rho);
    accr += q4.w * sre - wim * sim;
    acci += q4.w * sim + wim * sre;
    if (validate) {
      const double R = norm_ref(__dadd_rn(q4.x, -st[0]), __dadd_rn(q4.y, -st[1]),
                                __dadd_rn(q4.z, -st[2]));
      unsigned long long kj = (unsigned long long)TSQBX_ERR_KEY_NONE;
      if (R == 0.0) kj = (unsigned long long)j;
      else if (__dmul_rn(R, 1.0 + 1e-12) < rref) kj = (1ull << 31) | (unsigned long long)j;
      key = kj < key ? kj : key;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    accr += __shfl_xor_sync(0xffffffffu, accr, off);
    acci += __shfl_xor_sync(0xffffffffu, acci, off);
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, off);
    key = ok < key ? ok : key;
  }
  if (lane == 0) {
    red_r[wid] = accr;
    red_i[wid] = acci;
    red_k[wid] = key;
  }
  __syncthreads();
  if (tid == 0) {
    accr = acci = 0.0;
    for (int w = 0; w < kOneBlock / 32; ++w) {
      accr += red_r[w];
      acci += red_i[w];
      key = red_k[w] < key ? red_k[w] : key;
    }
    if (equation == 0) {
      res[0] = accr / kFourPi;
      res[1] = acci / kFourPi;
    } else {
      const double pk = k / kFourPi;
      res[0] = -acci * pk;
      res[1] = accr * pk;
    }
    reinterpret_cast<unsigned long long*>(res)[2] = key;
  }
}

__global__ void pack_kernel(int64_t n, const double* __restrict__ xyz,
                            const double* __restrict__ w, const double* __restrict__ nrm,
                            const int32_t* __restrict__ perm, double4* __restrict__ sp,
                            double* __restrict__ swi, double4* __restrict__ snrm,
                            unsigned* __restrict__ imag_flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool imag = false;
  if (i < n) {
    const int64_t s = perm ? (int64_t)perm[i] : i;
    sp[i] = make_double4(xyz[3 * s], xyz[3 * s + 1], xyz[3 * s + 2], w[2 * s]);
    const double wi = w[2 * s + 1];
    swi[i] = wi;
    imag = wi != 0.0;
    if (nrm) snrm[i] = make_double4(nrm[3 * s], nrm[3 * s + 1], nrm[3 * s + 2], 0.0);
  }
  if (__any_sync(0xffffffffu, imag) && (threadIdx.x & 31) == 0) atomicOr(imag_flag, 1u);
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
constexpr int kMaxFastOrder = 16;

template <int P, int NT, bool VAL>
void launch_fast(int equation, bool sell, const EvalParams& a, int64_t n_ctr, cudaStream_t st) {
  if (sell) {
    const int blocks = (int)((n_ctr + kSellBlock - 1) / kSellBlock);
    if (equation == TSQBX_EQ_LAPLACE) {
      // on the SELL layout `group_lanes` is the row split S (threads per row)
      const int S = (a.G == 2 || a.G == 4) ? a.G : 1;
      const int rows = kSellBlock / S;
      const int lblocks = (int)((n_ctr + rows - 1) / rows);
      if (S == 4) laplace_sell_kernel<P, NT, VAL, 4><<<lblocks, kSellBlock, 0, st>>>(a);
      else if (S == 2) laplace_sell_kernel<P, NT, VAL, 2><<<lblocks, kSellBlock, 0, st>>>(a);
      else laplace_sell_kernel<P, NT, VAL, 1><<<lblocks, kSellBlock, 0, st>>>(a);
    } else {
      helmholtz_sell_kernel<P, NT, VAL><<<blocks, kSellBlock, 0, st>>>(a);
    }
    return;
  }
  const int blocks = (int)((n_ctr * a.G + 255) / 256);
  if (equation == TSQBX_EQ_LAPLACE)
    laplace_s_kernel<P, NT, VAL><<<blocks, 256, 0, st>>>(a);
  else
    helmholtz_s_kernel<P, NT, VAL><<<blocks, 256, 0, st>>>(a);
}

template <int P>
void launch_fast_p(int equation, bool sell, int nt, bool val, const EvalParams& a, int64_t n_ctr,
                   cudaStream_t st) {
  if (nt >= 2) {
    if (val) launch_fast<P, 2, true>(equation, sell, a, n_ctr, st);
    else launch_fast<P, 2, false>(equation, sell, a, n_ctr, st);
  } else {
    if (val) launch_fast<P, 1, true>(equation, sell, a, n_ctr, st);
    else launch_fast<P, 1, false>(equation, sell, a, n_ctr, st);
  }
}

template <int... Ps>
struct FastTable {
  static bool run(int p, int equation, bool sell, int nt, bool val, const EvalParams& a,
                  int64_t n_ctr, cudaStream_t st) {
    bool done = false;
    ((p == Ps ? (launch_fast_p<Ps>(equation, sell, nt, val, a, n_ctr, st), done = true) : false),
     ...);
    return done;
  }
};
using FastOrders = FastTable<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>;

template <int P>
void launch_deriv_p(int equation, int variant, int nt, const EvalParams& a, int64_t n_ctr,
                    cudaStream_t st) {
  const int blocks = (int)((n_ctr + kSellBlock - 1) / kSellBlock);
  if (equation == TSQBX_EQ_LAPLACE) {
    if (variant == 1) {
      if (nt >= 2) laplace_deriv_sell_kernel<P, 2, 1><<<blocks, kSellBlock, 0, st>>>(a);
      else laplace_deriv_sell_kernel<P, 1, 1><<<blocks, kSellBlock, 0, st>>>(a);
    } else {
      if (nt >= 2) laplace_deriv_sell_kernel<P, 2, 2><<<blocks, kSellBlock, 0, st>>>(a);
      else laplace_deriv_sell_kernel<P, 1, 2><<<blocks, kSellBlock, 0, st>>>(a);
    }
  } else {
    auto go = [&](auto kernel, int ntt, int terms) {
      const int smem = terms * (P + 1) * ntt * kSellBlock * (int)sizeof(double);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kernel<<<blocks, kSellBlock, smem, st>>>(a);
    };
    if (variant == 1) {
      if (nt >= 2) go(helmholtz_deriv_sell_kernel<P, 2, 1>, 2, 2);
      else go(helmholtz_deriv_sell_kernel<P, 1, 1>, 1, 2);
    } else {
      if (nt >= 2) go(helmholtz_deriv_sell_kernel<P, 2, 2>, 2, 1);
      else go(helmholtz_deriv_sell_kernel<P, 1, 2>, 1, 1);
    }
  }
}

template <int... Ps>
struct DerivTable {
  static bool run(int p, int equation, int variant, int nt, const EvalParams& a, int64_t n_ctr,
                  cudaStream_t st) {
    bool done = false;
    ((p == Ps ? (launch_deriv_p<Ps>(equation, variant, nt, a, n_ctr, st), done = true) : false),
     ...);
    return done;
  }
};
using DerivOrders = DerivTable<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>;

// [x y z Re w]*n | Im w * n | pad to 4 | [nx ny nz 0]*n (optional) | meta (4 doubles)
// meta[0] (as uint32) = 1 if any Im w != 0 (written by pack_kernel)
int64_t packed_doubles(int64_t n, int with_normals) {
  const int64_t base = (5 * n + 3) / 4 * 4;  // keep the normals 32-byte aligned
  return (with_normals ? base + 4 * n : base) + 4;
}
int64_t packed_meta_offset(int64_t n, int with_normals) {
  return packed_doubles(n, with_normals) - 4;
}

}  // namespace tsqbx

using namespace tsqbx;

extern "C" {

int tsqbx_abi_version(void) { return TSQBX_ABI_VERSION; }
const char* tsqbx_last_error(void) { return g_err; }

int tsqbx_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return TSQBX_OK;
}

int64_t tsqbx_packed_doubles(int64_t n_src, int with_normals) {
  return packed_doubles(n_src, with_normals);
}

int tsqbx_pack_sources(int64_t n_src, const double* xyz, const double* w, const double* nrm,
                       const int32_t* perm, double* packed, void* stream) {
  if (n_src < 0 || (n_src > 0 && (!xyz || !w || !packed)))
    return set_error(TSQBX_ERR_ARGUMENT, "pack_sources: bad arguments");
  if (n_src > 0 && (((uintptr_t)packed) & 31))
    return set_error(TSQBX_ERR_ARGUMENT, "pack_sources: packed buffer must be 32-byte aligned");
  if (n_src == 0) {
    if (packed) return check_cuda(cudaMemsetAsync(packed, 0, 4 * sizeof(double),
                                                  (cudaStream_t)stream), "pack memset");
    return TSQBX_OK;
  }
  const int64_t base = (5 * n_src + 3) / 4 * 4;
  double4* sp = reinterpret_cast<double4*>(packed);
  double* swi = packed + 4 * n_src;
  double4* sn = nrm ? reinterpret_cast<double4*>(packed + base) : nullptr;
  unsigned* flag = reinterpret_cast<unsigned*>(packed + packed_meta_offset(n_src, nrm != nullptr));
  cudaError_t e = cudaMemsetAsync(flag, 0, 4 * sizeof(double), (cudaStream_t)stream);
  if (e != cudaSuccess) return check_cuda(e, "pack_sources memset");
  const int blocks = (int)((n_src + 255) / 256);
  pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_src, xyz, w, nrm, perm, sp, swi, sn,
                                                          flag);
  return check_cuda(cudaGetLastError(), "pack_kernel launch");
}

int64_t tsqbx_eval_workspace_bytes(int equation, int variant, int p, int64_t n_tgt) {
  (void)variant;
  if (equation != TSQBX_EQ_HELMHOLTZ) return 0;
  // sized for the generic kernel's (j_n, j'_n) table so any flag combination fits
  return n_tgt * 2 * (p + 1) * (int64_t)sizeof(double) + 256;
}

int tsqbx_eval_packed(int equation, int variant, double k, int p, const double* packed,
                      int64_t n_src, int with_normals, const double* ctr_xyz, int64_t n_ctr,
                      const int64_t* near_ptr, const int32_t* near_idx,
                      const int64_t* sell_ptr, const int32_t* sell_idx, const double* tgt_xyz,
                      const double* tgt_nrm, const int64_t* tgt_ptr, int64_t n_tgt,
                      const int64_t* tgt_out, int64_t out_offset, unsigned flags,
                      int group_lanes, void* workspace, int64_t ws_bytes, double* out,
                      int64_t* err_key, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (equation != TSQBX_EQ_LAPLACE && equation != TSQBX_EQ_HELMHOLTZ)
    return set_error(TSQBX_ERR_ARGUMENT, "bad equation %d", equation);
  if (variant < 0 || variant > 2) return set_error(TSQBX_ERR_ARGUMENT, "bad variant %d", variant);
  if (p < 0 || p > TSQBX_MAX_ORDER)
    return set_error(TSQBX_ERR_ARGUMENT, "order p=%d outside [0, %d]", p, TSQBX_MAX_ORDER);
  if (equation == TSQBX_EQ_HELMHOLTZ && !(k > 0.0))
    return set_error(TSQBX_ERR_ARGUMENT, "Helmholtz requires k > 0");
  if (n_ctr < 0 || n_tgt < 0 || n_src < 0) return set_error(TSQBX_ERR_ARGUMENT, "negative size");
  if (variant == 2 && !with_normals)
    return set_error(TSQBX_ERR_ARGUMENT, "double-layer variant requires source normals");
  if (variant == 1 && n_tgt > 0 && !tgt_nrm)
    return set_error(TSQBX_ERR_ARGUMENT, "S' variant requires target normals");
  const bool val = (flags & TSQBX_FLAG_VALIDATE) != 0;
  if (val && !err_key) return set_error(TSQBX_ERR_ARGUMENT, "validation needs err_key");
  if (n_src > INT32_MAX) return set_error(TSQBX_ERR_ARGUMENT, "n_src exceeds int32 indexing");
  if (n_ctr > 0 && (!ctr_xyz || !near_ptr || !tgt_ptr || !out || (n_tgt > 0 && !tgt_xyz)))
    return set_error(TSQBX_ERR_ARGUMENT, "null array");
  if ((sell_ptr == nullptr) != (sell_idx == nullptr))
    return set_error(TSQBX_ERR_ARGUMENT, "sell_ptr and sell_idx go together");
  int G = group_lanes <= 0 ? 8 : group_lanes;
  if (G > 32 || (G & (G - 1))) return set_error(TSQBX_ERR_ARGUMENT, "group_lanes must be 1..32, pow2");
  if (val) set_key<<<1, 1, 0, st>>>((unsigned long long*)err_key, (unsigned long long)TSQBX_ERR_KEY_NONE);
  if (n_ctr == 0 || n_tgt == 0) return check_cuda(cudaGetLastError(), "eval");

  const bool fast = variant == 0 && p <= kMaxFastOrder && !(flags & TSQBX_FLAG_GENERIC);
  // S' / D with compile-time order on the SELL layout
  const bool fast_deriv = variant != 0 && sell_ptr && p <= kMaxFastOrder &&
                          !(flags & TSQBX_FLAG_GENERIC);
  if (!((fast || fast_deriv) && sell_ptr) && !near_idx)
    return set_error(TSQBX_ERR_ARGUMENT, "near_idx (CSR entries) required for this kernel");
  EvalParams a{};
  a.sp = reinterpret_cast<const double4*>(packed);
  a.swi = packed + 4 * n_src;
  a.snrm = with_normals ? reinterpret_cast<const double4*>(packed + (5 * n_src + 3) / 4 * 4)
                        : nullptr;
  a.imag_flag = reinterpret_cast<const unsigned*>(packed + packed_meta_offset(n_src, with_normals));
  a.ctr = ctr_xyz;
  a.nptr = near_ptr;
  a.nidx = near_idx;
  a.sell_ptr = sell_ptr;
  a.sell_idx = sell_idx;
  a.real_w = (flags & TSQBX_FLAG_REAL_WEIGHTS) ? 1 : 0;
  a.tgt = tgt_xyz;
  a.tnrm = tgt_nrm;
  a.tptr = tgt_ptr;
  a.tout = tgt_out;
  a.out_offset = out_offset;
  a.out = reinterpret_cast<double2*>(out);
  a.err = (unsigned long long*)err_key;
  a.n_ctr = n_ctr;
  a.p = p;
  a.variant = variant;
  a.G = G;
  a.log2G = __builtin_ctz((unsigned)G);
  a.validate = val ? 1 : 0;
  a.k = k;
  if (equation == TSQBX_EQ_HELMHOLTZ) {
    a.ttab_stride = fast ? p + 1 : 2 * (p + 1);
    const int64_t need = n_tgt * a.ttab_stride * (int64_t)sizeof(double);
    if (!workspace || ws_bytes < need)
      return set_error(TSQBX_ERR_ARGUMENT, "workspace too small: need %lld bytes", (long long)need);
    a.ttab = static_cast<const double*>(workspace);
    // the SELL fast kernels compute their targets' Bessel coefficients themselves
    if (!((fast || fast_deriv) && sell_ptr))
      helmholtz_target_table<<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
          ctr_xyz, n_ctr, tgt_xyz, tgt_ptr, p, k, fast ? 0 : 1, static_cast<double*>(workspace),
          a.ttab_stride);
  }
  const int nt = (n_tgt >= 2 * n_ctr && !(flags & TSQBX_FLAG_ONE_TARGET)) ? 2 : 1;
  if (fast) {
    FastOrders::run(p, equation, sell_ptr != nullptr, nt, val, a, n_ctr, st);
  } else if (fast_deriv) {
    DerivOrders::run(p, equation, variant, nt, a, n_ctr, st);
  } else {
    const int blocks = (int)((n_ctr * G + 127) / 128);
    generic_kernel<<<blocks, 128, 0, st>>>(a, equation);
  }
  return check_cuda(cudaGetLastError(), "tsqbx eval launch");
}

int64_t tsqbx_user_workspace_bytes(int equation, int variant, int p, int64_t n_src,
                                   int64_t n_tgt) {
  const int64_t packed = packed_doubles(n_src, variant == 2) * (int64_t)sizeof(double);
  return (packed + 255) / 256 * 256 + tsqbx_eval_workspace_bytes(equation, variant, p, n_tgt);
}

static int eval_user(int equation, int variant, double k, int p, const double* src_xyz,
                     const double* src_w, const double* src_nrm, int64_t n_src,
                     const double* ctr_xyz, int64_t n_ctr, const int64_t* near_ptr,
                     const int32_t* near_idx, const double* tgt_xyz, const double* tgt_nrm,
                     const int64_t* tgt_ptr, int64_t n_tgt, unsigned flags, void* workspace,
                     int64_t ws_bytes, double* out, int64_t* err_key, void* stream) {
  const int64_t need = tsqbx_user_workspace_bytes(equation, variant, p, n_src, n_tgt);
  if (!workspace || ws_bytes < need)
    return set_error(TSQBX_ERR_ARGUMENT, "workspace too small: need %lld bytes", (long long)need);
  if (variant == 2 && !src_nrm)
    return set_error(TSQBX_ERR_ARGUMENT, "double-layer variant requires source normals");
  double* packed = static_cast<double*>(workspace);
  const int64_t pbytes = (packed_doubles(n_src, variant == 2) * (int64_t)sizeof(double) + 255) /
                         256 * 256;
  int rc = tsqbx_pack_sources(n_src, src_xyz, src_w, variant == 2 ? src_nrm : nullptr, nullptr,
                              packed, stream);
  if (rc) return rc;
  return tsqbx_eval_packed(equation, variant, k, p, packed, n_src, variant == 2, ctr_xyz, n_ctr,
                           near_ptr, near_idx, nullptr, nullptr, tgt_xyz, tgt_nrm, tgt_ptr,
                           n_tgt, nullptr, 0,
                           flags, 0, static_cast<char*>(workspace) + pbytes, ws_bytes - pbytes,
                           out, err_key, stream);
}

int tsqbx_eval_laplace(int variant, int p, const double* src_xyz, const double* src_w,
                       const double* src_nrm, int64_t n_src, const double* ctr_xyz,
                       int64_t n_ctr, const int64_t* near_ptr, const int32_t* near_idx,
                       const double* tgt_xyz, const double* tgt_nrm, const int64_t* tgt_ptr,
                       int64_t n_tgt, unsigned flags, void* workspace, int64_t ws_bytes,
                       double* out, int64_t* err_key, void* stream) {
  return eval_user(TSQBX_EQ_LAPLACE, variant, 0.0, p, src_xyz, src_w, src_nrm, n_src, ctr_xyz,
                   n_ctr, near_ptr, near_idx, tgt_xyz, tgt_nrm, tgt_ptr, n_tgt, flags, workspace,
                   ws_bytes, out, err_key, stream);
}

int tsqbx_eval_helmholtz(int variant, double k, int p, const double* src_xyz,
                         const double* src_w, const double* src_nrm, int64_t n_src,
                         const double* ctr_xyz, int64_t n_ctr, const int64_t* near_ptr,
                         const int32_t* near_idx, const double* tgt_xyz, const double* tgt_nrm,
                         const int64_t* tgt_ptr, int64_t n_tgt, unsigned flags, void* workspace,
                         int64_t ws_bytes, double* out, int64_t* err_key, void* stream) {
  return eval_user(TSQBX_EQ_HELMHOLTZ, variant, k, p, src_xyz, src_w, src_nrm, n_src, ctr_xyz,
                   n_ctr, near_ptr, near_idx, tgt_xyz, tgt_nrm, tgt_ptr, n_tgt, flags, workspace,
                   ws_bytes, out, err_key, stream);
}

int tsqbx_fp64_probe(double* out, int64_t iters, int blocks, int threads, void* stream) {
  if (!out || iters <= 0 || blocks <= 0 || threads <= 0 || threads > 1024)
    return set_error(TSQBX_ERR_ARGUMENT, "fp64_probe: bad arguments");
  fp64_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters);
  return check_cuda(cudaGetLastError(), "fp64_probe launch");
}

int tsqbx_validate(const double* packed, int64_t n_src, const double* ctr_xyz, int64_t n_ctr,
                   const int64_t* near_ptr, const int32_t* near_idx,
                   const double* tgt_xyz, const int64_t* tgt_ptr, int64_t n_tgt,
                   int64_t* err_key, void* stream) {
  (void)n_src;
  (void)n_tgt;
  if (!err_key) return set_error(TSQBX_ERR_ARGUMENT, "validate: err_key is null");
  cudaStream_t st = (cudaStream_t)stream;
  set_key<<<1, 1, 0, st>>>((unsigned long long*)err_key, (unsigned long long)TSQBX_ERR_KEY_NONE);
  if (n_ctr > 0) {
    const int blocks = (int)((n_ctr * 32 + 255) / 256);
    validate_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const double4*>(packed), ctr_xyz,
                                            n_ctr, near_ptr, near_idx, tgt_xyz,
                                            tgt_ptr, (unsigned long long*)err_key);
  }
  return check_cuda(cudaGetLastError(), "validate launch");
}

int64_t tsqbx_one_staging_doubles(int64_t n_src, int with_normals) {
  return 16 + 4 * n_src + ((n_src + 3) & ~(int64_t)3) + (with_normals ? 4 * n_src : 0);
}

int tsqbx_eval_one(int equation, int variant, double k, int p, const double* staged_host,
                   int64_t n_src, unsigned flags, double* device_buf, int64_t device_doubles,
                   double* result_host, void* stream) {
  if (equation != TSQBX_EQ_LAPLACE && equation != TSQBX_EQ_HELMHOLTZ)
    return set_error(TSQBX_ERR_ARGUMENT, "eval_one: bad equation %d", equation);
  if (variant < 0 || variant > 2) return set_error(TSQBX_ERR_ARGUMENT, "eval_one: bad variant");
  if (p < 0 || p > TSQBX_MAX_ORDER) return set_error(TSQBX_ERR_ARGUMENT, "eval_one: bad order");
  if (n_src < 0 || n_src > INT32_MAX || !staged_host || !device_buf || !result_host)
    return set_error(TSQBX_ERR_ARGUMENT, "eval_one: bad arguments");
  if (equation == TSQBX_EQ_HELMHOLTZ && !(k > 0.0))
    return set_error(TSQBX_ERR_ARGUMENT, "eval_one: Helmholtz needs k > 0");
  const int64_t nd = tsqbx_one_staging_doubles(n_src, variant == TSQBX_VARIANT_D);
  if (device_doubles < nd + 4) return set_error(TSQBX_ERR_ARGUMENT, "eval_one: device buffer too small");
  const cudaStream_t st = (cudaStream_t)stream;
  // small batches: the kernel reads the pinned staging buffer and writes the
  // result in place over PCIe (mapped pinned memory under UVA) -- no copies
  if (nd <= kOneZeroCopyDoubles) {
    cudaPointerAttributes in{}, out{};
    if (cudaPointerGetAttributes(&in, staged_host) == cudaSuccess &&
        cudaPointerGetAttributes(&out, result_host) == cudaSuccess &&
        in.type == cudaMemoryTypeHost && out.type == cudaMemoryTypeHost && in.devicePointer &&
        out.devicePointer) {
      one_kernel<<<1, kOneBlock, 0, st>>>(equation, variant, k, p,
                                          static_cast<const double*>(in.devicePointer),
                                          (int)n_src, static_cast<double*>(out.devicePointer),
                                          (flags & TSQBX_FLAG_VALIDATE) ? 1 : 0);
      const cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) return check_cuda(le, "one_kernel launch");
      return check_cuda(cudaStreamSynchronize(st), "eval_one sync");
    }
    cudaGetLastError();   // not pinned: fall through to the copies
  }
  cudaError_t e = cudaMemcpyAsync(device_buf, staged_host, nd * sizeof(double),
                                  cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "eval_one H2D");
  double* dres = device_buf + ((nd + 3) & ~(int64_t)3);
  one_kernel<<<1, kOneBlock, 0, st>>>(equation, variant, k, p, device_buf, (int)n_src, dres,
                                      (flags & TSQBX_FLAG_VALIDATE) ? 1 : 0);
  e = cudaGetLastError();
  if (e != cudaSuccess) return check_cuda(e, "one_kernel launch");
  e = cudaMemcpyAsync(result_host, dres, 3 * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return check_cuda(e, "eval_one D2H");
  return check_cuda(cudaStreamSynchronize(st), "eval_one sync");
}

}  // extern "C"
