// eval_laplace.cu -- Laplace S kernels (compile-time order P <= 16): the
// SELL-32x4 thread-per-row kernel (the hot path) and the CSR group kernel.
#include "eval_bodies.cuh"

namespace tsqbx {

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

// real weights (the usual Laplace density) skip every Im w load and FMA; the
// pack kernel records whether any Im w is nonzero, so no host round trip decides
//
// S > 1 splits every row over S threads of one warp (lanes 32/S apart take
// the row's SELL blocks round-robin; a CTA covers kSellBlock/S rows).  A
// thread's row takes ~100 µs on the dense presets whatever else runs on its
// SM (latency-bound per thread), so with whole rows the last partial wave of
// rows leaves most slots idle; S rows-parts per row make the work units S
// times shorter and the tail S times cheaper.
#ifdef TSQBX_CTA_TIMING
// debug builds only (tools/cta_timing_probe.py): per-CTA start/end globaltimer and SM id
__device__ unsigned long long g_cta_t[2 * 8192];
__device__ unsigned g_cta_sm[8192];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cta_mark_start() {
  if (threadIdx.x == 0 && blockIdx.x < 8192) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_cta_t[2 * blockIdx.x] = gtimer();
    g_cta_sm[blockIdx.x] = sm;
  }
}
__device__ __forceinline__ void cta_mark_end() {
  if (blockIdx.x < 8192) atomicMax(&g_cta_t[2 * blockIdx.x + 1], gtimer());
}
}  // namespace tsqbx
extern "C" int tsqbx_debug_cta_times(unsigned long long* t, unsigned* sm, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(t, tsqbx::g_cta_t, sizeof(unsigned long long) * 2 * n);
  cudaMemcpyFromSymbol(sm, tsqbx::g_cta_sm, sizeof(unsigned) * n);
  static unsigned long long zero[2 * 8192];
  cudaMemcpyToSymbol(tsqbx::g_cta_t, zero, sizeof(zero));
  return 0;
}
namespace tsqbx {
#define CTA_START() cta_mark_start()
#define CTA_END() cta_mark_end()
#else
#define CTA_START()
#define CTA_END()
#endif

template <int P, int NT, bool VAL, int S, int UNI>
__global__ void __launch_bounds__(kSellBlock, NT == 1 ? TSQBX_LAP_MINB1 : (UNI > 0 ? TSQBX_LAP_MINB_UNI : TSQBX_LAP_MINB)) laplace_sell_kernel(const EvalParams a) {
  CTA_START();
  __shared__ int4 ring[kSlots * kSellBlock];
  constexpr int kRowsPerWarp = 32 / S;
  const int lane = threadIdx.x & 31;
  const int part = lane / kRowsPerWarp, rig = lane % kRowsPerWarp;
  const int64_t g = (int64_t)blockIdx.x * (kSellBlock / S) + (threadIdx.x >> 5) * kRowsPerWarp + rig;
  unsigned gmask = 0u;
#pragma unroll
  for (int k = 0; k < S; ++k) gmask |= 1u << (rig + k * kRowsPerWarp);
  if (g < a.n_ctr) {
    const RowHead h = load_head<UNI>(a, g);
    const bool realw = a.real_w || *a.imag_flag == 0u;
    if (realw)
      laplace_sell_body<P, NT, VAL, true, S>(a, g, h, ring, part, gmask);
    else
      laplace_sell_body<P, NT, VAL, false, S>(a, g, h, ring, part, gmask);
  }
  CTA_END();
}

// Two rows per thread (short near lists, uniform target runs): a warp takes two
// adjacent slices, lane l rows 64 w + l (A) and 64 w + 32 + l (B) -- Morton
// neighbours, so both rows gather from the same L1-resident sources.  Both rows' heads are loaded and
// both index rings start filling before row A computes, so row B's dependent
// chain (slice offset -> index block -> source record) is served while row A
// evaluates instead of in a second wave of threads.
#ifndef TSQBX_LAP_MINB2
#define TSQBX_LAP_MINB2 3
#endif
template <int P, int NT, bool VAL, int UNI>
__global__ void __launch_bounds__(kSellBlock, TSQBX_LAP_MINB2) laplace_sell2_kernel(const EvalParams a) {
  __shared__ int4 ring[2][kSlots * kSellBlock];
  const int64_t ga = ((int64_t)blockIdx.x * (kSellBlock / 32) + (threadIdx.x >> 5)) * 64 +
                     (threadIdx.x & 31);
  const int64_t gb = ga + 32;
  if (ga >= a.n_ctr) return;
  const bool has_b = gb < a.n_ctr;
  const RowHead ha = load_head<UNI>(a, ga);
  RowHead hb{};
  if (has_b) hb = load_head<UNI>(a, gb);
  const bool realw = a.real_w || *a.imag_flag == 0u;
  using Stream = SellStream<false, (P >= 12 ? 2 : TSQBX_GATHER_DEPTH)>;
  { Stream pre(a, ha.soff, ga, ha.len, realw, ring[0], false); }   // A's first blocks
  if (has_b) { Stream pre(a, hb.soff, gb, hb.len, realw, ring[1], false); }   // then B's
  if (realw) {
    laplace_sell_body<P, NT, VAL, true, 1>(a, ga, ha, ring[0], 0, 0xffffffffu, true, has_b);
    if (has_b) laplace_sell_body<P, NT, VAL, true, 1>(a, gb, hb, ring[1], 0, 0xffffffffu, true);
  } else {
    laplace_sell_body<P, NT, VAL, false, 1>(a, ga, ha, ring[0], 0, 0xffffffffu, true, has_b);
    if (has_b) laplace_sell_body<P, NT, VAL, false, 1>(a, gb, hb, ring[1], 0, 0xffffffffu, true);
  }
}

constexpr int kWinRecBytes = (kSellBlock / 32) * TSQBX_WINDOW * 32;
constexpr int kWinSmemBytes = kWinRecBytes + (kSellBlock / 32) * TSQBX_WINDOW * 8;

// Windowed SELL (short lists, tsqbx_sell_window): every warp is one slice; it
// stages its slice's distinct sources (<= TSQBX_WINDOW records) in shared
// memory once -- all loads independent, issued together -- while its rows'
// index rings fill, and the rows then read their sources from the window
// instead of one dependent global gather per entry.
template <int P, int NT, bool VAL, int UNI>
__global__ void __launch_bounds__(kSellBlock, NT == 1 ? TSQBX_LAP_MINB1 : TSQBX_LAP_MINB_UNI)
    laplace_sellw_kernel(const EvalParams a) {
  __shared__ int4 ring[kSlots * kSellBlock];
  // dynamic: [8 warps][W] double4 records, then [8 warps][W] Im w
  extern __shared__ __align__(16) unsigned char win_smem[];
  double4* wq_all = reinterpret_cast<double4*>(win_smem);
  double* wwi_all = reinterpret_cast<double*>(win_smem + kWinRecBytes);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double4* wq = wq_all + w * TSQBX_WINDOW;
  double* wwi = wwi_all + w * TSQBX_WINDOW;
  const int64_t g = (int64_t)blockIdx.x * kSellBlock + threadIdx.x;
  const int64_t s = g >> 5;
  if ((s << 5) >= a.n_ctr) return;                 // warp-uniform
  const bool valid = g < a.n_ctr;
  RowHead h{};
  if (valid) h = load_head<UNI>(a, g);
  const bool realw = a.real_w || *a.imag_flag == 0u;
  if (valid) {                                     // this row's first index blocks
    SellStream<false, TSQBX_GATHER_DEPTH, true> pre(a, h.soff, g, h.len, realw, ring, false);
  }
  const int wl = a.win_len[s];
  for (int i = lane; i < wl; i += 32) {
    const int j = a.win_src[s * TSQBX_WINDOW + i];
    wq[i] = ld256(a.sp + j);
    if (!realw) wwi[i] = __ldg(a.swi + j);
  }
  __syncwarp();
  if (!valid) return;
  if (wl < 0) {            // an overflowed slice: global indices, global gathers
    if (realw) laplace_sell_body<P, NT, VAL, true, 1>(a, g, h, ring, 0, 0xffffffffu, true);
    else laplace_sell_body<P, NT, VAL, false, 1>(a, g, h, ring, 0, 0xffffffffu, true);
    return;
  }
  if (realw)
    laplace_sell_body<P, NT, VAL, true, 1, true>(a, g, h, ring, 0, 0xffffffffu, true, false,
                                                 wq, wwi);
  else
    laplace_sell_body<P, NT, VAL, false, 1, true>(a, g, h, ring, 0, 0xffffffffu, true, false,
                                                  wq, wwi);
}

template <template <int> class F, int... Ps>
struct OrderTable {
  template <class... Args>
  static bool run(int p, Args&&... args) {
    bool done = false;
    ((p == Ps ? (F<Ps>::go(args...), done = true) : false), ...);
    return done;
  }
};

template <int P>
struct LaplaceLaunch {
  template <int NT, bool VAL, int UNI>
  static void sell_launch(int S, int blocks, const EvalParams& a, cudaStream_t st) {
    if (S == 4) laplace_sell_kernel<P, NT, VAL, 4, UNI><<<blocks, kSellBlock, 0, st>>>(a);
    else if (S == 2) laplace_sell_kernel<P, NT, VAL, 2, UNI><<<blocks, kSellBlock, 0, st>>>(a);
    else laplace_sell_kernel<P, NT, VAL, 1, UNI><<<blocks, kSellBlock, 0, st>>>(a);
  }
  template <int NT, bool VAL>
  static void one(bool sell, const EvalParams& a, int64_t n_ctr, cudaStream_t st) {
    if (sell) {
      // on the SELL layout `group_lanes` is the row split S (threads per row)
      const int S = (a.G == 2 || a.G == 4) ? a.G : 1;
      if (S == 1 && a.win_src && a.tuni == NT) {
        // the window exceeds the 48 KB default; per call (the attribute is per device)
        cudaFuncSetAttribute(laplace_sellw_kernel<P, NT, VAL, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kWinSmemBytes);
        laplace_sellw_kernel<P, NT, VAL, NT><<<(int)((n_ctr + kSellBlock - 1) / kSellBlock),
                                               kSellBlock, kWinSmemBytes, st>>>(a);
        return;
      }
      if (S == 1 && a.two_rows && a.tuni == NT) {
        const int blocks2 = (int)((n_ctr + 2 * kSellBlock - 1) / (2 * kSellBlock));
        laplace_sell2_kernel<P, NT, VAL, NT><<<blocks2, kSellBlock, 0, st>>>(a);
        return;
      }
      const int rows = kSellBlock / S;
      const int blocks = (int)((n_ctr + rows - 1) / rows);
      if (a.tuni == NT) sell_launch<NT, VAL, NT>(S, blocks, a, st);
      else sell_launch<NT, VAL, 0>(S, blocks, a, st);
      return;
    }
    laplace_s_kernel<P, NT, VAL><<<(int)((n_ctr * a.G + 255) / 256), 256, 0, st>>>(a);
  }
  static void go(bool sell, int nt, bool val, const EvalParams& a, int64_t n_ctr,
                 cudaStream_t st) {
    if (nt >= 2) {
      if (val) one<2, true>(sell, a, n_ctr, st);
      else one<2, false>(sell, a, n_ctr, st);
    } else {
      if (val) one<1, true>(sell, a, n_ctr, st);
      else one<1, false>(sell, a, n_ctr, st);
    }
  }
};

bool launch_laplace_fast(int p, bool sell, int nt, bool val, const EvalParams& a, int64_t n_ctr,
                         cudaStream_t st) {
  return OrderTable<LaplaceLaunch, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::run(
      p, sell, nt, val, a, n_ctr, st);
}

}  // namespace tsqbx
