// eval_flat.cu -- Laplace S for short near lists (the literal presets, ~7-20
// sources per center).
//
// The SELL kernels give every thread one row: with a dozen entries per row and
// lengths that differ within a warp, the lanes of short rows idle while the
// longest row of the warp finishes (C2 literal: FP64 pipe 53 % busy for 38 % of
// the peak in useful pairs).  Here a warp takes 32 consecutive rows (processing
// order) and splits their CSR entries evenly over its lanes -- lane l takes the
// consecutive entries [l K, l K + K) of the warp's range -- so every lane
// evaluates the same number of pairs however the rows' lengths vary.
//
// Row data (center, targets relative to it, |t - c|^2, output slots) is staged
// once per row in shared memory by the row's own lane; a lane walking its
// entries switches rows at the row starts.  A row that lies inside one lane's
// range is finished by that lane; a row cut by lane boundaries is finished by
// the lane holding its start after a segmented suffix sum over the lanes that
// hold its remaining pieces (warp shuffles, once per warp) -- the summation
// order is fixed, results are deterministic.
//
// Reference: the per-(center, target) sum of _core.pyx:205-307 (Laplace S),
// same arithmetic as laplace_sell_kernel (rescaled-Bonnet Clenshaw series).
#include "eval_kernels.cuh"

namespace tsqbx {

template <int NT>
struct FlatRow {
  double cx, cy, cz;
  double tx[NT], ty[NT], tz[NT], r2[NT];
  long long slot[NT];
};

constexpr int kFlatBlock = 256;   // 8 warps, each one slice of 32 rows
#ifndef TSQBX_FLAT_MINB
#define TSQBX_FLAT_MINB 3
#endif

// NT = targets per row (uniform target runs only: row g owns tbase + NT g ...)
template <int P, int NT, bool VAL, bool REALW>
__device__ __forceinline__ void laplace_flat_warp(const EvalParams& a, int64_t g0,
                                                  FlatRow<NT>* rows, int* start) {
  const int lane = threadIdx.x & 31;
  const int64_t g = g0 + lane;
  const int64_t gl = min(g, a.n_ctr);
  const int64_t e_lane = a.nptr[gl];
  const int64_t e_end = a.nptr[min(g0 + 32, a.n_ctr)];
  const int64_t e0 = __shfl_sync(0xffffffffu, e_lane, 0);
  const int E = (int)(e_end - e0);
  // this lane's row: record for the walkers; an empty row is written here
  start[lane] = (int)(e_lane - e0);
  if (lane == 31) start[32] = E;
  if (g < a.n_ctr) {
    FlatRow<NT>& R = rows[lane];
    const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
    R.cx = cx;
    R.cy = cy;
    R.cz = cz;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const int64_t t = a.tbase + g * NT + q;
      const double tx = a.tgt[3 * t] - cx, ty = a.tgt[3 * t + 1] - cy, tz = a.tgt[3 * t + 2] - cz;
      R.tx[q] = tx;
      R.ty[q] = ty;
      R.tz[q] = tz;
      R.r2[q] = fma(tz, tz, fma(ty, ty, tx * tx));
      R.slot[q] = out_slot(a, t);
    }
    if (a.nptr[g + 1] == e_lane) {          // no near sources: the potential is 0
#pragma unroll
      for (int q = 0; q < NT; ++q) a.out[R.slot[q]] = make_double2(0.0, 0.0);
    }
  }
  __syncwarp();

  // this lane's entries [lo, hi) of the warp's range
  const int K = (E + 31) >> 5;
  const int lo = min(lane * K, E), hi = min(lo + K, E);
  // the row holding entry lo: the last row starting at or before it (empty
  // rows share their start with the next row, so the last one is non-empty)
  int r = 0;
  if (lo < hi) {
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (r + step < 32 && start[r + step] <= lo) r += step;
  }
  const int r_first = r;
  double cx = 0, cy = 0, cz = 0, tx[NT], ty[NT], tz[NT], r2[NT];
  auto load_row = [&](int rr) {
    const FlatRow<NT>& R = rows[rr];
    cx = R.cx;
    cy = R.cy;
    cz = R.cz;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      tx[q] = R.tx[q];
      ty[q] = R.ty[q];
      tz[q] = R.tz[q];
      r2[q] = R.r2[q];
    }
  };
  load_row(r);
  int next = start[r + 1];
  double ar[NT], ai[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) ar[q] = ai[q] = 0.0;
  long long rmin = 0x7ff0000000000000ll;
  // the piece of a row that started before lo (finished by the row's start lane)
  double har[NT], hai[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) har[q] = hai[q] = 0.0;
  long long hmin = 0x7ff0000000000000ll;
  int hrow = -1;

  auto write_row = [&](int rr, const double* sr, const double* si, long long mn) {
    const FlatRow<NT>& R = rows[rr];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      a.out[R.slot[q]] = make_double2(sr[q] * kInvFourPi, si[q] * kInvFourPi);
      if (VAL && (!isfinite(sr[q]) || !isfinite(si[q]) ||
                  R.r2[q] > kSepScreen * __longlong_as_double(mn)))
        flag_suspect(a.err);
    }
  };
  // a row ends inside this lane's range: complete if it started here, else
  // it is the head piece of a row whose start lane finishes it
  auto close_row = [&]() {
    if (start[r] >= lo) {
      write_row(r, ar, ai, rmin);
    } else {
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        har[q] = ar[q];
        hai[q] = ai[q];
      }
      hmin = rmin;
      hrow = r;
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) ar[q] = ai[q] = 0.0;
    rmin = 0x7ff0000000000000ll;
  };

  SourceStream ss(a.nidx + e0 + lo, 1, hi - lo, a.sp, a.swi, REALW);
  for (int e = lo; e < hi; ++e) {
    if (e == next) {
      close_row();
      do {
        ++r;
      } while (start[r + 1] <= e);
      next = start[r + 1];
      load_row(r);
    }
    double4 q4;
    double wim;
    ss.next(q4, wim);
    const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
    const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
    const double iR = rsqrt_fast(R2);
    const double iR2 = iR * iR;
    const double wr = q4.w * iR;
    const double wi = REALW ? 0.0 : wim * iR;
    if (VAL) rmin = min(rmin, __double_as_longlong(R2));
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const double A = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR2;
      const double B = r2[q] * iR2;
      const double ser = laplace_series<P>(A, B);
      ar[q] = fma(ser, wr, ar[q]);
      if (!REALW) ai[q] = fma(ser, wi, ai[q]);
    }
  }
  // the row open at hi: complete if it started here and ends at hi; a tail
  // piece (started here, continues) waits for the other lanes' pieces
  int trow = -1;
  if (lo < hi) {
    if (next == hi) {
      close_row();
    } else if (start[r] < lo) {                 // the lane's range lies inside row r
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        har[q] = ar[q];
        hai[q] = ai[q];
      }
      hmin = rmin;
      hrow = r;
    } else {
      trow = r;
    }
  }
  (void)r_first;
  // segmented suffix sum of the head pieces over lanes with the same row (a
  // row's pieces sit in consecutive lanes); the start lane adds lane + 1's sum
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int kr = __shfl_down_sync(0xffffffffu, hrow, off);
    const bool take = lane + off < 32 && hrow >= 0 && kr == hrow;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const double vr = __shfl_down_sync(0xffffffffu, har[q], off);
      const double vi = REALW ? 0.0 : __shfl_down_sync(0xffffffffu, hai[q], off);
      if (take) {
        har[q] += vr;
        if (!REALW) hai[q] += vi;
      }
    }
    if (VAL) {
      const long long vm = __shfl_down_sync(0xffffffffu, hmin, off);
      if (take) hmin = min(hmin, vm);
    }
  }
  const int nrow = __shfl_down_sync(0xffffffffu, hrow, 1);
  double nr[NT], ni[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    nr[q] = __shfl_down_sync(0xffffffffu, har[q], 1);
    ni[q] = REALW ? 0.0 : __shfl_down_sync(0xffffffffu, hai[q], 1);
  }
  const long long nmin = __shfl_down_sync(0xffffffffu, hmin, 1);
  if (trow >= 0) {
    // pieces of row trow in lanes lane+1 ... (always at least one: the row
    // continues past hi, and the next lane's range starts at hi)
    const bool more = lane < 31 && nrow == trow;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      ar[q] += more ? nr[q] : 0.0;
      if (!REALW) ai[q] += more ? ni[q] : 0.0;
    }
    if (VAL && more) rmin = min(rmin, nmin);
    write_row(trow, ar, ai, rmin);
  }
}

template <int P, int NT, bool VAL>
__global__ void __launch_bounds__(kFlatBlock, TSQBX_FLAT_MINB) laplace_flat_kernel(const EvalParams a) {
  __shared__ FlatRow<NT> rows[kFlatBlock / 32][32];
  __shared__ int start[kFlatBlock / 32][33];
  const int w = threadIdx.x >> 5;
  const int64_t g0 = ((int64_t)blockIdx.x * (kFlatBlock / 32) + w) * 32;
  if (g0 >= a.n_ctr) return;
  const bool realw = a.real_w || *a.imag_flag == 0u;
  if (realw)
    laplace_flat_warp<P, NT, VAL, true>(a, g0, rows[w], start[w]);
  else
    laplace_flat_warp<P, NT, VAL, false>(a, g0, rows[w], start[w]);
}

template <int P>
struct FlatLaunch {
  static void go(int nt, bool val, const EvalParams& a, int64_t n_ctr, cudaStream_t st) {
    const int blocks = (int)((n_ctr + kFlatBlock - 1) / kFlatBlock);
    if (nt >= 2) {
      if (val) laplace_flat_kernel<P, 2, true><<<blocks, kFlatBlock, 0, st>>>(a);
      else laplace_flat_kernel<P, 2, false><<<blocks, kFlatBlock, 0, st>>>(a);
    } else {
      if (val) laplace_flat_kernel<P, 1, true><<<blocks, kFlatBlock, 0, st>>>(a);
      else laplace_flat_kernel<P, 1, false><<<blocks, kFlatBlock, 0, st>>>(a);
    }
  }
};

template <template <int> class F, int... Ps>
struct FlatOrders {
  template <class... Args>
  static bool run(int p, Args&&... args) {
    bool done = false;
    ((p == Ps ? (F<Ps>::go(args...), done = true) : false), ...);
    return done;
  }
};

bool launch_laplace_flat(int p, int nt, bool val, const EvalParams& a, int64_t n_ctr,
                         cudaStream_t st) {
  return FlatOrders<FlatLaunch, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::run(
      p, nt, val, a, n_ctr, st);
}

}  // namespace tsqbx
