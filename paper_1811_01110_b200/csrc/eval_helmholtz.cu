// eval_helmholtz.cu -- Helmholtz S kernels (compile-time order P <= 16): the
// SELL-32x4 thread-per-row kernel and the CSR group kernel.
#include "eval_bodies.cuh"

namespace tsqbx {

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
        hankel01(a.sc, k2 * R2, x, invx, hr[0], hi[0], h1r, h1i);
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

// UNI = NT: uniform target runs (row g owns targets [NT g, NT g + NT)), one
// pass and no tgt_ptr loads (TSQBX_FLAG_UNIFORM_TARGETS)
// CFR (one target per center only): 1 = the target coefficients in registers
// with 2 CTAs per SM instead of shared memory with 3 -- long rows (dense
// presets: C5 dense -2 %), where the extra warps of the 3-CTA build only help
// short rows hide their per-row latency (C5 literal +14 %)
template <int P, int NT, bool VAL, int UNI, int CFR = 0>
__global__ void __launch_bounds__(kSellBlock, NT == 1 ? (CFR ? 2 : TSQBX_HELM_MINB1) : TSQBX_HELM_MINB) helmholtz_sell_kernel(const EvalParams a) {
  extern __shared__ double cfs[];
  __shared__ int4 ring[kSlots * kSellBlock];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < a.n_ctr)
    helmholtz_sell_row<P, NT, VAL, UNI, CFR>(a, g, -1, (int)(a.nptr[g + 1] - a.nptr[g]), cfs, ring);
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
struct HelmholtzLaunch {
  template <int NT, bool VAL>
  static void one(bool sell, const EvalParams& a, int64_t n_ctr, cudaStream_t st) {
    if (sell)
    {
      const int grid = (int)((n_ctr + kSellBlock - 1) / kSellBlock);
      bool done = false;
      if constexpr (NT == 1) {
        if (a.long_rows) {
          (a.tuni == NT ? helmholtz_sell_kernel<P, NT, VAL, NT, 1>
                        : helmholtz_sell_kernel<P, NT, VAL, 0, 1>)<<<grid, kSellBlock, 0, st>>>(a);
          done = true;
        }
      }
      if (!done) {
        const int smem = NT == 1 ? (P + 1) * kSellBlock * (int)sizeof(double) : 0;
        (a.tuni == NT ? helmholtz_sell_kernel<P, NT, VAL, NT>
                      : helmholtz_sell_kernel<P, NT, VAL, 0>)<<<grid, kSellBlock, smem, st>>>(a);
      }
    }
    else
      helmholtz_s_kernel<P, NT, VAL><<<(int)((n_ctr * a.G + 255) / 256), 256, 0, st>>>(a);
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

bool launch_helmholtz_fast(int p, bool sell, int nt, bool val, const EvalParams& a,
                           int64_t n_ctr, cudaStream_t st) {
  return OrderTable<HelmholtzLaunch, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15,
                    16>::run(p, sell, nt, val, a, n_ctr, st);
}

}  // namespace tsqbx
