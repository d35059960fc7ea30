// eval_helmholtz.cu -- Helmholtz S kernels (compile-time order P <= 16): the
// SELL-32x4 thread-per-row kernel and the CSR group kernel.
#include "eval_kernels.cuh"

// 1: the SELL S kernel sums over orders by Clenshaw on the Hankel recurrence
// (5 DP instructions per order); 0: forward complex Hankel recurrence (8)
#ifndef TSQBX_HELM_CLENSHAW
#define TSQBX_HELM_CLENSHAW 1
#endif

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
  // per-thread target coefficients c_n = (2n+1) j_n(k r) kappa_n, in registers
  // (a shared-memory copy measured slower)
  // one target per center: the coefficients live in shared memory (fewer
  // registers, fewer spills: C5 literal +9 %, dense +2 %); with two targets the
  // register copy is faster (C3 dense -1.5 % from shared memory)
  constexpr bool kCfShared = NT == 1 && !CFR;
  constexpr bool kClenshaw = TSQBX_HELM_CLENSHAW != 0;
  extern __shared__ double cfs[];
  double cfr[kCfShared ? 1 : NT][kCfShared ? 1 : P + 1];
  auto cf = [&](int n, int q) -> double& {
    if constexpr (kCfShared) return cfs[(n * NT + q) * kSellBlock + threadIdx.x];
    else return cfr[q][n];
  };
#define CF(n, q) cf(n, q)
  __shared__ int4 ring[kSlots * kSellBlock];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < a.n_ctr) {
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int len = (int)(a.nptr[g + 1] - a.nptr[g]);
  const int64_t t0 = UNI > 0 ? a.tbase + g * UNI : a.tptr[g], t1 = UNI > 0 ? t0 + UNI : a.tptr[g + 1];
  const double k = a.k, k2 = a.k * a.k, invk = 1.0 / a.k;
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], ar[NT], ai[NT];
    // VAL: min |s-c|^2 over the row as its IEEE bit pattern (R^2 >= 0, so the
    // integer order is the numeric order): integer-pipe min, screen r^2 > R^2
    long long rmin = 0x7ff0000000000000ll;
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
          sph_j_reg<P + 1>(k * rr, jn);
        } else {
#pragma unroll
          for (int n = 0; n <= P; ++n) jn[n] = n == 0 && ok ? 1.0 : 0.0;
        }
#pragma unroll
        for (int n = 0; n <= P; ++n)
          CF(n, q) = kClenshaw ? c_leg.hsc[n] * jn[n] : (2.0 * n + 1.0) * jn[n] * c_leg.kappa[n];
      }
      ar[q] = ai[q] = 0.0;
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
      hankel01(a.sc, k2 * R2, k * (R2 * iR), invx, hmr, hmi, hcr, hci, a.series);
      double cg[NT], pm[NT], pc[NT], sr[NT], si[NT];
      if constexpr (kClenshaw) {
        // sum_n a_n h_n, a_n = c_n P_n(cos g) real, by Clenshaw over the Hankel
        // recurrence h_{n+1} = (2n+1) u h_n - h_{n-1} (u = 1/x, _core.pyx:192-193):
        // y_n = a_n + (2n+1) u y_{n+1} - y_{n+2}, sum = h_0 (a_0 - y_2) + h_1 y_1.
        // With g_n = (2n-1)!! y_n the middle coefficient is u itself:
        // g_n = (2n-1)!! a_n + u g_{n+1} - g_{n+2} / ((2n+1)(2n+3)), y_1 = g_1,
        // y_2 = g_2 / 3.  The scaled a'_n = (2n-1)!! a_n come from the Legendre
        // recurrence (stored: Clenshaw runs downward), so each order costs 5 DP
        // instructions (Legendre 2, a'_n 1, Clenshaw 2) against 8 for the
        // forward complex Hankel recurrence -- and the h_n are never formed.
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          cg[q] = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR;
          double ap[P + 1];
          if constexpr (P >= 1) {
            double um = 1.0, uc = cg[q];
            ap[1] = CF(1, q) * uc;
#pragma unroll
            for (int n = 1; n < P; ++n) {
              const double un = fma(c_leg.alpha[n] * cg[q], uc, -um);
              um = uc;
              uc = un;
              ap[n + 1] = CF(n + 1, q) * un;
            }
          }
          double g1 = 0.0, g2 = 0.0;            // g_{n+1}, g_{n+2}
          if constexpr (P >= 1) {
            g1 = ap[P];                          // g_P
            if constexpr (P >= 2) {
              g2 = g1;
              g1 = fma(invx, g2, ap[P - 1]);     // g_{P-1}
            }
#pragma unroll
            for (int n = P - 2; n >= 1; --n) {
              const double g = fma(invx, g1, fma(-c_leg.gam[n], g2, ap[n]));
              g2 = g1;
              g1 = g;
            }
          }
          // sum = h_0 (a_0 - g_2 / 3) + h_1 g_1
          const double t0 = P >= 2 ? fma(-1.0 / 3.0, g2, CF(0, q)) : CF(0, q);
          sr[q] = fma(hcr, g1, hmr * t0);
          si[q] = fma(hci, g1, hmi * t0);
        }
      } else {
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
      }   // forward recurrence
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        ar[q] = fma(q4.w, sr[q], fma(-wim, si[q], ar[q]));
        ai[q] = fma(q4.w, si[q], fma(wim, sr[q], ai[q]));
      }
      if (VAL) rmin = min(rmin, __double_as_longlong(R2));
    }
    const double pk = k * kInvFourPi;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1) {
        a.out[slot[q]] = make_double2(-ai[q] * pk, ar[q] * pk);  // (ik/4pi) acc
        if (VAL && (!isfinite(ar[q]) || !isfinite(ai[q]) || r2[q] > kSepScreen * __longlong_as_double(rmin)))
          flag_suspect(a.err);
      }
    }
  }
}  // rows
}
#undef CF

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
