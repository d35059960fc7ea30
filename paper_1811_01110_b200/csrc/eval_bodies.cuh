// eval_bodies.cuh -- the per-row bodies of the SELL-32x4 S kernels (Laplace
// and Helmholtz), shared by their stand-alone kernels (eval_laplace.cu,
// eval_helmholtz.cu) and the fused build+evaluate kernel (fused.cu).
#pragma once

#include <type_traits>

#include "eval_kernels.cuh"

// 1: the SELL S kernel sums over orders by Clenshaw on the Hankel recurrence
// (5 DP instructions per order); 0: forward complex Hankel recurrence (8)
#ifndef TSQBX_HELM_CLENSHAW
#define TSQBX_HELM_CLENSHAW 1
#endif

namespace tsqbx {

template <int P, int NT, bool VAL, bool REALW, int S = 1, bool WIN = false>
__device__ __forceinline__ void laplace_sell_body(const EvalParams& a, int64_t g,
                                                  const RowHead& h, int4* ring, int part = 0,
                                                  unsigned gmask = 0xffffffffu,
                                                  bool issued = false, bool foreign = false,
                                                  const double4* win_q = nullptr,
                                                  const double* win_w = nullptr) {
  const double cx = h.cx, cy = h.cy, cz = h.cz;
  const int len = h.len;
  const int64_t t0 = h.t0, t1 = h.t1;
  // high orders have more arithmetic per source to cover a second gather in
  // flight (measured: C4 literal p = 12 +7 %; p = 8 -2 %); split rows (S > 1,
  // the dense presets) keep one in flight (C4 dense +2.2 %)
  using Stream = SellStream<false, (P >= 12 && S == 1 && !WIN ? 2 : TSQBX_GATHER_DEPTH), WIN>;
  // the index ring starts filling before the target range is known
  Stream ss(a, h.soff, g, len, REALW, ring, false, part, S, issued, foreign, win_q, win_w);
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
      tx[q] = ok ? a.tgt[3 * (tb + q)] - cx : 0.0;
      ty[q] = ok ? a.tgt[3 * (tb + q) + 1] - cy : 0.0;
      tz[q] = ok ? a.tgt[3 * (tb + q) + 2] - cz : 0.0;
      r2[q] = fma(tz[q], tz[q], fma(ty[q], ty[q], tx[q] * tx[q]));
      ar[q] = ai[q] = 0.0;
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
      if (VAL) rmin = min(rmin, __double_as_longlong(R2));
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const double A = fma(dz, tz[q], fma(dy, ty[q], dx * tx[q])) * iR2;
        const double B = r2[q] * iR2;
        const double ser = laplace_series<P>(A, B);
        ar[q] = fma(ser, wr, ar[q]);
        if (!REALW) ai[q] = fma(ser, wi, ai[q]);
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
        }
        if (VAL) rmin = min(rmin, __shfl_xor_sync(gmask, rmin, off));
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1 && part == 0) {
        a.out[slot[q]] = make_double2(ar[q] * kInvFourPi, ai[q] * kInvFourPi);
        if (VAL && (!isfinite(ar[q]) || !isfinite(ai[q]) || r2[q] > kSepScreen * __longlong_as_double(rmin)))
          flag_suspect(a.err);
      }
    }
  }
  if (t0 >= t1) cp_async_wait<0>();   // no pass consumed the ring: drain it before exit
}

// One row of the Helmholtz S SELL kernel (row g, its SELL slice at `soff`
// entries from a.sell_idx, or a.sell_ptr[g / 32] when soff < 0; `len` near
// sources): shared by helmholtz_sell_kernel and the fused build+evaluate kernel.
// cfs: the kernel's dynamic shared memory (one target per center, CFR = 0).
template <int P, int NT, bool VAL, int UNI, int CFR>
__device__ __forceinline__ void helmholtz_sell_row(const EvalParams& a, int64_t g, int64_t soff,
                                                   int len, double* cfs, int4* ring) {
  // per-thread target coefficients c_n = (2n+1) j_n(k r) kappa_n, in registers
  // (a shared-memory copy measured slower)
  // one target per center: the coefficients live in shared memory (fewer
  // registers, fewer spills: C5 literal +9 %, dense +2 %); with two targets the
  // register copy is faster (C3 dense -1.5 % from shared memory)
  constexpr bool kCfShared = NT == 1 && !CFR;
  constexpr bool kClenshaw = TSQBX_HELM_CLENSHAW != 0;
  double cfr[kCfShared ? 1 : NT][kCfShared ? 1 : P + 1];
  auto cf = [&](int n, int q) -> double& {
    if constexpr (kCfShared) return cfs[(n * NT + q) * kSellBlock + threadIdx.x];
    else return cfr[q][n];
  };
#define CF(n, q) cf(n, q)
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
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
    // A single dependent DFMA chain fills the FP64 pipe of an SM to 66 % at
    // most (tools/micro/dp_chain.cu), so the chains of one source -- 1/R, the
    // two Horner chains of sin/cos, the Legendre recurrence, the Clenshaw
    // recurrence -- should sit in ONE basic block for the scheduler to
    // interleave; hankel01's choice of series branches per source and cuts the
    // block in three.  kStruct picks how the choice is made (measured per
    // kernel family, C5/C3 dense and literal):
    //   2 (one target, long rows): the row's loop exists once per series
    //     (LOOP_ 1 narrow, 2 wide, 0 per-source choice with the library
    //     fallback), picked outside the loop from the k R hint, so a source's
    //     whole arithmetic is one block (C5 dense 12.31 -> 11.86 ms).  The hint
    //     is checked per row on the integer pipe (largest R^2 as its bit
    //     pattern); a row that violates it is recomputed on the generic loop.
    //   1 (two targets): one warp-uniform branch per source picks the series
    //     and everything after it is one block (C3 dense 0.506 -> 0.497 ms).
    //   0 (one target, short rows): hankel01 as it is -- the copies of the
    //     loop cost the short rows more than the interleaving gives (C5
    //     literal 0.619 ms against 0.647 / 0.680 ms).
    constexpr int kStruct = NT == 1 ? (CFR ? 2 : 0) : 1;
    long long rmax = 0;
    auto run = [&](auto loop_tag) {
    constexpr int LOOP_ = decltype(loop_tag)::value;
#pragma unroll
    for (int q = 0; q < NT; ++q) ar[q] = ai[q] = 0.0;
    SellStream<> ss(a, soff >= 0 ? soff : a.sell_ptr[g >> 5], g, len, false, ring, true);
    while (ss.more()) {
      double4 q4;
      double wim;
      ss.next(q4, wim);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double iR = rsqrt_fast(R2);
      const double invx = iR * invk;
      auto rest = [&](auto series_tag) {
      constexpr int MODE_ = decltype(series_tag)::value;
      double hmr, hmi, hcr, hci;                 // h_{n-1}, h_n
      if constexpr (MODE_ == 0) {
        // (kStruct 2 gets here without a hint or after the hint failed: series 0)
        hankel01(a.sc, k2 * R2, k * (R2 * iR), invx, hmr, hmi, hcr, hci,
                 kStruct == 2 ? 0 : a.series);
      } else {
        double sinc, cs;
        sinc_cos_series<MODE_ == 2>(a.sc, k2 * R2, sinc, cs);
        hmr = sinc;
        hmi = -cs * invx;
        hcr = fma(hmr, invx, hmi);
        hci = fma(hmi, invx, -hmr);
      }
      double cg[NT], sr[NT], si[NT];
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
      double pm[NT], pc[NT];
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
      };
      if constexpr (kStruct == 1) {
        // the series picked per source by a warp-uniform branch; everything
        // after it is one basic block
        if (a.series == 1) rest(std::integral_constant<int, 1>{});
        else if (a.series == 2 && __all_sync(__activemask(), k2 * R2 <= kWideX2))
          rest(std::integral_constant<int, 2>{});
        else rest(std::integral_constant<int, 0>{});
      } else {
        rest(loop_tag);
      }
      if (VAL) rmin = min(rmin, __double_as_longlong(R2));
      if (kStruct == 2 && LOOP_ != 0) rmax = max(rmax, __double_as_longlong(R2));
    }
    };
    if constexpr (kStruct == 2) {
      // (an explicit fourth copy for the recomputation: folding it into a loop
      // over `series` costs 9 % on C5 dense)
      if (a.series == 1) run(std::integral_constant<int, 1>{});
      else if (a.series == 2) run(std::integral_constant<int, 2>{});
      else run(std::integral_constant<int, 0>{});
      if (a.series != 0 &&
          k2 * __longlong_as_double(rmax) > (a.series == 1 ? kSmallX2 : kWideX2) * (1.0 + 1e-9))
        run(std::integral_constant<int, 0>{});   // the k R hint does not hold for this row
    } else {
      run(std::integral_constant<int, 0>{});
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
}
#undef CF

}  // namespace tsqbx
