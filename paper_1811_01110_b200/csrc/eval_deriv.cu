// eval_deriv.cu -- S' and D kernels (Laplace and Helmholtz, compile-time
// order P <= 16) on the SELL-32x4 layout.
#include "eval_kernels.cuh"

namespace tsqbx {

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
// Laplace S'/D run the kappa-scaled recurrence of common.cuh (X_n = G_n / kappa_n,
// U_n = T_n / kappa_n: U_{n+1} = alpha_n A U_n - B U_{n-1}, 3 DP per order) and
// carry the P' ladder divided by rho (W_n = E_n / rho, Y_n = (F_n - delta_n) / rho:
// W_{n+1} = B W_{n-1} + (2n+1) kappa_n U_n, 2 DP per order); the sums use the
// constant weights kd = (n+1) kappa_n, kn = n kappa_n, ke = (2n+1) kappa_n.
#ifndef TSQBX_LAP_DERIV_MINB
#define TSQBX_LAP_DERIV_MINB 2   // CTAs per SM requested from ptxas (Laplace S'/D)
#endif

struct Bonnet {
  double a[TSQBX_MAX_ORDER + 2], b[TSQBX_MAX_ORDER + 2];
  double kap[TSQBX_MAX_ORDER + 2], alp[TSQBX_MAX_ORDER + 2];
  double kd[TSQBX_MAX_ORDER + 2], kn[TSQBX_MAX_ORDER + 2], ke[TSQBX_MAX_ORDER + 2];
  constexpr Bonnet() : a(), b(), kap(), alp(), kd(), kn(), ke() {
    for (int n = 0; n < TSQBX_MAX_ORDER + 2; ++n) {
      a[n] = double(2 * n + 1) / double(n + 1);
      b[n] = double(n) / double(n + 1);
    }
    kap[0] = 1.0;
    kap[1] = 1.0;
    for (int n = 1; n + 1 < TSQBX_MAX_ORDER + 2; ++n) kap[n + 1] = b[n] * kap[n - 1];
    for (int n = 1; n + 1 < TSQBX_MAX_ORDER + 2; ++n) alp[n] = a[n] * kap[n] / kap[n + 1];
    for (int n = 0; n < TSQBX_MAX_ORDER + 2; ++n) {
      kd[n] = double(n + 1) * kap[n];
      kn[n] = double(n) * kap[n];
      ke[n] = double(2 * n + 1) * kap[n];
    }
  }
};
static __constant__ Bonnet c_bon = Bonnet();

// UNI = NT: uniform target runs (TSQBX_FLAG_UNIFORM_TARGETS), no tgt_ptr loads
template <int P, int NT, int VARIANT, int UNI>
__global__ void __launch_bounds__(kSellBlock, TSQBX_LAP_DERIV_MINB) laplace_deriv_sell_kernel(const EvalParams a) {
  __shared__ int4 ring[kSlots * kSellBlock];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.n_ctr) return;
  const bool val = a.validate != 0;
  const bool realw = a.real_w || *a.imag_flag == 0u;
  const double cx = a.ctr[3 * g], cy = a.ctr[3 * g + 1], cz = a.ctr[3 * g + 2];
  const int len = (int)(a.nptr[g + 1] - a.nptr[g]);
  const int64_t t0 = UNI > 0 ? a.tbase + g * UNI : a.tptr[g], t1 = UNI > 0 ? t0 + UNI : a.tptr[g + 1];
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], rr[NT], ir[NT], nx[NT], ny[NT], nz[NT], ntt[NT];
    double ar[NT], ai[NT];
    long long rmin = 0x7ff0000000000000ll;   // min |s-c|^2 bits (see eval_laplace.cu)
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
      ar[q] = ai[q] = 0.0;
    }
    SellStream<VARIANT == 2> ss(a, g, len, realw, ring);
    while (ss.more()) {
      double4 q4, n4;
      double wim;
      ss.next(q4, wim, n4);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      if (val) rmin = min(rmin, __double_as_longlong(R2));
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
            // S1 = sum n G_n = sum kn_n X_n;  S2 = sum F_n = rho sum Y_n + sum_{odd n} B^((n-1)/2)
            double Xm = cg, Ym = 0.0;                          // X_1 = G_1, Y_1
            S1 = Xm;
            double Sy = 0.0;
            if constexpr (P >= 2) {
              double Xc = fma(3.0 * cg, A, -rho), Yc = 3.0 * cg;   // X_2 = G_2 / kappa_2, Y_2
              S1 = fma(c_bon.kn[2], Xc, S1);
              Sy = Yc;
#pragma unroll
              for (int n = 2; n < P; ++n) {
                const double Xn = fma(c_bon.alp[n] * A, Xc, -(B * Xm));
                const double Yn = fma(B, Ym, c_bon.ke[n] * Xc);
                Xm = Xc;
                Xc = Xn;
                Ym = Yc;
                Yc = Yn;
                S1 = fma(c_bon.kn[n + 1], Xn, S1);
                Sy += Yn;
              }
            }
            double gs = 1.0;                                   // F_1's ladder: 1 + B + B^2 ...
#pragma unroll
            for (int i = 1; i <= (P - 1) / 2; ++i) gs = fma(gs, B, 1.0);
            S2 = fma(rho, Sy, gs);
          }
          sval = fma(nth, S1, (nts - nth * cg) * S2);
        } else {
          const double nst = r0 ? nss
                                : fma(n4.z, tz[q], fma(n4.y, ty[q], n4.x * tx[q])) * ir[q];
          // S1 = sum (n+1) T_n = sum kd_n U_n;  S2 = sum E_n = rho sum W_n
          double Um = 1.0, Wm = 0.0;                           // U_0, W_0
          double S1 = 1.0, S2 = 0.0;
          if constexpr (P >= 1) {
            double Uc = A, Wc = 1.0;                           // U_1, W_1 = E_1 / rho
            S1 = fma(2.0, Uc, S1);
            double Sw = Wc;
#pragma unroll
            for (int n = 1; n < P; ++n) {
              const double Un = fma(c_bon.alp[n] * A, Uc, -(B * Um));
              const double Wn = fma(B, Wm, c_bon.ke[n] * Uc);
              Um = Uc;
              Uc = Un;
              Wm = Wc;
              Wc = Wn;
              S1 = fma(c_bon.kd[n + 1], Un, S1);
              Sw += Wn;
            }
            S2 = rho * Sw;
          }
          sval = fma(-nss, S1, (nst - nss * cg) * S2);
        }
        ar[q] = fma(sval, wr, ar[q]);
        ai[q] = fma(sval, wi, ai[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1) {
        a.out[slot[q]] = make_double2(ar[q] * kInvFourPi, ai[q] * kInvFourPi);
        if (val && (!isfinite(ar[q]) || !isfinite(ai[q]) || r2[q] > kSepScreen * __longlong_as_double(rmin)))
          flag_suspect(a.err);
      }
    }
  }
}

template <int P, int NT, int VARIANT, int UNI>
// CTAs per SM requested from ptxas: D at 2 (~128 registers, some spills: C3
// literal D +18 %, dense equal); S' at 1 (184-198 registers: 2 CTAs cost C3
// dense S' 11 %)
__global__ void __launch_bounds__(kSellBlock, VARIANT == 2 ? 2 : 1) helmholtz_deriv_sell_kernel(const EvalParams a) {
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
  const int64_t t0 = UNI > 0 ? a.tbase + g * UNI : a.tptr[g], t1 = UNI > 0 ? t0 + UNI : a.tptr[g + 1];
  const double k = a.k, k2 = a.k * a.k, invk = 1.0 / a.k;
  for (int64_t tb = t0; tb < t1; tb += NT) {
    double tx[NT], ty[NT], tz[NT], r2[NT], nx[NT], ny[NT], nz[NT], ntt[NT];
    double ar[NT], ai[NT];
    long long rmin = 0x7ff0000000000000ll;   // min |s-c|^2 bits (see eval_laplace.cu)
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
        sph_j_reg<P + 2>(k * rr, jn);
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
          CFA(n, q) = tw * k * jp * c_bon.kap[n];         // multiplies nt.t^ U_n h_n
          CFB(n, q) = rr > 0.0 ? tw * jn[n] * ir : 0.0;   // multiplies (...) P'_n h_n
        } else {
          CFA(n, q) = tw * jn[n];               // (D allocates only the first term)
        }
      }
      ar[q] = ai[q] = 0.0;
    }
    SellStream<VARIANT == 2> ss(a, g, len, false, ring);
    while (ss.more()) {
      double4 q4, n4;
      double wim;
      ss.next(q4, wim, n4);
      const double dx = q4.x - cx, dy = q4.y - cy, dz = q4.z - cz;
      const double R2 = fma(dz, dz, fma(dy, dy, dx * dx));
      if (val) rmin = min(rmin, __double_as_longlong(R2));
      const double iR = rsqrt_fast(R2);
      const double invx = iR * invk;
      double hmr, hmi, hcr, hci;                       // h_{n-1}, h_n, starting at n = 1
      hankel01(a.sc, k2 * R2, k * (R2 * iR), invx, hmr, hmi, hcr, hci, a.series);
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
        // here (hm, hc) = (h_{n-1}, h_n); P_n = pc (S': kappa_n pc), P'_n = dc
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
            // S': kappa-scaled Legendre (pc = U_n = P_n / kappa_n, kappa_n folded
            // into CFA); D weights P_n and P'_n with the same CFA, so it keeps P_n
            double pn, dn;
            if (VARIANT == 1) {
              pn = fma(c_bon.alp[n] * cg[q], pc[q], -pm[q]);
              dn = fma(c_bon.ke[n], pc[q], dm[q]);        // P'_{n+1} = P'_{n-1} + (2n+1) P_n
            } else {
              pn = fma(c_bon.a[n] * cg[q], pc[q], -c_bon.b[n] * pm[q]);
              dn = fma(2.0 * n + 1.0, pc[q], dm[q]);
            }
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
      }
    }
    const double pk = k * kInvFourPi;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (tb + q < t1) {
        a.out[slot[q]] = make_double2(-ai[q] * pk, ar[q] * pk);
        if (val && (!isfinite(ar[q]) || !isfinite(ai[q]) || r2[q] > kSepScreen * __longlong_as_double(rmin)))
          flag_suspect(a.err);
      }
    }
  }
#undef CFA
#undef CFB
}

template <int P>
void launch_deriv_p(int equation, int variant, int nt, const EvalParams& a, int64_t n_ctr,
                    cudaStream_t st) {
  const int blocks = (int)((n_ctr + kSellBlock - 1) / kSellBlock);
  if (equation == TSQBX_EQ_LAPLACE) {
#define LAP_DK(NT_, V_) (a.tuni == NT_ ? laplace_deriv_sell_kernel<P, NT_, V_, NT_> \
                                          : laplace_deriv_sell_kernel<P, NT_, V_, 0>)
    if (variant == 1) {
      if (nt >= 2) LAP_DK(2, 1)<<<blocks, kSellBlock, 0, st>>>(a);
      else LAP_DK(1, 1)<<<blocks, kSellBlock, 0, st>>>(a);
    } else {
      if (nt >= 2) LAP_DK(2, 2)<<<blocks, kSellBlock, 0, st>>>(a);
      else LAP_DK(1, 2)<<<blocks, kSellBlock, 0, st>>>(a);
    }
#undef LAP_DK
  } else {
    auto go = [&](auto kernel, int ntt, int terms) {
      const int smem = terms * (P + 1) * ntt * kSellBlock * (int)sizeof(double);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kernel<<<blocks, kSellBlock, smem, st>>>(a);
    };
#define HELM_DK(NT_, V_) (a.tuni == NT_ ? helmholtz_deriv_sell_kernel<P, NT_, V_, NT_> \
                                           : helmholtz_deriv_sell_kernel<P, NT_, V_, 0>)
    if (variant == 1) {
      if (nt >= 2) go(HELM_DK(2, 1), 2, 2);
      else go(HELM_DK(1, 1), 1, 2);
    } else {
      // D keeps the tgt_ptr kernel: its uniform-target build allocates worse
      // (C3 dense D 1.078 -> 1.159 ms)
      if (nt >= 2) go(helmholtz_deriv_sell_kernel<P, 2, 2, 0>, 2, 1);
      else go(helmholtz_deriv_sell_kernel<P, 1, 2, 0>, 1, 1);
    }
#undef HELM_DK
  }
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
struct DerivLaunch {
  static void go(int equation, int variant, int nt, const EvalParams& a, int64_t n_ctr,
                 cudaStream_t st) {
    launch_deriv_p<P>(equation, variant, nt, a, n_ctr, st);
  }
};

bool launch_deriv_fast(int p, int equation, int variant, int nt, const EvalParams& a,
                       int64_t n_ctr, cudaStream_t st) {
  return OrderTable<DerivLaunch, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::run(
      p, equation, variant, nt, a, n_ctr, st);
}

}  // namespace tsqbx
