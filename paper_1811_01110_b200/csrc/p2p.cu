// p2p.cu -- point-to-point direct interactions on sm_100a.
//
// The reference's `laplace_p2p` / `helmholtz_p2p` (_core.pyx:94-165): for
// every target, out = sum_j w_j K(t, s_j) with K the free-space kernel
// (S: 1/(4 pi r), e^{ikr}/(4 pi r); S' / D: its target / source normal
// derivative).  Two callers in the reference:
//   * kernels.direct_sum (kernels.py:114-136): every target sees every source
//     ("dense");
//   * driver.direct_stage (driver.py:187-210): per target box, the box's
//     conventional targets see the sources of the box's interaction list
//     ("rows": row r = targets [row_tgt[r], row_tgt[r+1]) over the sources
//     row_idx[row_ptr[r] .. row_ptr[r+1])).
//
// Design.  A CTA of 128 threads owns a tile of TT targets (TT a power of two
// <= 128) and streams its sources through shared memory in tiles of 128
// records (the packed {x, y, z, Re w} + Im w (+ normal) layout of
// tsqbx_pack_sources); the 128 / TT "source lanes" that share a target split
// each tile and are reduced in a fixed order at the end (deterministic).  A
// dense sum over few targets also splits the sources over blockIdx.y chunks
// whose partial sums a second kernel adds in chunk order.  The per-pair work is
// FP64-pipe bound (rsqrt, sincos), so the design goal is just to keep the
// FP64 pipe fed: every source record is read from HBM/L2 once per CTA and
// broadcast from shared memory to all target lanes.
//
// Singular pairs (r2 == 0, the reference's ValueError) are screened: such a
// pair makes the sum non-finite, the kernel flags TSQBX_ERR_KEY_SUSPECT and
// tsqbx_p2p_find_singular locates the first (target-major) pair exactly; a
// non-finite sum with no singular pair (ftz of a subnormal r2) is recomputed
// by the caller with TSQBX_FLAG_PRECISE (IEEE division and sqrt).
#include <algorithm>
#include <cstdio>

#include "common.cuh"

namespace tsqbx {

int64_t packed_doubles(int64_t n, int with_normals);

namespace {

constexpr int kP2PBlock = 128;   // threads per CTA == sources per shared tile
#ifndef TSQBX_P2P_TPT
#define TSQBX_P2P_TPT 4
#endif
constexpr int kP2PTpt = TSQBX_P2P_TPT;   // targets per thread on large dense sums
// Helmholtz e^{ikr}: Cody-Waite reduction + the near-minimax pair (sincos_cw)
// instead of the library sincos
#ifndef TSQBX_P2P_CW
#define TSQBX_P2P_CW 1
#endif

struct P2PParams {
  const double4* __restrict__ sp;     // {x, y, z, Re w}
  const double* __restrict__ swi;     // Im w
  const double4* __restrict__ snrm;   // {nx, ny, nz, 0} (D only)
  const double* __restrict__ tgt;
  const double* __restrict__ tnrm;    // S' only
  const int64_t* __restrict__ row_tgt;
  const int64_t* __restrict__ row_ptr;  // null: dense
  const int32_t* __restrict__ row_idx;
  double* __restrict__ out;           // (n_tgt, 2)
  double* __restrict__ part;          // dense chunks > 1: (chunks, n_tgt, 2)
  unsigned long long* err;
  int64_t n_src, n_tgt, n_rows, chunk_len;
  int log2_tt;
  int screen;
  double k;
};

// Per-pair kernel values, accumulated unscaled (the 1/(4 pi) is applied once
// per target).  d = t - s, exactly the reference's dx, dy, dz.
template <int EQ, int VARIANT, bool PRECISE>
struct PairKernel {
  double tnx, tny, tnz;
  double k;

  __device__ __forceinline__ void add(double dx, double dy, double dz, double wr, double wi,
                                      const double4& sn, double& ar, double& ai) const {
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    double rinv;
    if (PRECISE) rinv = 1.0 / sqrt(r2);
    else rinv = rsqrt_fast(r2);
    if (EQ == TSQBX_EQ_LAPLACE) {
      if (VARIANT == TSQBX_VARIANT_S) {
        ar = fma(wr, rinv, ar);
        ai = fma(wi, rinv, ai);
      } else {
        // S': -nu_t.d / r^3 (_core.pyx:117-119); D: +nu_s.d / r^3 (:120-123)
        const double dot = VARIANT == TSQBX_VARIANT_SPRIME
                               ? fma(tnz, dz, fma(tny, dy, tnx * dx))
                               : -fma(sn.z, dz, fma(sn.y, dy, sn.x * dx));
        const double c = dot * (rinv * rinv) * rinv;
        ar = fma(-wr, c, ar);
        ai = fma(-wi, c, ai);
      }
    } else {
      const double r = r2 * rinv;
      double s, co;
#if TSQBX_P2P_CW
      sincos_cw(k * r, s, co);
#else
      sincos(k * r, &s, &co);
#endif
      if (VARIANT == TSQBX_VARIANT_S) {
        // w e^{ikr} / r (_core.pyx:151-152)
        const double pr = co * rinv, pi = s * rinv;
        ar = fma(wr, pr, fma(-wi, pi, ar));
        ai = fma(wr, pi, fma(wi, pr, ai));
      } else {
        // radial = e^{ikr} (ikr - 1) / r^3 (:154); S': +w nu_t.d radial, D: -w nu_s.d radial
        const double dot = VARIANT == TSQBX_VARIANT_SPRIME
                               ? fma(tnz, dz, fma(tny, dy, tnx * dx))
                               : -fma(sn.z, dz, fma(sn.y, dy, sn.x * dx));
        const double kr = k * r;
        const double c = dot * (rinv * rinv) * rinv;
        const double qr = fma(-s, kr, -co) * c;    // Re[(co + i s)(-1 + i kr)] * c
        const double qi = fma(co, kr, -s) * c;     // Im
        ar = fma(wr, qr, fma(-wi, qi, ar));
        ai = fma(wr, qi, fma(wi, qr, ai));
      }
    }
  }
};

struct SourceTile {
  double4 q[kP2PBlock];
  double wi[kP2PBlock];
  double4 n[kP2PBlock];
};

// Accumulate sources [j0, j1) of the current list (dense: consecutive; rows:
// through row_idx) into (ar, ai)[k] for the thread's TPT targets; source lane
// `si` of `sl` takes every sl-th source of a tile.  TPT independent targets
// per thread give the FP64 pipe independent dependency chains (one pair's
// chain -- d, r2, rsqrt, accumulate -- is ~11 dependent FP64 operations).
template <int EQ, int VARIANT, bool PRECISE, int TPT>
__device__ __forceinline__ void p2p_stream(const P2PParams& a, SourceTile& st, int64_t j0,
                                           int64_t j1, bool indexed, int si, int sl,
                                           const double (&tx)[TPT], const double (&ty)[TPT],
                                           const double (&tz)[TPT],
                                           const PairKernel<EQ, VARIANT, PRECISE> (&K)[TPT],
                                           double (&ar)[TPT], double (&ai)[TPT]) {
  const int tid = threadIdx.x;
  for (int64_t jb = j0; jb < j1; jb += kP2PBlock) {
    const int nt = (int)min((int64_t)kP2PBlock, j1 - jb);
    __syncthreads();
    if (tid < nt) {
      const int64_t s = indexed ? (int64_t)a.row_idx[jb + tid] : jb + tid;
      st.q[tid] = ld256(a.sp + s);
      st.wi[tid] = __ldg(a.swi + s);
      if (VARIANT == TSQBX_VARIANT_D) st.n[tid] = ld256(a.snrm + s);
    }
    __syncthreads();
#pragma unroll(TPT == 1 ? 4 : 1)
    for (int j = si; j < nt; j += sl) {
      const double4 q = st.q[j];
      const double wi = st.wi[j];
      const double4 sn = VARIANT == TSQBX_VARIANT_D ? st.n[j] : make_double4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < TPT; ++u)
        K[u].add(tx[u] - q.x, ty[u] - q.y, tz[u] - q.z, q.w, wi, sn, ar[u], ai[u]);
    }
  }
}

// CTA = 128 threads = (128 >> log2_tt) source lanes x (1 << log2_tt) target
// lanes; each target lane owns TPT targets spaced by the lane count.
// CTAs per SM requested from ptxas: 8 (64 registers) for Helmholtz and the
// Laplace double layer (65536^2: Helmholtz S / S' / D +3 / +10 / +12 %, Laplace
// D +8 %); the Laplace S and S' kernels keep their natural allocation (S' -23 %
// at 8).
template <int EQ, int VARIANT, bool PRECISE, int TPT>
__global__ void __launch_bounds__(kP2PBlock, (EQ == TSQBX_EQ_HELMHOLTZ || VARIANT == 2) ? 8 : 1) p2p_kernel(P2PParams a) {
  __shared__ SourceTile st;
  __shared__ double2 red[kP2PBlock];
  const int tid = threadIdx.x;
  const int tl = 1 << a.log2_tt;                // target lanes
  const int tile = tl * TPT;                    // targets per pass
  const int ti = tid & (tl - 1), si = tid >> a.log2_tt, sl = kP2PBlock >> a.log2_tt;
  const bool dense = a.row_ptr == nullptr;

  // dense: one target tile per blockIdx.x, sources chunk blockIdx.y;
  // rows: one row per blockIdx.x, all of its target tiles in turn
  int64_t t_begin, t_end, j0, j1;
  if (dense) {
    t_begin = (int64_t)blockIdx.x * tile;
    t_end = min(t_begin + tile, a.n_tgt);
    j0 = (int64_t)blockIdx.y * a.chunk_len;
    j1 = min(j0 + a.chunk_len, a.n_src);
  } else {
    const int64_t r = blockIdx.x;
    t_begin = a.row_tgt[r];
    t_end = a.row_tgt[r + 1];
    j0 = a.row_ptr[r];
    j1 = a.row_ptr[r + 1];
  }
  for (int64_t tb = t_begin; tb < t_end; tb += tile) {
    PairKernel<EQ, VARIANT, PRECISE> K[TPT];
    double tx[TPT], ty[TPT], tz[TPT], ar[TPT], ai[TPT];
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      const int64_t t = tb + ti + (int64_t)u * tl;
      K[u].k = a.k;
      tx[u] = ty[u] = tz[u] = 0.0;
      K[u].tnx = K[u].tny = K[u].tnz = 0.0;
      ar[u] = ai[u] = 0.0;
      if (t < t_end) {
        tx[u] = a.tgt[3 * t];
        ty[u] = a.tgt[3 * t + 1];
        tz[u] = a.tgt[3 * t + 2];
        if (VARIANT == TSQBX_VARIANT_SPRIME) {
          K[u].tnx = a.tnrm[3 * t];
          K[u].tny = a.tnrm[3 * t + 1];
          K[u].tnz = a.tnrm[3 * t + 2];
        }
      }
    }
    p2p_stream<EQ, VARIANT, PRECISE, TPT>(a, st, j0, j1, !dense, si, sl, tx, ty, tz, K, ar, ai);
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      if (sl > 1) {
        red[tid] = make_double2(ar[u], ai[u]);
        __syncthreads();
        if (si == 0) {
          for (int q = 1; q < sl; ++q) {
            const double2 v = red[ti + (q << a.log2_tt)];
            ar[u] += v.x;
            ai[u] += v.y;
          }
        }
        __syncthreads();
      }
      const int64_t t = tb + ti + (int64_t)u * tl;
      if (si == 0 && t < t_end) {
        if (a.part) {
          reinterpret_cast<double2*>(a.part)[(int64_t)blockIdx.y * a.n_tgt + t] =
              make_double2(ar[u], ai[u]);
        } else {
          const double vr = ar[u] * kInvFourPi, vi = ai[u] * kInvFourPi;
          reinterpret_cast<double2*>(a.out)[t] = make_double2(vr, vi);
          if (a.screen && !(isfinite(vr) && isfinite(vi)))
            atomicMin(a.err, (unsigned long long)TSQBX_ERR_KEY_SUSPECT);
        }
      }
    }
  }
}

// Dense chunked sums: out[t] = (1/4pi) sum_c part[c][t], chunks in order.
__global__ void p2p_reduce_kernel(const double2* __restrict__ part, int64_t chunks, int64_t n_tgt,
                                  double2* __restrict__ out, int screen,
                                  unsigned long long* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tgt) return;
  double ar = 0.0, ai = 0.0;
  for (int64_t c = 0; c < chunks; ++c) {
    const double2 v = part[c * n_tgt + t];
    ar += v.x;
    ai += v.y;
  }
  ar *= kInvFourPi;
  ai *= kInvFourPi;
  out[t] = make_double2(ar, ai);
  if (screen && !(isfinite(ar) && isfinite(ai)))
    atomicMin(err, (unsigned long long)TSQBX_ERR_KEY_SUSPECT);
}

// Many chunks, few targets: a warp per target, lane l adds chunks l, l+32, ...
// and a fixed shuffle tree combines the lanes (deterministic).
__global__ void p2p_reduce_warp_kernel(const double2* __restrict__ part, int64_t chunks,
                                       int64_t n_tgt, double2* __restrict__ out, int screen,
                                       unsigned long long* err) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n_tgt) return;
  double ar = 0.0, ai = 0.0;
  for (int64_t c = lane; c < chunks; c += 32) {
    const double2 v = part[c * n_tgt + t];
    ar += v.x;
    ai += v.y;
  }
  for (int off = 16; off > 0; off >>= 1) {
    ar += __shfl_xor_sync(0xffffffffu, ar, off);
    ai += __shfl_xor_sync(0xffffffffu, ai, off);
  }
  if (lane == 0) {
    ar *= kInvFourPi;
    ai *= kInvFourPi;
    out[t] = make_double2(ar, ai);
    if (screen && !(isfinite(ar) && isfinite(ai)))
      atomicMin(err, (unsigned long long)TSQBX_ERR_KEY_SUSPECT);
  }
}

// Exact singular-pair search (r2 == 0; the fused and unfused sums of squares
// vanish together): key = (target << 32) | source, minimised.
__global__ void p2p_singular_kernel(const double4* __restrict__ sp, int64_t n_src,
                                    const double* __restrict__ tgt, int64_t n_tgt,
                                    const int64_t* __restrict__ row_tgt,
                                    const int64_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ row_idx, int64_t n_rows,
                                    unsigned long long* err) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n_tgt) return;
  int64_t j0 = 0, j1 = n_src;
  if (row_ptr) {
    int64_t lo = 0, hi = n_rows;   // the row owning t: row_tgt[lo] <= t < row_tgt[lo + 1]
    while (hi - lo > 1) {
      const int64_t m = (lo + hi) >> 1;
      if (row_tgt[m] <= t) lo = m; else hi = m;
    }
    j0 = row_ptr[lo];
    j1 = row_ptr[lo + 1];
  }
  const double tx = tgt[3 * t], ty = tgt[3 * t + 1], tz = tgt[3 * t + 2];
  for (int64_t q = j0 + lane; q < j1; q += 32) {
    const int64_t s = row_ptr ? (int64_t)row_idx[q] : q;
    const double4 v = sp[s];
    const double dx = tx - v.x, dy = ty - v.y, dz = tz - v.z;
    if (dx * dx + dy * dy + dz * dz == 0.0)
      atomicMin(err, ((unsigned long long)t << 32) | (unsigned long long)s);
  }
}

__global__ void p2p_set_key(unsigned long long* key, unsigned long long v) { *key = v; }

// per-device SM counts (a process may drive several GPUs; B200 has 148)
static int g_sms[64] = {0};

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 148;      // B200; only reached for size queries without a device
  }
  if (g_sms[dev] == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      g_sms[dev] = n;
    else
      g_sms[dev] = 148;
    cudaGetLastError();
  }
  return g_sms[dev];
}

int ilog2_ceil(int64_t v) {
  int l = 0;
  while ((int64_t{1} << l) < v) ++l;
  return l;
}

struct P2PPlan {
  int log2_tt, tpt;
  int64_t chunks, chunk_len, blocks_x;
};

// dense: TT = min(128, pow2 >= n_tgt); the sources are split into chunks
// (blockIdx.y) so that tiles x chunks fills whole waves of the kernel's
// resident CTAs (`slots`; 0 = unknown, size for the largest choice), each chunk
// >= 1024 sources.  rows: TT from the mean targets per row.
P2PPlan p2p_plan(int64_t n_src, int64_t n_tgt, int64_t n_rows, bool dense, int64_t slots) {
  P2PPlan p{};
  p.tpt = 1;
  if (dense) {
    p.log2_tt = std::min(7, ilog2_ceil(std::max<int64_t>(n_tgt, 1)));
    const int64_t want = 8LL * sm_count();
    const int64_t max_chunks = std::max<int64_t>(1, n_src / 1024);
    // enough targets (with source chunks still filling the machine): 4 per
    // thread -- independent FP64 chains and 4x fewer shared-memory reads
    const int64_t per4 = (int64_t)kP2PTpt * kP2PBlock;
    if (kP2PTpt > 1 && n_tgt >= per4 && ((n_tgt + per4 - 1) / per4) * max_chunks >= want)
      p.tpt = kP2PTpt;
    const int64_t per = (int64_t)p.tpt << p.log2_tt;
    const int64_t tiles = (n_tgt + per - 1) / per;
    const int64_t sl = slots > 0 ? slots : 16LL * sm_count();     // 16 = 2048 / 128 threads
    int64_t chunks = 1;
    if (tiles < sl) {
      const int64_t cmax = std::max<int64_t>(1, std::min(max_chunks, (2 * sl + tiles - 1) / tiles));
      if (slots <= 0) {
        chunks = cmax;                                 // sizing: the largest possible choice
      } else {
        double best = -1.0;
        for (int64_t c = 1; c <= cmax; ++c) {
          const double x = (double)(tiles * c) / (double)sl;
          const double score = x / std::ceil(x) * std::min(1.0, x);
          if (score > best + 1e-3) {
            best = score;
            chunks = c;
          }
        }
      }
    }
    p.chunk_len = (n_src + chunks - 1) / chunks;
    p.chunk_len = std::max<int64_t>(kP2PBlock, (p.chunk_len + kP2PBlock - 1) / kP2PBlock * kP2PBlock);
    p.chunks = std::max<int64_t>(1, (n_src + p.chunk_len - 1) / p.chunk_len);
    p.blocks_x = tiles;
  } else {
    const int64_t mean = (n_tgt + std::max<int64_t>(n_rows, 1) - 1) / std::max<int64_t>(n_rows, 1);
    p.log2_tt = std::min(7, ilog2_ceil(std::max<int64_t>(mean, 1)));
    p.chunks = 1;
    p.chunk_len = 0;
    p.blocks_x = n_rows;
  }
  return p;
}

// resident CTAs of the p2p kernel instance the plan will launch
template <int EQ, int VARIANT>
int64_t p2p_slots(bool tpt4, bool precise) {
  int nb = 0;
  cudaError_t e;
  if (tpt4)
    e = precise ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, p2p_kernel<EQ, VARIANT, true, kP2PTpt>, kP2PBlock, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, p2p_kernel<EQ, VARIANT, false, kP2PTpt>, kP2PBlock, 0);
  else
    e = precise ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, p2p_kernel<EQ, VARIANT, true, 1>, kP2PBlock, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, p2p_kernel<EQ, VARIANT, false, 1>, kP2PBlock, 0);
  if (e != cudaSuccess || nb <= 0) {
    cudaGetLastError();
    return 0;
  }
  return (int64_t)nb * sm_count();
}

int64_t slots_for(int equation, int variant, bool tpt4, bool precise) {
  if (equation == TSQBX_EQ_LAPLACE)
    return variant == 0 ? p2p_slots<TSQBX_EQ_LAPLACE, 0>(tpt4, precise)
         : variant == 1 ? p2p_slots<TSQBX_EQ_LAPLACE, 1>(tpt4, precise)
                        : p2p_slots<TSQBX_EQ_LAPLACE, 2>(tpt4, precise);
  return variant == 0 ? p2p_slots<TSQBX_EQ_HELMHOLTZ, 0>(tpt4, precise)
       : variant == 1 ? p2p_slots<TSQBX_EQ_HELMHOLTZ, 1>(tpt4, precise)
                      : p2p_slots<TSQBX_EQ_HELMHOLTZ, 2>(tpt4, precise);
}

template <int EQ, int VARIANT>
int launch_p2p(const P2PParams& a, const P2PPlan& pl, bool precise, cudaStream_t st) {
  const dim3 grid((unsigned)pl.blocks_x, (unsigned)pl.chunks);
  if (pl.tpt == kP2PTpt && kP2PTpt > 1) {
    if (precise) p2p_kernel<EQ, VARIANT, true, kP2PTpt><<<grid, kP2PBlock, 0, st>>>(a);
    else p2p_kernel<EQ, VARIANT, false, kP2PTpt><<<grid, kP2PBlock, 0, st>>>(a);
  } else {
    if (precise) p2p_kernel<EQ, VARIANT, true, 1><<<grid, kP2PBlock, 0, st>>>(a);
    else p2p_kernel<EQ, VARIANT, false, 1><<<grid, kP2PBlock, 0, st>>>(a);
  }
  return check_cuda(cudaGetLastError(), "p2p_kernel launch");
}

}  // namespace
}  // namespace tsqbx

using namespace tsqbx;

extern "C" {

int64_t tsqbx_p2p_workspace_bytes(int64_t n_src, int64_t n_tgt, int64_t n_rows, int dense) {
  const P2PPlan pl = p2p_plan(n_src, n_tgt, n_rows, dense != 0, 0);
  return pl.chunks > 1 ? pl.chunks * n_tgt * 2 * (int64_t)sizeof(double) : 0;
}

int tsqbx_p2p_packed(int equation, int variant, double k, const double* packed, int64_t n_src,
                     int with_normals, int64_t n_rows, const int64_t* row_tgt,
                     const int64_t* row_ptr, const int32_t* row_idx, const double* tgt_xyz,
                     const double* tgt_nrm, int64_t n_tgt, unsigned flags, void* workspace,
                     int64_t ws_bytes, double* out, int64_t* err_key, void* stream) {
  if (equation != TSQBX_EQ_LAPLACE && equation != TSQBX_EQ_HELMHOLTZ)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: bad equation %d", equation);
  if (variant < 0 || variant > 2) return set_error(TSQBX_ERR_ARGUMENT, "p2p: bad variant %d", variant);
  if (n_src < 0 || n_tgt < 0 || n_src > INT32_MAX || n_tgt > INT32_MAX)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: bad sizes");
  if (n_tgt > 0 && (!tgt_xyz || !out))
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: missing targets or output");
  if (variant == TSQBX_VARIANT_SPRIME && n_tgt > 0 && !tgt_nrm)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: S' needs target normals");
  if (variant == TSQBX_VARIANT_D && n_src > 0 && !with_normals)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: D needs packed source normals");
  if (row_ptr && (!row_tgt || (!row_idx && n_rows > 0) || n_rows < 0))
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: rows need row_tgt, row_ptr and row_idx");
  if ((flags & TSQBX_FLAG_VALIDATE) && !err_key)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: validation needs err_key");
  const cudaStream_t st = (cudaStream_t)stream;
  if (flags & TSQBX_FLAG_VALIDATE) {
    p2p_set_key<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long*>(err_key),
                                 (unsigned long long)TSQBX_ERR_KEY_NONE);
    const int rc = check_cuda(cudaGetLastError(), "p2p err init");
    if (rc) return rc;
  }
  if (n_tgt == 0) return TSQBX_OK;
  const bool dense = row_ptr == nullptr;
  if (n_src == 0 || (!dense && n_rows == 0)) {
    return check_cuda(cudaMemsetAsync(out, 0, n_tgt * 2 * sizeof(double), st), "p2p zero");
  }
  if (!packed || (((uintptr_t)packed) & 31))
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: packed sources must be 32-byte aligned");
  const bool precise = (flags & TSQBX_FLAG_PRECISE) != 0;
  P2PPlan pl = p2p_plan(n_src, n_tgt, n_rows, dense, 0);
  if (dense) pl = p2p_plan(n_src, n_tgt, n_rows, dense,
                           slots_for(equation, variant, pl.tpt == kP2PTpt && kP2PTpt > 1, precise));
  if (pl.blocks_x > INT32_MAX || pl.chunks > 65535)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: grid too large");
  const int64_t need = tsqbx_p2p_workspace_bytes(n_src, n_tgt, n_rows, dense);
  if (need > 0 && (!workspace || ws_bytes < need))
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: workspace too small (%lld < %lld bytes)",
                     (long long)ws_bytes, (long long)need);
  // rows: the kernel trusts row_tgt to partition [0, n_tgt) in order (the
  // host wrapper checks it)

  P2PParams a{};
  a.sp = reinterpret_cast<const double4*>(packed);
  a.swi = packed + 4 * n_src;
  const int64_t base = (5 * n_src + 3) / 4 * 4;
  a.snrm = with_normals ? reinterpret_cast<const double4*>(packed + base) : nullptr;
  a.tgt = tgt_xyz;
  a.tnrm = tgt_nrm;
  a.row_tgt = row_tgt;
  a.row_ptr = row_ptr;
  a.row_idx = row_idx;
  a.out = out;
  a.part = pl.chunks > 1 ? static_cast<double*>(workspace) : nullptr;
  a.err = reinterpret_cast<unsigned long long*>(err_key);
  a.n_src = n_src;
  a.n_tgt = n_tgt;
  a.n_rows = n_rows;
  a.chunk_len = dense ? pl.chunk_len : 0;
  a.log2_tt = pl.log2_tt;
  a.screen = (flags & TSQBX_FLAG_VALIDATE) ? 1 : 0;
  a.k = k;

  int rc;
  if (equation == TSQBX_EQ_LAPLACE) {
    rc = variant == 0 ? launch_p2p<TSQBX_EQ_LAPLACE, 0>(a, pl, precise, st)
       : variant == 1 ? launch_p2p<TSQBX_EQ_LAPLACE, 1>(a, pl, precise, st)
                      : launch_p2p<TSQBX_EQ_LAPLACE, 2>(a, pl, precise, st);
  } else {
    rc = variant == 0 ? launch_p2p<TSQBX_EQ_HELMHOLTZ, 0>(a, pl, precise, st)
       : variant == 1 ? launch_p2p<TSQBX_EQ_HELMHOLTZ, 1>(a, pl, precise, st)
                      : launch_p2p<TSQBX_EQ_HELMHOLTZ, 2>(a, pl, precise, st);
  }
  if (rc || pl.chunks == 1) return rc;
  const int blocks = (int)((n_tgt + 255) / 256);
  if (pl.chunks >= 64 && n_tgt * 32 <= 8LL * 256 * sm_count())
    p2p_reduce_warp_kernel<<<(unsigned)((n_tgt * 32 + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const double2*>(a.part), pl.chunks, n_tgt,
        reinterpret_cast<double2*>(out), a.screen, a.err);
  else
    p2p_reduce_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(a.part), pl.chunks,
                                              n_tgt, reinterpret_cast<double2*>(out), a.screen,
                                              a.err);
  return check_cuda(cudaGetLastError(), "p2p_reduce launch");
}

int64_t tsqbx_p2p_user_workspace_bytes(int variant, int64_t n_src, int64_t n_tgt) {
  const int64_t pbytes = packed_doubles(n_src, variant == TSQBX_VARIANT_D) * (int64_t)sizeof(double);
  return (pbytes + 255) / 256 * 256 + tsqbx_p2p_workspace_bytes(n_src, n_tgt, 0, 1);
}

static int p2p_user(int equation, int variant, double k, const double* src_xyz,
                    const double* src_w, const double* src_nrm, int64_t n_src,
                    const double* tgt_xyz, const double* tgt_nrm, int64_t n_tgt, unsigned flags,
                    void* workspace, int64_t ws_bytes, double* out, int64_t* err_key,
                    void* stream) {
  if (variant == TSQBX_VARIANT_D && n_src > 0 && !src_nrm)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: D needs source normals");
  const int64_t need = tsqbx_p2p_user_workspace_bytes(variant, n_src, n_tgt);
  if (!workspace || ws_bytes < need)
    return set_error(TSQBX_ERR_ARGUMENT, "p2p: workspace too small (%lld < %lld bytes)",
                     (long long)ws_bytes, (long long)need);
  double* packed = static_cast<double*>(workspace);
  const int64_t pbytes =
      (packed_doubles(n_src, variant == TSQBX_VARIANT_D) * (int64_t)sizeof(double) + 255) / 256 * 256;
  int rc = tsqbx_pack_sources(n_src, src_xyz, src_w, variant == TSQBX_VARIANT_D ? src_nrm : nullptr,
                              nullptr, packed, stream);
  if (rc) return rc;
  return tsqbx_p2p_packed(equation, variant, k, packed, n_src, variant == TSQBX_VARIANT_D, 0,
                          nullptr, nullptr, nullptr, tgt_xyz, tgt_nrm, n_tgt, flags,
                          static_cast<char*>(workspace) + pbytes, ws_bytes - pbytes, out, err_key,
                          stream);
}

int tsqbx_p2p_laplace(int variant, const double* src_xyz, const double* src_w,
                      const double* src_nrm, int64_t n_src, const double* tgt_xyz,
                      const double* tgt_nrm, int64_t n_tgt, unsigned flags, void* workspace,
                      int64_t ws_bytes, double* out, int64_t* err_key, void* stream) {
  return p2p_user(TSQBX_EQ_LAPLACE, variant, 0.0, src_xyz, src_w, src_nrm, n_src, tgt_xyz,
                  tgt_nrm, n_tgt, flags, workspace, ws_bytes, out, err_key, stream);
}

int tsqbx_p2p_helmholtz(int variant, double k, const double* src_xyz, const double* src_w,
                        const double* src_nrm, int64_t n_src, const double* tgt_xyz,
                        const double* tgt_nrm, int64_t n_tgt, unsigned flags, void* workspace,
                        int64_t ws_bytes, double* out, int64_t* err_key, void* stream) {
  return p2p_user(TSQBX_EQ_HELMHOLTZ, variant, k, src_xyz, src_w, src_nrm, n_src, tgt_xyz,
                  tgt_nrm, n_tgt, flags, workspace, ws_bytes, out, err_key, stream);
}

int tsqbx_p2p_find_singular(const double* packed, int64_t n_src, int64_t n_rows,
                            const int64_t* row_tgt, const int64_t* row_ptr,
                            const int32_t* row_idx, const double* tgt_xyz, int64_t n_tgt,
                            int64_t* err_key, void* stream) {
  if (!err_key || n_src < 0 || n_tgt < 0) return set_error(TSQBX_ERR_ARGUMENT, "p2p_find_singular: bad arguments");
  const cudaStream_t st = (cudaStream_t)stream;
  p2p_set_key<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long*>(err_key),
                               (unsigned long long)TSQBX_ERR_KEY_NONE);
  const int rc = check_cuda(cudaGetLastError(), "p2p_find_singular init");
  if (rc) return rc;
  if (n_tgt == 0 || n_src == 0) return TSQBX_OK;
  const int64_t blocks = (n_tgt * 32 + 255) / 256;
  p2p_singular_kernel<<<(unsigned)blocks, 256, 0, st>>>(
      reinterpret_cast<const double4*>(packed), n_src, tgt_xyz, n_tgt, row_tgt, row_ptr, row_idx,
      n_rows, reinterpret_cast<unsigned long long*>(err_key));
  return check_cuda(cudaGetLastError(), "p2p_singular launch");
}

}  // extern "C"
