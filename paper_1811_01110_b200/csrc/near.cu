// near.cu -- device radius-ball near-list (CSR) builder for sm_100a.
//
// BASELINE.json defines a center's near list as every source within a radius
// of it (self included); the reference has no such builder (its driver uses
// tree lists, driver.py:197-228 / ilists.py:93-218; the closest analogue is
// cKDTree.query_ball_point, costmodel.py:361-365).
//
// Pipeline (stream-ordered but for one read-back of the bounding box; the
// caller reads the totals once):
//   1. bounding box, min/max radius        (block-reduced ordered-int atomics)
//   2. fine Morton keys of sources/centers  (<= 21 bits/axis; a level-L cell is
//      the key prefix fine >> (3 + L), L chosen per center from its radius)
//   3. CUB radix sort of both over the key bits in use
//                                           -> src_perm, ctr_order ("tree leaf" order)
//   4. open-addressed hash: (cell, level) -> [start, end) in the sorted sources
//   5. bound (SELL) or count (CSR): one warp per 32 consecutive centers sweeps
//      the union of their neighbour cells (or each distinct cell's 27
//      neighbours) through a shared-memory tile
//   6. CUB exclusive scans -> near_ptr, SELL-32x4 slice offsets, totals
//   7. fill: the same sweep; per-lane member bit masks, each lane appends its
//      own members to its SELL column (16-byte blocks); CSR entries on demand
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "near_sweep.cuh"

namespace tsqbx {
namespace {

using namespace nsw;

__device__ __forceinline__ long long ord_of(double d) {
  const long long b = __double_as_longlong(d);
  return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
}
__device__ __forceinline__ double of_ord(long long b) {
  return __longlong_as_double(b >= 0 ? b : b ^ 0x7fffffffffffffffLL);
}

__global__ void init_bounds(long long* mm) {
  const int i = threadIdx.x;
  if (i < 3) mm[i] = LLONG_MAX;                 // min x, y, z
  else if (i < 6) mm[i] = LLONG_MIN;            // max x, y, z
  else if (i == 6) mm[i] = LLONG_MIN;           // max radius
  else if (i == 7) mm[i] = LLONG_MAX;           // min radius
}

__global__ void bounds_kernel(const double* __restrict__ src, int64_t n_src,
                              const double* __restrict__ ctr, const double* __restrict__ rad,
                              int64_t n_ctr, long long* mm) {
  long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
  long long hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  long long rm = LLONG_MIN, rn = LLONG_MAX;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_src + n_ctr;
       i += stride) {
    const double* p = i < n_src ? src + 3 * i : ctr + 3 * (i - n_src);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const long long o = ord_of(p[d]);
      lo[d] = min(lo[d], o);
      hi[d] = max(hi[d], o);
    }
    if (i >= n_src) {
      const long long o = ord_of(rad[i - n_src]);
      rm = max(rm, o);
      rn = min(rn, o);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = min(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], off));
      hi[d] = max(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], off));
    }
    rm = max(rm, __shfl_xor_sync(0xffffffffu, rm, off));
    rn = min(rn, __shfl_xor_sync(0xffffffffu, rn, off));
  }
  // block reduction through shared memory, then one atomic per value per block
  __shared__ long long red[8][32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      red[d][w] = lo[d];
      red[3 + d][w] = hi[d];
    }
    red[6][w] = rm;
    red[7][w] = rn;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int v = threadIdx.x;
    const bool is_min = v < 3 || v == 7;
    long long acc = red[v][0];
    for (int q = 1; q < nw; ++q) acc = is_min ? min(acc, red[v][q]) : max(acc, red[v][q]);
    if (is_min) atomicMin(&mm[v], acc);
    else atomicMax(&mm[v], acc);
  }
}

// prm = {lo_x, lo_y, lo_z, fine cell, top level}
__global__ void grid_params(const long long* mm, double* prm, int levels) {
  double lo[3], ext = 0.0;
  for (int d = 0; d < 3; ++d) {
    lo[d] = of_ord(mm[d]);
    ext = fmax(ext, of_ord(mm[3 + d]) - lo[d]);
  }
  const double rmax = mm[6] == LLONG_MIN ? 0.0 : of_ord(mm[6]);
  const double rmin = mm[7] == LLONG_MAX ? 0.0 : of_ord(mm[7]);
  // level-0 cell >= the smallest radius (with slack for rounding of the cell
  // index), but no finer than the top level needs to reach rmax; 2^21 fine
  // cells per axis max
  const double rlo = fmax(fmax(rmin, 0.0), rmax / (double)(1 << (levels - 1)));
  double fine = fmax(rlo * (1.0 + 1e-9) / (1 << kSubBits),
                     ext / (double)((1 << kFineBits) - 4 * kFineOffset));
  if (!(fine > 0.0)) fine = 1.0;
  int top = 0;
  while (top < levels - 1 && fine * (double)(1 << (kSubBits + top)) < rmax * (1.0 + 1e-9)) ++top;
  prm[0] = lo[0];
  prm[1] = lo[1];
  prm[2] = lo[2];
  prm[3] = fine;
  prm[4] = (double)top;
}

__global__ void key_kernel(const double* __restrict__ pts, int64_t n, const double* prm,
                           unsigned long long* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long f[3];
  fine_coords(pts + 3 * i, prm, f);
  key[i] = morton3(f[0], f[1], f[2]);
  val[i] = (int32_t)i;
}

__global__ void gather_sorted(const double* __restrict__ src, const int32_t* __restrict__ perm,
                              int64_t n, double4* __restrict__ sxyz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = perm[i];
  sxyz[i] = make_double4(src[3 * s], src[3 * s + 1], src[3 * s + 2], 0.0);
}

__global__ void hash_clear(unsigned long long* hkey, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cap) hkey[i] = kEmpty;
}

__device__ __forceinline__ int64_t hash_slot(unsigned long long* hkey, int64_t cap,
                                             unsigned long long ck) {
  int64_t h = (int64_t)(hash64(ck) & (unsigned long long)(cap - 1));
  while (true) {
    const unsigned long long prev = atomicCAS(&hkey[h], kEmpty, ck);
    if (prev == kEmpty || prev == ck) return h;
    h = (h + 1) & (cap - 1);
  }
}

__global__ void hash_insert(const unsigned long long* __restrict__ skey, int64_t n,
                            const double* __restrict__ prm, unsigned long long* hkey, int32_t* hst,
                            int32_t* hen, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int top = (int)prm[4];
  for (int lv = 0; lv <= top; ++lv) {
    const int sh = 3 * (kSubBits + lv);
    const unsigned long long ck = skey[i] >> sh;
    const bool head = i == 0 || (skey[i - 1] >> sh) != ck;
    const bool tail = i == n - 1 || (skey[i + 1] >> sh) != ck;
    if (!head && !tail) continue;
    const int64_t h = hash_slot(hkey, cap, ck | level_tag(lv));
    if (head) hst[h] = (int32_t)i;
    if (tail) hen[h] = (int32_t)(i + 1);
  }
}

// one warp per 32 consecutive centers (near_sweep.cuh: sweep_warp)
template <int MODE>
__global__ void __launch_bounds__(128, 8) sweep_cell_kernel(
    const double* __restrict__ ctr, const double* __restrict__ rad, int64_t n_ctr,
    const int32_t* __restrict__ order, const double* __restrict__ prm,
    const double4* __restrict__ sxyz, const unsigned long long* __restrict__ hkey,
    const int32_t* __restrict__ hst, const int32_t* __restrict__ hen, int64_t cap,
    int64_t* __restrict__ cnt, const int64_t* __restrict__ nptr, int32_t* __restrict__ nidx,
    const int64_t* __restrict__ sptr, int32_t* __restrict__ sidx,
    const int64_t* __restrict__ mptr = nullptr, unsigned* __restrict__ mask = nullptr) {
  __shared__ SweepSmem sm[4];
  constexpr bool STAGED = (MODE == 1 || MODE == 5) && kStagedAppend;
  __shared__ int32_t stage[STAGED ? 4 * kStageWords : 1];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = g < n_ctr;
  // MODE 3: CSR row; MODE 1 / 5: SELL-32x4 column, entry k at dst[128 (k / 4) + k % 4]
  int32_t* dst = (MODE == 3 && valid) ? nidx + nptr[g]
                 : ((MODE == 1 || MODE == 5) && valid) ? sidx + sptr[g >> 5] + 4 * (g & 31)
                                                       : nullptr;
  const SweepIn in{ctr, rad, n_ctr, order, prm, sxyz, hkey, hst, hen, cap};
  int k = 0;
  int64_t ub = 0;
  // MODE 4 / 5: the slice's member masks (see near_sweep.cuh)
  unsigned* mk = ((MODE == 4 || MODE == 5) && (g >> 5) * 32 < n_ctr) ? mask + mptr[g >> 5] : nullptr;
  sweep_warp<MODE, STAGED>(in, sm[threadIdx.x >> 5], g, dst, INT_MAX, k, ub, mk,
                           STAGED ? stage + (threadIdx.x >> 5) * kStageWords : nullptr);
  if ((MODE == 0 || MODE == 4) && valid) cnt[g] = k;
  if ((MODE == 1 || MODE == 5) && valid && cnt) cnt[g] = k;
  if (MODE == 2 && (threadIdx.x & 31) == 0 && (g >> 5) * 32 < n_ctr)
    cnt[g >> 5] = 32 * ((ub + 3) & ~3ll);
}

// CSR rows from the SELL-32x4 copy (thread per row; materialised on demand)
__global__ void sell_to_csr_kernel(const int64_t* __restrict__ nptr, int64_t n_rows,
                                   const int64_t* __restrict__ sptr,
                                   const int32_t* __restrict__ sidx, int32_t* __restrict__ nidx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t b = nptr[r], len = nptr[r + 1] - b;
  const int4* blk = reinterpret_cast<const int4*>(sidx + sptr[r >> 5]) + (r & 31);
  for (int64_t i = 0; i < len; i += 4) {
    const int4 v = blk[32 * (i >> 2)];
    nidx[b + i] = v.x;
    if (i + 1 < len) nidx[b + i + 1] = v.y;
    if (i + 2 < len) nidx[b + i + 2] = v.z;
    if (i + 3 < len) nidx[b + i + 3] = v.w;
  }
}

// a warp per slice: the first dst-width blocks of a (wider) source slice
__global__ void sell_compact_kernel(int64_t n_sl, const int64_t* __restrict__ sptr_src,
                                    const int32_t* __restrict__ sidx_src,
                                    const int64_t* __restrict__ sptr_dst,
                                    int32_t* __restrict__ sidx_dst) {
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= n_sl) return;
  const int64_t n4 = (sptr_dst[sl + 1] - sptr_dst[sl]) >> 2;      // int4s to copy
  const int4* src = reinterpret_cast<const int4*>(sidx_src + sptr_src[sl]);
  int4* dst = reinterpret_cast<int4*>(sidx_dst + sptr_dst[sl]);
  for (int64_t q = lane; q < n4; q += 32) dst[q] = src[q];
}

// Windowed SELL (short near lists): per 32-row slice, the unique sources of its
// rows (at most TSQBX_WINDOW, in win_src[s * W ...], count win_len[s]) and the
// entries rewritten as indices into that window (loc_idx, same SELL-32x4
// positions as sell_idx).  A warp per slice: its lanes insert their rows'
// entries into a shared-memory hash set (open addressing, 2W slots), rank the
// occupied slots by a ballot scan, write the window and map every entry to its
// rank.  A slice with more than W distinct sources keeps its global indices
// (win_len = -1) and counts in *overflow.
constexpr int kWinHash = 2 * TSQBX_WINDOW;
__global__ void __launch_bounds__(128) sell_window_kernel(
    const int64_t* __restrict__ nptr, int64_t n_rows, const int64_t* __restrict__ sptr,
    const int32_t* __restrict__ sidx, int32_t* __restrict__ loc, int32_t* __restrict__ win_src,
    int32_t* __restrict__ win_len, unsigned* __restrict__ overflow) {
  __shared__ int32_t key[4][kWinHash];
  __shared__ int16_t rank[4][kWinHash];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = g >> 5;
  if ((s << 5) >= n_rows) return;                  // whole warps only
  for (int i = lane; i < kWinHash; i += 32) key[w][i] = -1;
  __syncwarp();
  const int len = g < n_rows ? (int)(nptr[g + 1] - nptr[g]) : 0;
  const int32_t* col = sidx + sptr[s] + 4 * (g & 31);
  auto slot_of = [&](int32_t j, bool insert) {
    unsigned h = ((unsigned)j * 2654435761u) % (unsigned)kWinHash;
    for (int probe = 0; probe < kWinHash; ++probe) {
      const int32_t cur = insert ? atomicCAS(&key[w][h], -1, j) : key[w][h];
      if (cur == -1 || cur == j) return (int)h;
      h = h + 1 == (unsigned)kWinHash ? 0u : h + 1;
    }
    return -1;
  };
  bool full = false;
  for (int k = 0; k < len; ++k) full |= slot_of(col[((k >> 2) << 7) | (k & 3)], true) < 0;
  __syncwarp();
  // rank the occupied slots (slot order), lane l owning slots [l*R, l*R + R)
  constexpr int R = kWinHash / 32;
  int occ = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) occ += key[w][lane * R + i] != -1;
  int pre = occ;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, off);
    if (lane >= off) pre += v;
  }
  const int total = __shfl_sync(0xffffffffu, pre, 31);
  pre -= occ;
  const bool over = __any_sync(0xffffffffu, full) || total > TSQBX_WINDOW;
  if (over) {
    // too many distinct sources for the window: this slice keeps global
    // indices (win_len = -1; its warp gathers from HBM/L2 as the plain kernel)
    if (lane == 0) {
      win_len[s] = -1;
      atomicAdd(overflow, 1u);
    }
    int32_t* lcol = loc + sptr[s] + 4 * (g & 31);
    for (int k = 0; k < len; ++k) {
      const int at = ((k >> 2) << 7) | (k & 3);
      lcol[at] = col[at];
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int h = lane * R + i;
    const int32_t j = key[w][h];
    if (j != -1) {
      rank[w][h] = (int16_t)pre;
      win_src[s * TSQBX_WINDOW + pre] = j;
      ++pre;
    }
  }
  if (lane == 0) win_len[s] = total;
  __syncwarp();
  int32_t* lcol = loc + sptr[s] + 4 * (g & 31);
  for (int k = 0; k < len; ++k) {
    const int at = ((k >> 2) << 7) | (k & 3);
    lcol[at] = rank[w][slot_of(col[at], false)];
  }
}

__global__ void set_tail(int64_t* cnt, int64_t n) { cnt[n] = 0; }
__global__ void set_key64(int64_t* p, int64_t v) { *p = v; }

// one warp per 32-row slice: width = longest row; writes 32 * width (slice entries)
__global__ void sell_width(const int64_t* __restrict__ nptr, int64_t n_rows,
                           int64_t* __restrict__ wid) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (n_rows + 31) / 32 * 32) return;       // whole warps only
  int64_t m = r < n_rows ? nptr[r + 1] - nptr[r] : 0;
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) wid[r >> 5] = 32 * ((m + 3) & ~3ll);   // width: multiple of 4
}

__global__ void sell_tail(int64_t* wid, int64_t n_sl) { wid[n_sl] = 0; }

// mask words of a slice from its bound width (32 x its candidate bound, a
// multiple of 4): 32 lanes x one word per 32-candidate group
__global__ void mask_width(const int64_t* __restrict__ wid, int64_t n_sl,
                           int64_t* __restrict__ mw) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > n_sl) return;
  mw[s] = s < n_sl ? 32 * (((wid[s] >> 5) + 31) >> 5) : 0;
}



// --- targets into processing order -------------------------------------------
// Per-row target counts in processing order.  Malformed caller offsets (not
// starting at 0, decreasing, past n_tgt, or not ending at n_tgt) raise *bad and
// give the row no targets, so nothing downstream leaves the target arrays.
__global__ void order_count(const int32_t* __restrict__ order, const int64_t* __restrict__ tptr,
                            int64_t n, int64_t n_tgt, int64_t* __restrict__ cnt,
                            int64_t* __restrict__ bad) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g > n) return;
  if (g == n) {
    cnt[n] = 0;
    if ((tptr[0] != 0 || tptr[n] != n_tgt) && bad) *bad = 1;
    return;
  }
  const int64_t ic = order[g];
  const int64_t a = tptr[ic], b = tptr[ic + 1];
  const bool ok = 0 <= a && a <= b && b <= n_tgt;
  if (!ok && bad) *bad = 1;
  cnt[g] = ok ? b - a : 0;
}

__global__ void order_copy(const int32_t* __restrict__ order, const double* __restrict__ ctr,
                           const int64_t* __restrict__ tptr, const double* __restrict__ tgt,
                           const double* __restrict__ tnrm, int64_t n, int64_t n_tgt,
                           const int64_t* __restrict__ cnt_in, int64_t* __restrict__ tptr_out,
                           double* __restrict__ ctr_out,
                           double* __restrict__ tgt_out, double* __restrict__ tnrm_out,
                           int64_t* __restrict__ tidx) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int64_t ic = order[g];
  ctr_out[3 * g] = ctr[3 * ic];
  ctr_out[3 * g + 1] = ctr[3 * ic + 1];
  ctr_out[3 * g + 2] = ctr[3 * ic + 2];
  // cnt: the checked count of order_count (0 for a malformed row); with
  // malformed offsets the prefix can pass n_tgt, so the copy and the row
  // offsets the kernels read are clamped to the target arrays
  const int64_t src0 = tptr[ic], dst0 = tptr_out[g];
  const int64_t cnt = min(cnt_in[g], max((int64_t)0, n_tgt - dst0));
  if (dst0 > n_tgt) tptr_out[g] = n_tgt;
  if (g == 0 && tptr_out[n] > n_tgt) tptr_out[n] = n_tgt;
  for (int64_t j = 0; j < cnt; ++j) {
    for (int d = 0; d < 3; ++d) {
      tgt_out[3 * (dst0 + j) + d] = tgt[3 * (src0 + j) + d];
      if (tnrm) tnrm_out[3 * (dst0 + j) + d] = tnrm[3 * (src0 + j) + d];
    }
    tidx[dst0 + j] = src0 + j;
  }
}

__global__ void sell_fill_kernel(const int64_t* __restrict__ nptr,
                                 const int32_t* __restrict__ nidx, int64_t n_rows,
                                 const int64_t* __restrict__ sptr, int32_t* __restrict__ sidx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t b = nptr[r], len = nptr[r + 1] - b;
  // blocks of 4 columns: entry (r, i) at sptr[slice] + (i / 4) * 128 + (r % 32) * 4 + i % 4
  int32_t* base = sidx + sptr[r >> 5] + 4 * (r & 31);
  for (int64_t i = 0; i < len; ++i) base[(i >> 2) * 128 + (i & 3)] = nidx[b + i];
}

__global__ void scatter_c128(int64_t n, const int64_t* __restrict__ dest,
                             const double2* __restrict__ src, double2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[dest ? dest[i] : i] = src[i];
}

}  // namespace
}  // namespace tsqbx

using namespace tsqbx;

extern "C" {

int64_t tsqbx_near_workspace_bytes(int64_t n_ctr, int64_t n_src) {
  if (n_ctr < 0 || n_src < 0) return -1;
  return (int64_t)near_layout(n_ctr, n_src).total;
}

}  // extern "C"

// index_only: bounding box, Morton sorts and cell hash (the state the sweeps
// and the fused kernel read), no sweep
static int near_count_impl(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                           const double* src_xyz, int64_t n_src, void* workspace,
                           int64_t ws_bytes, int32_t* src_perm, int32_t* ctr_order,
                           int64_t* near_ptr, int64_t* sell_ptr, int64_t* totals, void* stream,
                           bool index_only) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_ctr < 0 || n_src < 0 || n_src > INT32_MAX - 64 || n_ctr > INT32_MAX - 64)
    return set_error(TSQBX_ERR_ARGUMENT, "near_count: bad sizes");
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_count: workspace too small (need %lld)",
                     (long long)L.total);
  if ((!index_only && (!near_ptr || !totals)) || (n_ctr > 0 && (!ctr_xyz || !radius || !ctr_order)) ||
      (n_src > 0 && (!src_xyz || !src_perm)))
    return set_error(TSQBX_ERR_ARGUMENT, "near_count: null array");
  char* ws = static_cast<char*>(workspace);
  long long* mm = reinterpret_cast<long long*>(ws + L.off_mm);
  double* prm = reinterpret_cast<double*>(ws + L.off_prm);
  auto* skey_in = reinterpret_cast<unsigned long long*>(ws + L.off_skey_in);
  auto* skey = reinterpret_cast<unsigned long long*>(ws + L.off_skey);
  auto* sval_in = reinterpret_cast<int32_t*>(ws + L.off_sval_in);
  auto* ckey_in = reinterpret_cast<unsigned long long*>(ws + L.off_ckey_in);
  auto* ckey = reinterpret_cast<unsigned long long*>(ws + L.off_ckey);
  auto* cval_in = reinterpret_cast<int32_t*>(ws + L.off_cval_in);
  auto* sxyz = reinterpret_cast<double4*>(ws + L.off_sxyz);
  auto* hkey = reinterpret_cast<unsigned long long*>(ws + L.off_hkey);
  auto* hst = reinterpret_cast<int32_t*>(ws + L.off_hst);
  auto* hen = reinterpret_cast<int32_t*>(ws + L.off_hen);
  auto* cnt = reinterpret_cast<int64_t*>(ws + L.off_cnt);
  void* tmp = ws + L.off_tmp;

  init_bounds<<<1, 32, 0, st>>>(mm);
  if (n_src + n_ctr > 0) {
    int nb = (int)std::min<int64_t>((n_src + n_ctr + 255) / 256, 148 * 8);
    bounds_kernel<<<nb, 256, 0, st>>>(src_xyz, n_src, ctr_xyz, radius, n_ctr, mm);
  }
  grid_params<<<1, 1, 0, st>>>(mm, prm, n_src <= kMultiLevelMaxSources ? kLevels : 1);
  // Radix-sort only the key bits in use: one read-back of the grid (the
  // caller synchronises after this call anyway) halves the sort passes of a
  // compact geometry (C2: 9 bits per axis, 27-bit keys, 4 passes instead of 8)
  int key_bits = 3 * kFineBits;
  if (n_src + n_ctr > 0) {
    long long hm[8];
    double hp[8];
    cudaError_t e0 = cudaMemcpyAsync(hm, mm, 8 * sizeof(long long), cudaMemcpyDeviceToHost, st);
    if (e0 == cudaSuccess)
      e0 = cudaMemcpyAsync(hp, prm, 5 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e0 == cudaSuccess) e0 = cudaStreamSynchronize(st);
    if (e0 != cudaSuccess) return check_cuda(e0, "near_count grid read-back");
    int bits = 1;
    for (int d = 0; d < 3; ++d) {
      const double lo = hp[d], hi = hm[3 + d] >= 0 ? __builtin_bit_cast(double, hm[3 + d])
                                                   : __builtin_bit_cast(double, hm[3 + d] ^ 0x7fffffffffffffffLL);
      double q = std::floor((hi - lo) / hp[3]);
      q = std::min(std::max(q, 0.0), (double)((1 << kFineBits) - 2 * kFineOffset));
      const unsigned long long fmax = (unsigned long long)q + kFineOffset + 1;
      int b = 1;
      while (b < kFineBits && (fmax >> b) != 0) ++b;
      bits = std::max(bits, b);
    }
    key_bits = 3 * bits;
  }
  size_t tb = L.tmp_bytes;
  if (n_src > 0) {
    key_kernel<<<(int)((n_src + 255) / 256), 256, 0, st>>>(src_xyz, n_src, prm, skey_in, sval_in);
    cub::DeviceRadixSort::SortPairs(tmp, tb, skey_in, skey, sval_in, src_perm, (int)n_src, 0,
                                    key_bits, st);
    gather_sorted<<<(int)((n_src + 255) / 256), 256, 0, st>>>(src_xyz, src_perm, n_src, sxyz);
  }
  hash_clear<<<(int)((L.cap + 255) / 256), 256, 0, st>>>(hkey, L.cap);
  if (n_src > 0)
    hash_insert<<<(int)((n_src + 255) / 256), 256, 0, st>>>(skey, n_src, prm, hkey, hst, hen, L.cap);
  if (n_ctr > 0) {
    key_kernel<<<(int)((n_ctr + 255) / 256), 256, 0, st>>>(ctr_xyz, n_ctr, prm, ckey_in, cval_in);
    tb = L.tmp_bytes;
    cub::DeviceRadixSort::SortPairs(tmp, tb, ckey_in, ckey, cval_in, ctr_order, (int)n_ctr, 0,
                                    key_bits, st);
    if (!sell_ptr && !index_only)
      sweep_cell_kernel<0><<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
          ctr_xyz, radius, n_ctr, ctr_order, prm, sxyz, hkey, hst, hen, L.cap, cnt, nullptr,
          nullptr, nullptr, nullptr);
  }
  if (index_only) return check_cuda(cudaGetLastError(), "near_index launch");
  cudaError_t e;
  if (!sell_ptr) {                      // exact row lengths -> CSR offsets
    set_tail<<<1, 1, 0, st>>>(cnt, n_ctr);
    tb = L.tmp_bytes;
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, near_ptr, (int)(n_ctr + 1), st);
    e = cudaMemcpyAsync(totals, near_ptr + n_ctr, sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return check_cuda(e, "near_count copy");
  } else {
    // SELL-32x4 offsets from candidate-count bounds (no distance tests): the
    // fill writes every row into its slice directly and produces the exact
    // lengths (near_ptr, totals[0]) itself.  Slots past a row's length are
    // never read.
    const int64_t n_sl = (n_ctr + 31) / 32;
    int64_t* wid = reinterpret_cast<int64_t*>(ws + L.off_wid);
    if (n_ctr > 0)
      sweep_cell_kernel<2><<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
          ctr_xyz, radius, n_ctr, ctr_order, prm, sxyz, hkey, hst, hen, L.cap, wid, nullptr,
          nullptr, nullptr, nullptr);
    sell_tail<<<1, 1, 0, st>>>(wid, n_sl);
    tb = L.tmp_bytes;
    cub::DeviceScan::ExclusiveSum(tmp, tb, wid, sell_ptr, (int)(n_sl + 1), st);
    e = cudaMemcpyAsync(totals + 1, sell_ptr + n_sl, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                        st);
    if (e != cudaSuccess) return check_cuda(e, "near_count copy");
    set_key64<<<1, 1, 0, st>>>(totals, -1);
  }
  return check_cuda(cudaGetLastError(), "near_count launch");
}

extern "C" {

int tsqbx_near_count(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                     const double* src_xyz, int64_t n_src, void* workspace, int64_t ws_bytes,
                     int32_t* src_perm, int32_t* ctr_order, int64_t* near_ptr,
                     int64_t* sell_ptr, int64_t* totals, void* stream) {
  return near_count_impl(ctr_xyz, radius, n_ctr, src_xyz, n_src, workspace, ws_bytes, src_perm,
                         ctr_order, near_ptr, sell_ptr, totals, stream, false);
}

int tsqbx_near_index(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                     const double* src_xyz, int64_t n_src, void* workspace, int64_t ws_bytes,
                     int32_t* src_perm, int32_t* ctr_order, void* stream) {
  return near_count_impl(ctr_xyz, radius, n_ctr, src_xyz, n_src, workspace, ws_bytes, src_perm,
                         ctr_order, nullptr, nullptr, nullptr, stream, true);
}

int tsqbx_near_fill(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                    const double* src_xyz, int64_t n_src, void* workspace, int64_t ws_bytes,
                    const int32_t* ctr_order, int64_t* near_ptr, int32_t* near_idx,
                    const int64_t* sell_ptr, int32_t* sell_idx, int64_t* totals, void* stream) {
  (void)src_xyz;
  cudaStream_t st = (cudaStream_t)stream;
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_fill: workspace too small");
  const bool sell = sell_idx != nullptr;
  if (sell && (near_idx || !sell_ptr || !totals || !near_ptr))
    return set_error(TSQBX_ERR_ARGUMENT,
                     "near_fill: the SELL fill takes sell_ptr/sell_idx/near_ptr/totals and "
                     "no CSR entries (derive them with tsqbx_sell_to_csr)");
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + L.off_cnt);
  if (!sell && n_ctr > 0 && !near_idx)
    return set_error(TSQBX_ERR_ARGUMENT, "near_fill: no output (near_idx or sell_idx)");
  const int nb = (int)((n_ctr + 127) / 128);
  const double* prm = reinterpret_cast<const double*>(ws + L.off_prm);
  const double4* sxyz = reinterpret_cast<const double4*>(ws + L.off_sxyz);
  const auto* hkey = reinterpret_cast<const unsigned long long*>(ws + L.off_hkey);
  const auto* hst = reinterpret_cast<const int32_t*>(ws + L.off_hst);
  const auto* hen = reinterpret_cast<const int32_t*>(ws + L.off_hen);
  if (n_ctr > 0 && sell)
    sweep_cell_kernel<1><<<nb, 128, 0, st>>>(ctr_xyz, radius, n_ctr, ctr_order, prm, sxyz, hkey,
                                             hst, hen, L.cap, cnt, near_ptr, nullptr, sell_ptr,
                                             sell_idx);
  else if (n_ctr > 0)
    sweep_cell_kernel<3><<<nb, 128, 0, st>>>(ctr_xyz, radius, n_ctr, ctr_order, prm, sxyz, hkey,
                                             hst, hen, L.cap, nullptr, near_ptr, near_idx,
                                             nullptr, nullptr);
  if (sell) {                           // exact lengths -> near_ptr, totals[0]
    set_tail<<<1, 1, 0, st>>>(cnt, n_ctr);
    size_t tb = L.tmp_bytes;
    cub::DeviceScan::ExclusiveSum(ws + L.off_tmp, tb, cnt, near_ptr, (int)(n_ctr + 1), st);
    const cudaError_t e = cudaMemcpyAsync(totals, near_ptr + n_ctr, sizeof(int64_t),
                                          cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return check_cuda(e, "near_fill copy");
  }
  return check_cuda(cudaGetLastError(), "near_fill launch");
}

int tsqbx_near_recount(const double* ctr_xyz, const double* radius, int64_t n_ctr, int64_t n_src,
                       void* workspace, int64_t ws_bytes, const int32_t* ctr_order,
                       int64_t* near_ptr, int64_t* totals, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_recount: workspace too small");
  if (!near_ptr || !totals || (n_ctr > 0 && (!ctr_xyz || !radius || !ctr_order)))
    return set_error(TSQBX_ERR_ARGUMENT, "near_recount: null array");
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + L.off_cnt);
  if (n_ctr > 0)
    sweep_cell_kernel<0><<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
        ctr_xyz, radius, n_ctr, ctr_order, reinterpret_cast<const double*>(ws + L.off_prm),
        reinterpret_cast<const double4*>(ws + L.off_sxyz),
        reinterpret_cast<const unsigned long long*>(ws + L.off_hkey),
        reinterpret_cast<const int32_t*>(ws + L.off_hst),
        reinterpret_cast<const int32_t*>(ws + L.off_hen), L.cap, cnt, nullptr, nullptr, nullptr,
        nullptr);
  set_tail<<<1, 1, 0, st>>>(cnt, n_ctr);
  size_t tb = L.tmp_bytes;
  cub::DeviceScan::ExclusiveSum(ws + L.off_tmp, tb, cnt, near_ptr, (int)(n_ctr + 1), st);
  const cudaError_t e = cudaMemcpyAsync(totals, near_ptr + n_ctr, sizeof(int64_t),
                                        cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "near_recount copy");
  return check_cuda(cudaGetLastError(), "near_recount launch");
}

int64_t tsqbx_near_mask_bytes(int64_t n_ctr, int64_t n_sell_bound) {
  if (n_ctr < 0 || n_sell_bound < 0) return -1;
  const int64_t n_sl = (n_ctr + 31) / 32;
  // per slice 32 * ceil(bound / 32) words, bound = slice slots / 32
  return (int64_t)(align256((n_sl + 1) * sizeof(int64_t)) +
                   align256(sizeof(unsigned) * (size_t)(n_sell_bound / 32 + 32 * n_sl + 32)));
}

int tsqbx_near_recount_masks(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                             int64_t n_src, void* workspace, int64_t ws_bytes,
                             const int32_t* ctr_order, int64_t* near_ptr, int64_t* totals,
                             void* mask_ws, int64_t mask_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_recount_masks: workspace too small");
  const int64_t n_sl = (n_ctr + 31) / 32;
  const size_t head = align256((n_sl + 1) * sizeof(int64_t));
  if (!near_ptr || !totals || !mask_ws || mask_bytes < (int64_t)head ||
      (n_ctr > 0 && (!ctr_xyz || !radius || !ctr_order)))
    return set_error(TSQBX_ERR_ARGUMENT, "near_recount_masks: null array or mask workspace");
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + L.off_cnt);
  // mask offsets per slice from the bound widths the SELL-mode count left in
  // the workspace (in-place scan)
  int64_t* mptr = reinterpret_cast<int64_t*>(mask_ws);
  unsigned* mask = reinterpret_cast<unsigned*>(static_cast<char*>(mask_ws) + head);
  mask_width<<<(int)((n_sl + 256) / 256), 256, 0, st>>>(
      reinterpret_cast<const int64_t*>(ws + L.off_wid), n_sl, mptr);
  size_t tb = L.tmp_bytes;
  cub::DeviceScan::ExclusiveSum(ws + L.off_tmp, tb, mptr, mptr, (int)(n_sl + 1), st);
  if (n_ctr > 0)
    sweep_cell_kernel<4><<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
        ctr_xyz, radius, n_ctr, ctr_order, reinterpret_cast<const double*>(ws + L.off_prm),
        reinterpret_cast<const double4*>(ws + L.off_sxyz),
        reinterpret_cast<const unsigned long long*>(ws + L.off_hkey),
        reinterpret_cast<const int32_t*>(ws + L.off_hst),
        reinterpret_cast<const int32_t*>(ws + L.off_hen), L.cap, cnt, nullptr, nullptr, nullptr,
        nullptr, mptr, mask);
  set_tail<<<1, 1, 0, st>>>(cnt, n_ctr);
  tb = L.tmp_bytes;
  cub::DeviceScan::ExclusiveSum(ws + L.off_tmp, tb, cnt, near_ptr, (int)(n_ctr + 1), st);
  const cudaError_t e = cudaMemcpyAsync(totals, near_ptr + n_ctr, sizeof(int64_t),
                                        cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "near_recount_masks copy");
  return check_cuda(cudaGetLastError(), "near_recount_masks launch");
}

int tsqbx_near_fill_masks(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                          int64_t n_src, void* workspace, int64_t ws_bytes,
                          const int32_t* ctr_order, int64_t* near_ptr, const int64_t* sell_ptr,
                          int32_t* sell_idx, int64_t* totals, const void* mask_ws,
                          int64_t mask_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_fill_masks: workspace too small");
  const int64_t n_sl = (n_ctr + 31) / 32;
  const size_t head = align256((n_sl + 1) * sizeof(int64_t));
  if (!near_ptr || !totals || !sell_ptr || !sell_idx || !mask_ws || mask_bytes < (int64_t)head ||
      (n_ctr > 0 && (!ctr_xyz || !radius || !ctr_order)))
    return set_error(TSQBX_ERR_ARGUMENT, "near_fill_masks: null array or mask workspace");
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + L.off_cnt);
  const int64_t* mptr = reinterpret_cast<const int64_t*>(mask_ws);
  unsigned* mask = reinterpret_cast<unsigned*>(
      const_cast<char*>(static_cast<const char*>(mask_ws)) + head);
  if (n_ctr > 0)
    sweep_cell_kernel<5><<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
        ctr_xyz, radius, n_ctr, ctr_order, reinterpret_cast<const double*>(ws + L.off_prm),
        reinterpret_cast<const double4*>(ws + L.off_sxyz),
        reinterpret_cast<const unsigned long long*>(ws + L.off_hkey),
        reinterpret_cast<const int32_t*>(ws + L.off_hst),
        reinterpret_cast<const int32_t*>(ws + L.off_hen), L.cap, cnt, near_ptr, nullptr, sell_ptr,
        sell_idx, mptr, mask);
  set_tail<<<1, 1, 0, st>>>(cnt, n_ctr);
  size_t tb = L.tmp_bytes;
  cub::DeviceScan::ExclusiveSum(ws + L.off_tmp, tb, cnt, near_ptr, (int)(n_ctr + 1), st);
  const cudaError_t e = cudaMemcpyAsync(totals, near_ptr + n_ctr, sizeof(int64_t),
                                        cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "near_fill_masks copy");
  return check_cuda(cudaGetLastError(), "near_fill_masks launch");
}

int tsqbx_near_fill_rows(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                         const double* src_xyz, int64_t n_src, void* workspace, int64_t ws_bytes,
                         const int32_t* ctr_order, int64_t g0, int64_t g1, int64_t* near_ptr,
                         const int64_t* sell_ptr, int32_t* sell_idx, int64_t* totals,
                         void* stream) {
  (void)src_xyz;
  cudaStream_t st = (cudaStream_t)stream;
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_fill_rows: workspace too small");
  if (g0 < 0 || g1 < g0 || g1 > n_ctr || (g0 & 31) || !near_ptr || !sell_ptr || !sell_idx ||
      !totals || (g1 > g0 && (!ctr_xyz || !radius || !ctr_order)))
    return set_error(TSQBX_ERR_ARGUMENT,
                     "near_fill_rows: bad row range (g0 must be a multiple of 32) or null array");
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + L.off_cnt);
  const int64_t n = g1 - g0;
  // rows g0..g1 of the processing order (a rank's shard): the same sweep as
  // tsqbx_near_fill with the row index shifted, the source grid and hash of
  // tsqbx_near_count shared by all ranges
  if (n > 0)
    sweep_cell_kernel<1><<<(int)((n + 127) / 128), 128, 0, st>>>(
        ctr_xyz, radius, n, ctr_order + g0, reinterpret_cast<const double*>(ws + L.off_prm),
        reinterpret_cast<const double4*>(ws + L.off_sxyz),
        reinterpret_cast<const unsigned long long*>(ws + L.off_hkey),
        reinterpret_cast<const int32_t*>(ws + L.off_hst),
        reinterpret_cast<const int32_t*>(ws + L.off_hen), L.cap, cnt, near_ptr, nullptr,
        sell_ptr, sell_idx);
  set_tail<<<1, 1, 0, st>>>(cnt, n);
  size_t tb = L.tmp_bytes;
  cub::DeviceScan::ExclusiveSum(ws + L.off_tmp, tb, cnt, near_ptr, (int)(n + 1), st);
  const cudaError_t e = cudaMemcpyAsync(totals, near_ptr + n, sizeof(int64_t),
                                        cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "near_fill_rows copy");
  return check_cuda(cudaGetLastError(), "near_fill_rows launch");
}

int64_t tsqbx_order_workspace_bytes(int64_t n_ctr) {
  if (n_ctr < 0) return -1;
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_ctr + 1));
  return (int64_t)(align256((n_ctr + 1) * sizeof(int64_t)) + align256(t));
}

int tsqbx_order_targets(int64_t n_ctr, const int32_t* ctr_order, const double* ctr_xyz,
                        const int64_t* tgt_ptr, const double* tgt_xyz, const double* tgt_nrm,
                        int64_t n_tgt, void* workspace, int64_t ws_bytes, double* ctr_out,
                        int64_t* tptr_out, double* tgt_out, double* tnrm_out, int64_t* tgt_index,
                        int64_t* bad, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_ctr < 0 || ws_bytes < tsqbx_order_workspace_bytes(n_ctr) || !workspace)
    return set_error(TSQBX_ERR_ARGUMENT, "order_targets: bad sizes or workspace");
  if (n_ctr > 0 && (!ctr_order || !ctr_xyz || !tgt_ptr || !ctr_out || !tptr_out || !tgt_index ||
                    (tgt_nrm && !tnrm_out)))
    return set_error(TSQBX_ERR_ARGUMENT, "order_targets: null array");
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws);
  void* tmp = ws + align256((n_ctr + 1) * sizeof(int64_t));
  size_t tb = (size_t)ws_bytes - align256((n_ctr + 1) * sizeof(int64_t));
  if (bad) {
    const cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int64_t), st);
    if (e != cudaSuccess) return check_cuda(e, "order_targets memset");
  }
  order_count<<<(int)((n_ctr + 256) / 256), 256, 0, st>>>(ctr_order, tgt_ptr, n_ctr, n_tgt, cnt,
                                                          bad);
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, tptr_out, (int)(n_ctr + 1), st);
  if (n_ctr > 0)
    order_copy<<<(int)((n_ctr + 255) / 256), 256, 0, st>>>(ctr_order, ctr_xyz, tgt_ptr, tgt_xyz,
                                                            tgt_nrm, n_ctr, n_tgt, cnt,
                                                            tptr_out, ctr_out,
                                                            tgt_out, tnrm_out, tgt_index);
  return check_cuda(cudaGetLastError(), "order_targets launch");
}

int64_t tsqbx_sell_workspace_bytes(int64_t n_rows) {
  if (n_rows < 0) return -1;
  const int64_t n_sl = (n_rows + 31) / 32;
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_sl + 1));
  return (int64_t)(align256((n_sl + 1) * sizeof(int64_t)) + align256(t));
}

int tsqbx_sell_size(int64_t n_rows, const int64_t* near_ptr, void* workspace, int64_t ws_bytes,
                    int64_t* sell_ptr, int64_t* n_entries, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows < 0 || !workspace || ws_bytes < tsqbx_sell_workspace_bytes(n_rows) || !sell_ptr ||
      !n_entries || (n_rows > 0 && !near_ptr))
    return set_error(TSQBX_ERR_ARGUMENT, "sell_size: bad arguments");
  const int64_t n_sl = (n_rows + 31) / 32;
  char* ws = static_cast<char*>(workspace);
  int64_t* wid = reinterpret_cast<int64_t*>(ws);
  void* tmp = ws + align256((n_sl + 1) * sizeof(int64_t));
  size_t tb = (size_t)ws_bytes - align256((n_sl + 1) * sizeof(int64_t));
  if (n_sl > 0)
    sell_width<<<(int)((n_sl * 32 + 255) / 256), 256, 0, st>>>(near_ptr, n_rows, wid);
  sell_tail<<<1, 1, 0, st>>>(wid, n_sl);
  cub::DeviceScan::ExclusiveSum(tmp, tb, wid, sell_ptr, (int)(n_sl + 1), st);
  cudaError_t e = cudaMemcpyAsync(n_entries, sell_ptr + n_sl, sizeof(int64_t),
                                  cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "sell_size copy");
  return check_cuda(cudaGetLastError(), "sell_size launch");
}

int tsqbx_sell_fill(int64_t n_rows, const int64_t* near_ptr, const int32_t* near_idx,
                    const int64_t* sell_ptr, int32_t* sell_idx, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!near_ptr || !sell_ptr || !sell_idx)))
    return set_error(TSQBX_ERR_ARGUMENT, "sell_fill: bad arguments");
  if (n_rows == 0) return TSQBX_OK;
  sell_fill_kernel<<<(int)((n_rows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      near_ptr, near_idx, n_rows, sell_ptr, sell_idx);
  return check_cuda(cudaGetLastError(), "sell_fill launch");
}

int tsqbx_sell_compact(int64_t n_rows, const int64_t* sell_ptr_src, const int32_t* sell_idx_src,
                       const int64_t* sell_ptr_dst, int32_t* sell_idx_dst, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!sell_ptr_src || !sell_idx_src || !sell_ptr_dst ||
                                    !sell_idx_dst)))
    return set_error(TSQBX_ERR_ARGUMENT, "sell_compact: bad arguments");
  const int64_t n_sl = (n_rows + 31) / 32;
  if (n_sl == 0) return TSQBX_OK;
  sell_compact_kernel<<<(unsigned)((n_sl * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      n_sl, sell_ptr_src, sell_idx_src, sell_ptr_dst, sell_idx_dst);
  return check_cuda(cudaGetLastError(), "sell_compact launch");
}

int tsqbx_sell_window(int64_t n_rows, const int64_t* near_ptr, const int64_t* sell_ptr,
                      const int32_t* sell_idx, int32_t* loc_idx, int32_t* win_src,
                      int32_t* win_len, unsigned* overflow, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!near_ptr || !sell_ptr || !sell_idx || !loc_idx ||
                                    !win_src || !win_len || !overflow)))
    return set_error(TSQBX_ERR_ARGUMENT, "sell_window: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(overflow, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return check_cuda(e, "sell_window memset");
  if (n_rows == 0) return TSQBX_OK;
  const int64_t threads = (n_rows + 31) / 32 * 32;
  sell_window_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(
      near_ptr, n_rows, sell_ptr, sell_idx, loc_idx, win_src, win_len, overflow);
  return check_cuda(cudaGetLastError(), "sell_window launch");
}

int tsqbx_sell_to_csr(int64_t n_rows, const int64_t* near_ptr, const int64_t* sell_ptr,
                      const int32_t* sell_idx, int32_t* near_idx, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!near_ptr || !sell_ptr || !sell_idx || !near_idx)))
    return set_error(TSQBX_ERR_ARGUMENT, "sell_to_csr: bad arguments");
  if (n_rows == 0) return TSQBX_OK;
  sell_to_csr_kernel<<<(int)((n_rows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      near_ptr, n_rows, sell_ptr, sell_idx, near_idx);
  return check_cuda(cudaGetLastError(), "sell_to_csr launch");
}

int tsqbx_scatter_c128(int64_t n, const int64_t* dest, const double* src, double* out,
                       void* stream) {
  if (n < 0 || (n > 0 && (!src || !out)))
    return set_error(TSQBX_ERR_ARGUMENT, "scatter_c128: bad arguments");
  if (n == 0) return TSQBX_OK;
  scatter_c128<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      n, dest, reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(out));
  return check_cuda(cudaGetLastError(), "scatter_c128 launch");
}

}  // extern "C"
