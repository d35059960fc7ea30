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

#include "common.cuh"

namespace tsqbx {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kFineBits = 21;
constexpr int kSubBits = 3;  // level-0 coarse cell = 8 fine cells per axis
// Cell levels: a center of radius r searches the 27 neighbours of its cell at
// the smallest level L whose cell (8 fine cells << L) is >= r.  The fine grid
// follows the smallest radius (down to rmax / 2^(kLevels-1)), so centers with
// small radii no longer scan cells sized for the largest (C5's 16 spheres of
// different radii, C4's per-source radii).  Level L cells are prefixes of the
// fine Morton keys, so one source sort serves every level; the hash key of a
// level-L cell carries L in bits 60-61.
constexpr int kLevels = 4;
// Levels multiply the hash entries; past ~1 M sources the table no longer
// stays in L2 and the extra inserts and lookups cost more than the candidate
// tests they save (C5 literal, 8.4 M sources: 10.8 ms one level, 12.3 ms four;
// C4 literal, 1 M sources: 1.87 ms one level, 1.53 ms four).
#ifndef TSQBX_MULTILEVEL_MAX_SRC
#define TSQBX_MULTILEVEL_MAX_SRC (1 << 20)
#endif
constexpr int64_t kMultiLevelMaxSources = TSQBX_MULTILEVEL_MAX_SRC;
constexpr int kFineOffset = 1 << (kSubBits + kLevels - 1);  // coarse coordinate >= 1 at every level

struct NearLayout {
  size_t off_mm, off_prm, off_skey_in, off_skey, off_sval_in, off_ckey_in, off_ckey, off_cval_in,
      off_sxyz, off_hkey, off_hst, off_hen, off_cnt, off_wid, off_tmp, total;
  int64_t cap;
  size_t tmp_bytes;
};

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

NearLayout near_layout(int64_t n_ctr, int64_t n_src) {
  NearLayout L{};
  int64_t cap = 1024;
  // room for the cells of every level while the table stays L2-resident
  const int64_t factor = n_src <= kMultiLevelMaxSources ? 4 : 2;
  while (cap < factor * n_src) cap <<= 1;
  L.cap = cap;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  L.off_mm = take(8 * sizeof(long long));
  L.off_prm = take(8 * sizeof(double));
  L.off_skey_in = take(n_src * sizeof(unsigned long long));
  L.off_skey = take(n_src * sizeof(unsigned long long));
  L.off_sval_in = take(n_src * sizeof(int32_t));
  L.off_ckey_in = take(n_ctr * sizeof(unsigned long long));
  L.off_ckey = take(n_ctr * sizeof(unsigned long long));
  L.off_cval_in = take(n_ctr * sizeof(int32_t));
  L.off_sxyz = take(n_src * sizeof(double4));
  L.off_hkey = take(cap * sizeof(unsigned long long));
  L.off_hst = take(cap * sizeof(int32_t));
  L.off_hen = take(cap * sizeof(int32_t));
  L.off_cnt = take((n_ctr + 1) * sizeof(int64_t));
  const int64_t n_sl = (n_ctr + 31) / 32;
  L.off_wid = take((n_sl + 1) * sizeof(int64_t));
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)n_src, 0, 3 * kFineBits);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)n_ctr, 0, 3 * kFineBits);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_ctr + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, t4, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_sl + 1));
  L.tmp_bytes = std::max(std::max(t1, t4), std::max(t2, t3)) + 256;
  L.off_tmp = take(L.tmp_bytes);
  L.total = o;
  return L;
}

__device__ __forceinline__ long long ord_of(double d) {
  const long long b = __double_as_longlong(d);
  return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
}
__device__ __forceinline__ double of_ord(long long b) {
  return __longlong_as_double(b >= 0 ? b : b ^ 0x7fffffffffffffffLL);
}

__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ unsigned long long morton3(unsigned long long x, unsigned long long y,
                                                      unsigned long long z) {
  return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}
__device__ __forceinline__ unsigned long long hash64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
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

// the level whose cells cover a ball of radius r (its 27 neighbours)
__device__ __forceinline__ int cell_level(double r, const double* prm) {
  const int top = (int)prm[4];
  int lv = 0;
  while (lv < top && prm[3] * (double)(1 << (kSubBits + lv)) < r * (1.0 + 1e-9)) ++lv;
  return lv;
}
__device__ __forceinline__ unsigned long long level_tag(int lv) {
  return (unsigned long long)lv << 60;
}

__device__ __forceinline__ void fine_coords(const double* p, const double* prm,
                                            unsigned long long* f) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double q = floor((p[d] - prm[d]) / prm[3]);
    q = fmin(fmax(q, 0.0), (double)((1 << kFineBits) - 2 * kFineOffset));
    f[d] = (unsigned long long)q + kFineOffset;  // coarse coordinate >= 1 at every level
  }
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

__device__ __forceinline__ bool hash_find(const unsigned long long* __restrict__ hkey,
                                          const int32_t* __restrict__ hst,
                                          const int32_t* __restrict__ hen, int64_t cap,
                                          unsigned long long ck, int& st, int& en) {
  int64_t h = (int64_t)(hash64(ck) & (unsigned long long)(cap - 1));
  while (true) {
    const unsigned long long k = hkey[h];
    if (k == ck) {
      st = hst[h];
      en = hen[h];
      return true;
    }
    if (k == kEmpty) return false;
    h = (h + 1) & (cap - 1);
  }
}

__device__ __forceinline__ bool member(const double4 s, double cx, double cy, double cz,
                                       double rad2) {
  const double dx = __dadd_rn(s.x, -cx), dy = __dadd_rn(s.y, -cy), dz = __dadd_rn(s.z, -cz);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return d2 <= rad2;
}

// one WARP per 32 consecutive centers (processing order).  Consecutive centers
// share their coarse cell (Morton order), so the warp walks the distinct cells
// of its lanes; for each cell the 27 neighbour cells are looked up once (lane
// l < 27 probes neighbour l) and their sources are staged into a per-warp
// shared-memory tile of kTile candidates (all neighbour-cell copies issued
// back to back, coalesced), which every lane of that cell then tests with
// broadcast reads.  Row order = neighbour order (dx, dy, dz), ascending within
// a cell -- identical in the count and the fill pass.
// 128-candidate tiles and <= 64 registers (8 CTAs of 128 threads per SM):
// measured equal on dense lists, 9 % faster on the literal preset
constexpr int kTile = 128;
constexpr int kMaxCells = 128;   // cells one union pass stages (non-empty ones)
// fill: members of the busiest lane in a 32-candidate group from which the
// append walks all 32 candidates instead of each lane's own members
#ifndef TSQBX_WALK_ABOVE
#define TSQBX_WALK_ABOVE 20
#endif
constexpr unsigned kWalkAbove = TSQBX_WALK_ABOVE;
// SELL fill: 16-byte block stores (1) or one 4-byte store per entry (0)
#ifndef TSQBX_INT4_STORES
#define TSQBX_INT4_STORES 1
#endif
constexpr bool kInt4Stores = TSQBX_INT4_STORES != 0;

// MODE 0: count members per row; 1: fill the SELL column (plus the row length
// when `cnt` is given); 3: fill the CSR row; 2: bound -- no distance tests, the
// slice width (32 x the largest candidate count of its rows, a multiple of 4)
// into `cnt[slice]`, so the fill can write before the exact lengths are known.
template <int MODE>
__global__ void __launch_bounds__(128, 8) sweep_cell_kernel(
    const double* __restrict__ ctr, const double* __restrict__ rad, int64_t n_ctr,
    const int32_t* __restrict__ order, const double* __restrict__ prm,
    const double4* __restrict__ sxyz, const unsigned long long* __restrict__ hkey,
    const int32_t* __restrict__ hst, const int32_t* __restrict__ hen, int64_t cap,
    int64_t* __restrict__ cnt, const int64_t* __restrict__ nptr, int32_t* __restrict__ nidx,
    const int64_t* __restrict__ sptr, int32_t* __restrict__ sidx) {
  constexpr bool FILL = MODE == 1 || MODE == 3;
  // staged candidates as fp32 offsets from the warp's reference point (see
  // run_cells) plus their sorted index; the exact fp64 test reads sxyz only for
  // the rare candidates inside the fp32 error band
  // candidate pairs for the packed-fp32 (FFMA2) test: pair p of the tile is
  // tab[p] = {x0, x1, y0, y1}, tcd[p] = {z0, z1, w0, w1}
  __shared__ float4 tab[4][kTile / 2], tcd[4][kTile / 2];
  __shared__ int32_t tid_[4][kTile];
  __shared__ int32_t cell_st[4][kMaxCells], cell_en[4][kMaxCells];   // a warp's cell list
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = g < n_ctr;
  double cx = 0.0, cy = 0.0, cz = 0.0, rad2 = -1.0;
  unsigned long long ccx = 0, ccy = 0, ccz = 0, ckey = kEmpty;
  int lv = 0;                          // this center's cell level
  if (valid) {
    const int64_t ic = order[g];
    cx = ctr[3 * ic];
    cy = ctr[3 * ic + 1];
    cz = ctr[3 * ic + 2];
    const double r = rad[ic];
    rad2 = __dmul_rn(r, r);
    const double pl[3] = {cx, cy, cz};
    const double prm_l[4] = {prm[0], prm[1], prm[2], prm[3]};
    unsigned long long f[3];
    fine_coords(pl, prm_l, f);
    lv = cell_level(r, prm);
    ccx = f[0] >> (kSubBits + lv);
    ccy = f[1] >> (kSubBits + lv);
    ccz = f[2] >> (kSubBits + lv);
    ckey = morton3(ccx, ccy, ccz) | level_tag(lv);
  }
  // MODE 3: CSR row; MODE 1: SELL-32x4 column, entry k at dst[128 (k / 4) + k % 4]
  int32_t* dst = (MODE == 3 && valid) ? nidx + nptr[g]
                 : (MODE == 1 && valid) ? sidx + sptr[g >> 5] + 4 * (g & 31) : nullptr;
  int k = 0;
  int4 pend = make_int4(0, 0, 0, 0);   // MODE 1 with kInt4Stores: the row's open block
  int64_t ub = 0;                      // MODE 2: candidates this row will test
  // Stage the sources of a list of up to kMaxCells cells (ranges [st, en) in
  // cell_st / cell_en of this warp, written by the caller) through the tile;
  // lanes with `mine` test them all.  o: the reference point (a center of this
  // warp); A: a bound on |p - o| (max norm) of every staged source and every
  // testing lane's center.
  auto run_cells = [&](int ncell, bool mine, double ox, double oy, double oz, double A) {
    // fp32 prefilter in dot-product form: with s' = s - o, c' = c - o (every
    // coordinate |.| <= A) a candidate is a member iff
    //   f = s'.c' - |s'|^2 / 2  >=  K = (|c'|^2 - rad^2) / 2,
    // i.e. three FFMAs per (candidate, lane) against a staged (s', -|s'|^2/2).
    // Rounding s', c', w' and K to fp32 and the fp32 FMAs move f - K by at
    // most ~40 u A^2 (u = 2^-24); candidates with |f - K| <= 2^-14 A^2 (> 10x
    // that) take the exact fp64 test (member()) after the group, the rest are
    // decided in fp32 -- membership stays bit-identical to the oracle
    const float tau = (float)(A * A * (1.0 / 16384.0));
    const double cdx = cx - ox, cdy = cy - oy, cdz = cz - oz;
    const float K = (float)(0.5 * (cdx * cdx + cdy * cdy + cdz * cdz - rad2));
    const float Khi = K + tau, Klo = K - tau;
    const float cfx = (float)cdx, cfy = (float)cdy, cfz = (float)cdz;
    // exclusive prefix of the cell sizes (cell c in lane c % 32, slot c / 32),
    // kept in cell_en, so that a tile of candidates spanning many small cells
    // is staged with all its loads in flight at once (one latency per tile)
    int total = 0;
    int pre[kMaxCells / 32];
#pragma unroll
    for (int q = 0; q < kMaxCells / 32; ++q) {
      const int c = lane + 32 * q;
      const int sz = c < ncell ? cell_en[wib][c] - cell_st[wib][c] : 0;
      int inc = sz;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += a;
      }
      pre[q] = total + inc - sz;
      total += __shfl_sync(0xffffffffu, inc, 31);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kMaxCells / 32; ++q) cell_en[wib][lane + 32 * q] = pre[q];
    __syncwarp();
    const int nc = min(ncell, kMaxCells);
    for (int base = 0; base < total; base += kTile) {
      const int fill = min(kTile, total - base);
#pragma unroll
      for (int r = 0; r < kTile / 32; ++r) {
        const int q = lane + 32 * r;
        if (q < fill) {
          const int t = base + q;
          int lo_c = 0, hi_c = nc - 1;               // last cell with prefix <= t
          while (lo_c < hi_c) {
            const int mid = (lo_c + hi_c + 1) >> 1;
            if (cell_en[wib][mid] <= t) lo_c = mid;
            else hi_c = mid - 1;
          }
          const int j = cell_st[wib][lo_c] + (t - cell_en[wib][lo_c]);
          const double4 sj = sxyz[j];
          const float x = (float)(sj.x - ox), y = (float)(sj.y - oy), z = (float)(sj.z - oz);
          float* pa = reinterpret_cast<float*>(&tab[wib][q >> 1]) + (q & 1);
          float* pc = reinterpret_cast<float*>(&tcd[wib][q >> 1]) + (q & 1);
          pa[0] = x;
          pa[2] = y;
          pc[0] = z;
          pc[2] = -0.5f * fmaf(z, z, fmaf(y, y, x * x));
          tid_[wib][q] = j;
        }
      }
      __syncwarp();
      if (mine) {
        // test 32 staged candidates into a per-lane bit mask, then append only
        // this lane's members (no per-candidate divergent work in the fill)
        for (int t0 = 0; t0 < fill; t0 += 32) {
          const int m = min(32, fill - t0);
          // candidate u lands in bit 31 - u: each test shifts the sign bit of
          // f - K -/+ tau into a mask with one funnel shift (SHF); candidates
          // go in pairs through packed fp32 (FFMA2 / FADD2), so a pair costs
          // 2 LDS.128 + 3 FFMA2 + 2 FADD2 + 4 SHF
          unsigned below_hi = 0u, below_lo = 0u;
          const float2 cx2 = make_float2(cfx, cfx), cy2 = make_float2(cfy, cfy),
                       cz2 = make_float2(cfz, cfz);
          const float2 nkhi = make_float2(-Khi, -Khi), nklo = make_float2(-Klo, -Klo);
#pragma unroll 4
          for (int u = 0; u < 32; u += 2) {
            const float4 a = tab[wib][(t0 + u) >> 1], c = tcd[wib][(t0 + u) >> 1];
            const float2 f = __ffma2_rn(make_float2(a.x, a.y), cx2,
                                        __ffma2_rn(make_float2(a.z, a.w), cy2,
                                                   __ffma2_rn(make_float2(c.x, c.y), cz2,
                                                              make_float2(c.z, c.w))));
            const float2 gh = __fadd2_rn(f, nkhi), gl = __fadd2_rn(f, nklo);
            below_hi = __funnelshift_l(__float_as_uint(gh.x), below_hi, 1);
            below_hi = __funnelshift_l(__float_as_uint(gh.y), below_hi, 1);
            below_lo = __funnelshift_l(__float_as_uint(gl.x), below_lo, 1);
            below_lo = __funnelshift_l(__float_as_uint(gl.y), below_lo, 1);
          }
          // slots past `m` hold stale candidates (low bits): masked, not branched on
          const unsigned live = m == 32 ? ~0u : ~((1u << (32 - m)) - 1u);
          unsigned bits = ~below_hi & live;                 // surely inside
          unsigned band = below_hi & ~below_lo & live;      // within tau of the sphere
          while (band) {                     // rare: the exact fp64 test
            const int u = __clz(band);
            band &= ~(0x80000000u >> u);
            if (member(sxyz[tid_[wib][t0 + u]], cx, cy, cz, rad2)) bits |= 0x80000000u >> u;
          }
          if (!FILL) {
            k += __popc(bits);
          } else {
            // append this lane's members to its row in candidate order.  A group
            // of 32 Morton-consecutive candidates is spatially compact, so a
            // lane whose ball covers it takes most of it while others take none:
            // with many members per lane a uniform walk over the candidates
            // (every lane stores its own) beats a per-lane loop that runs as
            // long as the busiest lane
            auto put = [&](int j) {
              if (MODE == 3 || !kInt4Stores) {
                dst[MODE == 3 ? k : ((k >> 2) << 7) | (k & 3)] = j;
              } else {
                // SELL: the row's current block as a 4-entry shift register,
                // one 16-byte store per completed block
                pend.x = pend.y;
                pend.y = pend.z;
                pend.z = pend.w;
                pend.w = j;
                if ((k & 3) == 3) *reinterpret_cast<int4*>(dst + ((k >> 2) << 7)) = pend;
              }
              ++k;
            };
            // (only the lanes testing this list are active here: per-cell mode)
            if (__reduce_max_sync(__activemask(), (unsigned)__popc(bits)) >= kWalkAbove) {
#pragma unroll 4
              for (int u = 0; u < 32; ++u) {
                const int j = tid_[wib][t0 + u];
                if ((int)(bits << u) < 0) put(j);
              }
            } else {
              while (bits) {
                const int u = __clz(bits);      // candidate order: bit 31 - u
                bits &= ~(0x80000000u >> u);
                put(tid_[wib][t0 + u]);
              }
            }
          }
        }
      }
      __syncwarp();
    }
  };
  auto lookup = [&](unsigned long long x, unsigned long long y, unsigned long long z, int level,
                    int& st, int& en) {
    st = en = 0;
    if (!hash_find(hkey, hst, hen, cap, morton3(x, y, z) | level_tag(level), st, en)) en = st;
  };
  // Union mode: every lane scans every cell that meets the warp's region
  // [bbox - Rmax, bbox + Rmax] (bbox of its 32 centers, Rmax their largest
  // radius) at the finest cell level where those cells number <= kMaxCells;
  // candidates outside a lane's own ball simply fail the distance test.  Any
  // level works here (not only cells >= r), so literal radii (a few sources
  // per center, cells smaller than the warp's span) use a coarser level
  // instead of falling back to the per-cell mode below.
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double blo[3] = {valid ? cx : inf, valid ? cy : inf, valid ? cz : inf};
  double bhi[3] = {valid ? cx : -inf, valid ? cy : -inf, valid ? cz : -inf};
  double rmx = valid ? sqrt(rad2) : 0.0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      blo[d] = fmin(blo[d], __shfl_xor_sync(0xffffffffu, blo[d], off));
      bhi[d] = fmax(bhi[d], __shfl_xor_sync(0xffffffffu, bhi[d], off));
    }
    rmx = fmax(rmx, __shfl_xor_sync(0xffffffffu, rmx, off));
  }
  const bool any_valid = __any_sync(0xffffffffu, valid);
  // slack: the rounded membership test may accept a source a few ulps outside
  // the exact ball; IEEE subtraction/division are monotone, so every source
  // inside the slackened box maps into the box's corner cells
  const double rb = rmx * (1.0 + 1e-9) + 1e-300;
  int lw = -1;                          // union level
  unsigned long long clo[3] = {0, 0, 0}, chi[3] = {0, 0, 0};
  if (any_valid) {
    const double plo[3] = {blo[0] - rb, blo[1] - rb, blo[2] - rb};
    const double phi[3] = {bhi[0] + rb, bhi[1] + rb, bhi[2] + rb};
    const double prm_l[4] = {prm[0], prm[1], prm[2], prm[3]};
    unsigned long long flo[3], fhi[3];
    fine_coords(plo, prm_l, flo);
    fine_coords(phi, prm_l, fhi);
    const int top = (int)prm[4];
    for (int L = 0; L <= top; ++L) {
      const int sh = kSubBits + L;
      const unsigned long long n = ((fhi[0] >> sh) - (flo[0] >> sh) + 1) *
                                   ((fhi[1] >> sh) - (flo[1] >> sh) + 1) *
                                   ((fhi[2] >> sh) - (flo[2] >> sh) + 1);
      if (n <= (unsigned long long)kMaxCells) {
        lw = L;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          clo[d] = flo[d] >> sh;
          chi[d] = fhi[d] >> sh;
        }
        break;
      }
    }
  }
  if (lw >= 0) {
    // the region's cells (x-major order), non-empty ones compacted in order
    const unsigned long long ex = chi[0] - clo[0] + 1, ey = chi[1] - clo[1] + 1,
                             ez = chi[2] - clo[2] + 1;
    const int ncell = (int)(ex * ey * ez);
    int n_ne = 0;
    int64_t mine_sz = 0;
#pragma unroll
    for (int slot = 0; slot < kMaxCells / 32; ++slot) {
      const int c = lane + 32 * slot;
      int st = 0, en = 0;
      if (c < ncell) {
        const unsigned eyz = (unsigned)(ey * ez), ezu = (unsigned)ez, cu = (unsigned)c;
        const unsigned ix = cu / eyz, iy = (cu / ezu) % (unsigned)ey, iz = cu % ezu;
        lookup(clo[0] + ix, clo[1] + iy, clo[2] + iz, lw, st, en);
      }
      const unsigned ne = __ballot_sync(0xffffffffu, en > st);
      const int at = n_ne + __popc(ne & ((1u << lane) - 1u));
      if (en > st) {
        cell_st[wib][at] = st;
        cell_en[wib][at] = en;
        mine_sz += en - st;
      }
      n_ne += __popc(ne);
    }
    __syncwarp();
    if (MODE == 2) {
      for (int off = 16; off > 0; off >>= 1) mine_sz += __shfl_xor_sync(0xffffffffu, mine_sz, off);
      ub = mine_sz;
    } else if (n_ne > 0) {
      // reference point: the first valid lane's center; every staged source
      // lies within one cell of the region, every lane center in the bbox
      const int l0 = __ffs(__ballot_sync(0xffffffffu, valid)) - 1;
      const double ox = __shfl_sync(0xffffffffu, cx, l0), oy = __shfl_sync(0xffffffffu, cy, l0),
                   oz = __shfl_sync(0xffffffffu, cz, l0);
      const double cs = prm[3] * (double)(1ull << (kSubBits + lw));
      const double A = fmax(bhi[0] - blo[0], fmax(bhi[1] - blo[1], bhi[2] - blo[2])) + rb + 2.0 * cs;
      run_cells(n_ne, valid, ox, oy, oz, A);
    }
  } else if (any_valid) {
    // per distinct cell of the warp: its 27 neighbours, only that cell's lanes test
    // one head per distinct (cell, level): lanes of one cell need not be
    // adjacent when their levels differ
    const unsigned peers = __match_any_sync(0xffffffffu, ckey);
    unsigned heads = __ballot_sync(0xffffffffu, valid && lane == __ffs(peers) - 1);
    while (heads) {
      const int a = __ffs(heads) - 1;
      heads &= heads - 1;
      const unsigned long long cell = __shfl_sync(0xffffffffu, ckey, a);
      const unsigned long long bx = __shfl_sync(0xffffffffu, ccx, a);
      const unsigned long long by = __shfl_sync(0xffffffffu, ccy, a);
      const unsigned long long bz = __shfl_sync(0xffffffffu, ccz, a);
      const int bl = __shfl_sync(0xffffffffu, lv, a);
      int st = 0, en = 0;
      if (lane < 27)
        lookup(bx + (lane / 9) - 1, by + ((lane / 3) % 3) - 1, bz + (lane % 3) - 1, bl, st, en);
      if (MODE == 2) {
        int64_t tot = en - st;
        for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
        if (valid && ckey == cell) ub = tot;
      } else {
        // reference point: the head lane's center; sources in the 3 x 3 x 3
        // cells around its cell, testing lanes' centers in that cell
        const double ox = __shfl_sync(0xffffffffu, cx, a), oy = __shfl_sync(0xffffffffu, cy, a),
                     oz = __shfl_sync(0xffffffffu, cz, a);
        const double A = 4.0 * prm[3] * (double)(1ull << (kSubBits + bl));
        __syncwarp();
        if (lane < 27) {
          cell_st[wib][lane] = st;
          cell_en[wib][lane] = en;
        }
        __syncwarp();
        run_cells(27, valid && ckey == cell, ox, oy, oz, A);
      }
    }
  }
  if (MODE == 1 && kInt4Stores && valid && (k & 3)) {   // the last, partial block
    const int r = k & 3;                                // entries pending in pend's tail
    int4 blk = pend;
    if (r == 1) blk.x = pend.w;
    if (r == 2) { blk.x = pend.z; blk.y = pend.w; }
    if (r == 3) { blk.x = pend.y; blk.y = pend.z; blk.z = pend.w; }
    *reinterpret_cast<int4*>(dst + ((k >> 2) << 7)) = blk;
  }
  if (MODE == 0 && valid) cnt[g] = k;
  if (MODE == 1 && valid && cnt) cnt[g] = k;
  if (MODE == 2) {
    for (int off = 16; off > 0; off >>= 1) ub = max(ub, __shfl_xor_sync(0xffffffffu, ub, off));
    if (lane == 0 && (g >> 5) * 32 < n_ctr) cnt[g >> 5] = 32 * ((ub + 3) & ~3ll);
  }
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

int tsqbx_near_count(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                     const double* src_xyz, int64_t n_src, void* workspace, int64_t ws_bytes,
                     int32_t* src_perm, int32_t* ctr_order, int64_t* near_ptr,
                     int64_t* sell_ptr, int64_t* totals, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_ctr < 0 || n_src < 0 || n_src > INT32_MAX - 64 || n_ctr > INT32_MAX - 64)
    return set_error(TSQBX_ERR_ARGUMENT, "near_count: bad sizes");
  const NearLayout L = near_layout(n_ctr, n_src);
  if (!workspace || ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "near_count: workspace too small (need %lld)",
                     (long long)L.total);
  if (!near_ptr || !totals || (n_ctr > 0 && (!ctr_xyz || !radius || !ctr_order)) ||
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
    if (!sell_ptr)
      sweep_cell_kernel<0><<<(int)((n_ctr + 127) / 128), 128, 0, st>>>(
          ctr_xyz, radius, n_ctr, ctr_order, prm, sxyz, hkey, hst, hen, L.cap, cnt, nullptr,
          nullptr, nullptr, nullptr);
  }
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
