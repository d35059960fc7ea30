// near_sweep.cuh -- the radius-ball membership sweep of the near-list builder
// (one warp per 32 consecutive centers), shared by the builder's kernels
// (near.cu) and the fused build+evaluate kernel (fused.cu), with the cell
// grid, Morton and hash helpers and the builder's workspace layout.
#pragma once

#include <cub/cub.cuh>

#include <algorithm>
#include <climits>

#include "common.cuh"

namespace tsqbx {
namespace nsw {

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

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

inline NearLayout near_layout(int64_t n_ctr, int64_t n_src) {
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
// SELL fill, dense groups: append row by row (every lane stores its own
// candidate for the row in turn, empty rows skipped) instead of lane by lane
#ifndef TSQBX_ROW_APPEND
#define TSQBX_ROW_APPEND 0
#endif
constexpr bool kRowAppend = TSQBX_ROW_APPEND != 0;
// SELL fill: members staged per lane in shared memory, 16 candidates at a
// time with branch-free stores (a dense 32-candidate group costs ~190
// instructions instead of ~770 for the register shift-register walk), whole
// blocks flushed with 16-byte stores
#ifndef TSQBX_STAGED_APPEND
#define TSQBX_STAGED_APPEND 1
#endif
constexpr bool kStagedAppend = TSQBX_STAGED_APPEND != 0;
constexpr int kStagePos = 20;                 // 3 pending + 16 new + 1 scratch slot
constexpr int kStageWords = kStagePos * 32;
#ifndef TSQBX_STAGE_ABOVE
#define TSQBX_STAGE_ABOVE 12
#endif
constexpr unsigned kStageAbove = TSQBX_STAGE_ABOVE;
// locate and L1-prefetch the next tile's candidates before testing this one
#ifndef TSQBX_SWEEP_PREFETCH
#define TSQBX_SWEEP_PREFETCH 1
#endif
constexpr bool kSweepPrefetch = TSQBX_SWEEP_PREFETCH != 0;

// MODE 0: count members per row; 1: fill the SELL column (plus the row length
// when `cnt` is given); 3: fill the CSR row; 2: bound -- no distance tests, the
// slice width (32 x the largest candidate count of its rows, a multiple of 4)
// into `cnt[slice]`, so the fill can write before the exact lengths are known.
// MODE 4 / 5 (the exact route's count and SELL fill): as 0 / 1, but a warp in
// union mode keeps its member masks -- the count writes one 32-bit word per
// (32-candidate group, lane) to `mask` (word 32 * group + lane: a coalesced
// 128-byte store per group), the fill reads them back instead of staging and
// testing the candidates a second time.  Warps in per-cell mode test twice.
struct SweepIn {
  const double* __restrict__ ctr;      // user order
  const double* __restrict__ rad;
  int64_t n_ctr;
  const int32_t* __restrict__ order;   // processing position -> user center
  const double* __restrict__ prm;
  const double4* __restrict__ sxyz;    // sources in Morton order
  const unsigned long long* __restrict__ hkey;
  const int32_t* __restrict__ hst;
  const int32_t* __restrict__ hen;
  int64_t cap;                         // hash capacity
};

// one warp's staging area
struct SweepSmem {
  // candidate pairs for the packed-fp32 (FFMA2) test: pair p of the tile is
  // tab[p] = {x0, x1, y0, y1}, tcd[p] = {z0, z1, w0, w1}
  float4 tab[kTile / 2], tcd[kTile / 2];
  int32_t tid[kTile];
  int32_t cell_st[kMaxCells], cell_en[kMaxCells];   // the warp's cell list
};

// The sweep of row g (processing order) by one lane of a warp whose 32 lanes
// hold 32 consecutive rows (all lanes must call it).  MODE 1 / 3 store the
// members at dst (1: SELL-32x4 column, entry k at dst[128 (k / 4) + k % 4];
// 3: CSR row, dst[k]) up to row_cap entries (a multiple of 4); k_out is the
// member count (> row_cap: the caller's buffer overflowed).  MODE 0 counts;
// MODE 2 returns in ub_out the warp's bound (the largest candidate count).
// STAGED (SELL fills): `stage` is a per-warp shared-memory buffer of
// kStageWords ints; a lane's members collect there ([position][lane], so a
// lane's accesses never leave its bank) and go out as whole 16-byte blocks.
template <int MODE, bool STAGED = false>
__device__ __forceinline__ void sweep_warp(const SweepIn& in, SweepSmem& sm, int64_t g,
                                           int32_t* dst, int row_cap, int& k_out,
                                           int64_t& ub_out, unsigned* mask = nullptr,
                                           int32_t* stage = nullptr) {
  const double* __restrict__ ctr = in.ctr;
  const double* __restrict__ rad = in.rad;
  const int64_t n_ctr = in.n_ctr;
  const int32_t* __restrict__ order = in.order;
  const double* __restrict__ prm = in.prm;
  const double4* __restrict__ sxyz = in.sxyz;
  const unsigned long long* __restrict__ hkey = in.hkey;
  const int32_t* __restrict__ hst = in.hst;
  const int32_t* __restrict__ hen = in.hen;
  const int64_t cap = in.cap;
  constexpr bool FILL = MODE == 1 || MODE == 3 || MODE == 5;
  constexpr bool SELLF = MODE == 1 || MODE == 5;      // fill of a SELL column
  // staged candidates as fp32 offsets from the warp's reference point (see
  // run_cells) plus their sorted index; the exact fp64 test reads sxyz only for
  // the rare candidates inside the fp32 error band
  const int lane = threadIdx.x & 31;
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
  int k = 0;
  int4 pend = make_int4(0, 0, 0, 0);   // SELL fill with kInt4Stores: the row's open block
  int64_t ub = 0;                      // MODE 2: candidates this row will test
  // Stage the sources of a list of up to kMaxCells cells (ranges [st, en) in
  // cell_st / cell_en of this warp, written by the caller) through the tile;
  // lanes with `mine` test them all.  o: the reference point (a center of this
  // warp); A: a bound on |p - o| (max norm) of every staged source and every
  // testing lane's center.
  // mk: the warp's member masks (MODE 4 writes them, MODE 5 reads them instead of
  // staging coordinates and testing), nullptr = test here.
  auto run_cells = [&](int ncell, bool mine, double ox, double oy, double oz, double A,
                       unsigned* mk) {
    const bool from_mask = MODE == 5 && mk != nullptr;
    const bool mine_all = __all_sync(0xffffffffu, mine);
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
      const int sz = c < ncell ? sm.cell_en[c] - sm.cell_st[c] : 0;
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
    for (int q = 0; q < kMaxCells / 32; ++q) sm.cell_en[lane + 32 * q] = pre[q];
    __syncwarp();
    const int nc = min(ncell, kMaxCells);
    // sorted-source index of candidate t: the last cell with prefix <= t
    auto cand = [&](int t) {
      int lo_c = 0, hi_c = nc - 1;
      while (lo_c < hi_c) {
        const int mid = (lo_c + hi_c + 1) >> 1;
        if (sm.cell_en[mid] <= t) lo_c = mid;
        else hi_c = mid - 1;
      }
      return sm.cell_st[lo_c] + (t - sm.cell_en[lo_c]);
    };
    // the next tile's candidates are located and prefetched into L1 before the
    // current tile is tested, so its staging gathers hit L1 instead of waiting
    // on L2/HBM (TSQBX_SWEEP_PREFETCH)
    int jn[kTile / 32];
#pragma unroll
    for (int r = 0; r < kTile / 32; ++r) jn[r] = lane + 32 * r < min(kTile, total) ? cand(lane + 32 * r) : 0;
    for (int base = 0; base < total; base += kTile) {
      const int fill = min(kTile, total - base);
      int jc[kTile / 32];
#pragma unroll
      for (int r = 0; r < kTile / 32; ++r) jc[r] = jn[r];
#pragma unroll
      for (int r = 0; r < kTile / 32; ++r) {
        const int q = lane + 32 * r;
        if (q < fill && from_mask) {
          sm.tid[q] = jc[r];
        } else if (q < fill) {
          const int j = jc[r];
          const double4 sj = sxyz[j];
          const float x = (float)(sj.x - ox), y = (float)(sj.y - oy), z = (float)(sj.z - oz);
          float* pa = reinterpret_cast<float*>(&sm.tab[q >> 1]) + (q & 1);
          float* pc = reinterpret_cast<float*>(&sm.tcd[q >> 1]) + (q & 1);
          pa[0] = x;
          pa[2] = y;
          pc[0] = z;
          pc[2] = -0.5f * fmaf(z, z, fmaf(y, y, x * x));
          sm.tid[q] = j;
        }
      }
      // MODE 5: this tile's mask words, all loads in flight before the appends
      unsigned mw[kTile / 32];
#pragma unroll
      for (int r = 0; r < kTile / 32; ++r)
        mw[r] = (from_mask && mine && 32 * r < fill) ? mk[(((base >> 5) + r) << 5) + lane] : 0u;
      __syncwarp();
      if (kSweepPrefetch && base + kTile < total) {
        const int nb = base + kTile, nfill = min(kTile, total - nb);
#pragma unroll
        for (int r = 0; r < kTile / 32; ++r) {
          const int q = lane + 32 * r;
          if (q < nfill) {
            jn[r] = cand(nb + q);
            if (!from_mask) asm volatile("prefetch.global.L1 [%0];" ::"l"(sxyz + jn[r]));
          }
        }
      } else if (!kSweepPrefetch && base + kTile < total) {
#pragma unroll
        for (int r = 0; r < kTile / 32; ++r)
          if (lane + 32 * r < min(kTile, total - base - kTile)) jn[r] = cand(base + kTile + lane + 32 * r);
      }
      if (mine) {
        // test 32 staged candidates into a per-lane bit mask, then append only
        // this lane's members (no per-candidate divergent work in the fill)
        for (int t0 = 0; t0 < fill; t0 += 32) {
          const int m = min(32, fill - t0);
          unsigned bits;
          if (from_mask) {
            bits = mw[0];
#pragma unroll
            for (int r = 1; r < kTile / 32; ++r)
              if (t0 == 32 * r) bits = mw[r];
          } else {
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
            const float4 a = sm.tab[(t0 + u) >> 1], c = sm.tcd[(t0 + u) >> 1];
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
          bits = ~below_hi & live;                          // surely inside
          unsigned band = below_hi & ~below_lo & live;      // within tau of the sphere
          while (band) {                     // rare: the exact fp64 test
            const int u = __clz(band);
            band &= ~(0x80000000u >> u);
            if (member(sxyz[sm.tid[t0 + u]], cx, cy, cz, rad2)) bits |= 0x80000000u >> u;
          }
          if (MODE == 4 && mk) mk[((base + t0) & ~31) + lane] = bits;
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
              if (!SELLF || !kInt4Stores || kRowAppend) {
                if (k < row_cap) dst[MODE == 3 ? k : ((k >> 2) << 7) | (k & 3)] = j;
              } else {
                // SELL: the row's current block as a 4-entry shift register,
                // one 16-byte store per completed block
                pend.x = pend.y;
                pend.y = pend.z;
                pend.z = pend.w;
                pend.w = j;
                if ((k & 3) == 3 && k < row_cap)
                  *reinterpret_cast<int4*>(dst + ((k >> 2) << 7)) = pend;
              }
              ++k;
            };
            // (only the lanes testing this list are active here: per-cell mode)
            if (SELLF && STAGED) {
              // the row's pending entries (k & 3 of them) sit at positions
              // 0 .. (k & 3) - 1 of this lane's stage column
              int32_t* const col = stage + lane;
              auto flush_block = [&](int b) {          // stage positions 4b .. 4b + 3 -> row block
                const int blk = (k >> 2) + b;
                int4 v;
                v.x = col[(4 * b) << 5];
                v.y = col[(4 * b + 1) << 5];
                v.z = col[(4 * b + 2) << 5];
                v.w = col[(4 * b + 3) << 5];
                if (4 * blk + 3 < row_cap) *reinterpret_cast<int4*>(dst + (blk << 7)) = v;
              };
              const unsigned am = __activemask();
              if (__reduce_max_sync(am, (unsigned)__popc(bits)) >= kStageAbove) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const unsigned hb = h == 0 ? bits >> 16 : bits & 0xffffu;   // candidate u: bit 15 - u
                  if (!__any_sync(am, hb != 0u)) continue;
                  const int r = k & 3;
                  int32_t* p = col + (r << 5);
                  const int4* tq = reinterpret_cast<const int4*>(&sm.tid[t0 + 16 * h]);
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const int4 j4 = tq[q];
                    // unconditional store, conditional advance: a rejected
                    // candidate is overwritten by the next one
                    *p = j4.x;
                    p += (hb & (0x8000u >> (4 * q))) ? 32 : 0;
                    *p = j4.y;
                    p += (hb & (0x4000u >> (4 * q))) ? 32 : 0;
                    *p = j4.z;
                    p += (hb & (0x2000u >> (4 * q))) ? 32 : 0;
                    *p = j4.w;
                    p += (hb & (0x1000u >> (4 * q))) ? 32 : 0;
                  }
                  const int n = r + __popc(hb);
                  const int nb = n >> 2;
                  const int top = (int)__reduce_max_sync(am, (unsigned)nb);
                  for (int b = 0; b < top; ++b)
                    if (b < nb) flush_block(b);
                  if (nb > 0) {                        // the open block moves to the front
                    const int32_t* tail = col + ((4 * nb) << 5);
                    const int a0 = tail[0], a1 = tail[32], a2 = tail[64];
                    col[0] = a0;
                    col[32] = a1;
                    col[64] = a2;
                  }
                  k = k - r + n;
                }
              } else {
                while (bits) {
                  const int u = __clz(bits);
                  bits &= ~(0x80000000u >> u);
                  col[(k & 3) << 5] = sm.tid[t0 + u];
                  if ((k & 3) == 3) {
                    k -= 3;
                    flush_block(0);
                    k += 3;
                  }
                  ++k;
                }
              }
            } else if (SELLF && kRowAppend && mine_all) {
              // Whole warp testing one list (union mode, 32 valid rows).  A dense
              // group is appended row by row: the row's mask and length are
              // broadcast, lane u stores candidate u (still in its register from
              // the staging) at the row's next free slot plus the rank of bit u;
              // rows without a member in the group are skipped, which is most of
              // them -- a row's members fill a few of the warp's groups.  Sparse
              // groups (few members per lane) keep the per-lane loop.
              const unsigned rows_ne = __ballot_sync(0xffffffffu, bits != 0u);
              const unsigned busiest = __reduce_max_sync(0xffffffffu, (unsigned)__popc(bits));
              if (5u * (unsigned)__popc(rows_ne) < 4u * busiest) {
                int my = jc[0];
#pragma unroll
                for (int r = 1; r < kTile / 32; ++r)
                  if (t0 == 32 * r) my = jc[r];
                int32_t* const slice = dst - 4 * lane;
                unsigned rows = rows_ne;
                while (rows) {
                  const int r = __ffs(rows) - 1;
                  rows &= rows - 1;
                  const unsigned b = __shfl_sync(0xffffffffu, bits, r);
                  const int kr = __shfl_sync(0xffffffffu, k, r);
                  const int kk = kr + __popc((b >> 1) >> (31 - lane));   // members before bit 31 - lane
                  if ((int)(b << lane) < 0 && kk < row_cap)
                    slice[4 * r + (((kk >> 2) << 7) | (kk & 3))] = my;
                }
                k += __popc(bits);
              } else {
                while (bits) {
                  const int u = __clz(bits);
                  bits &= ~(0x80000000u >> u);
                  put(sm.tid[t0 + u]);
                }
              }
            } else if (__reduce_max_sync(__activemask(), (unsigned)__popc(bits)) >= kWalkAbove) {
#pragma unroll 4
              for (int u = 0; u < 32; ++u) {
                const int j = sm.tid[t0 + u];
                if ((int)(bits << u) < 0) put(j);
              }
            } else {
              while (bits) {
                const int u = __clz(bits);      // candidate order: bit 31 - u
                bits &= ~(0x80000000u >> u);
                put(sm.tid[t0 + u]);
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
        sm.cell_st[at] = st;
        sm.cell_en[at] = en;
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
      run_cells(n_ne, valid, ox, oy, oz, A, mask);
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
          sm.cell_st[lane] = st;
          sm.cell_en[lane] = en;
        }
        __syncwarp();
        run_cells(27, valid && ckey == cell, ox, oy, oz, A, nullptr);
      }
    }
  }
  if (SELLF && STAGED) {
    if (valid && (k & 3) && (k | 3) < row_cap) {        // the last, partial block (tail slots unread)
      const int32_t* col = stage + lane;
      *reinterpret_cast<int4*>(dst + ((k >> 2) << 7)) = make_int4(col[0], col[32], col[64], 0);
    }
  } else if (SELLF && kInt4Stores && !kRowAppend && valid && (k & 3) && k < row_cap) {   // the last, partial block
    const int r = k & 3;                                // entries pending in pend's tail
    int4 blk = pend;
    if (r == 1) blk.x = pend.w;
    if (r == 2) { blk.x = pend.z; blk.y = pend.w; }
    if (r == 3) { blk.x = pend.y; blk.y = pend.z; blk.z = pend.w; }
    *reinterpret_cast<int4*>(dst + ((k >> 2) << 7)) = blk;
  }
  if (MODE == 2)
    for (int off = 16; off > 0; off >>= 1) ub = max(ub, __shfl_xor_sync(0xffffffffu, ub, off));
  k_out = k;
  ub_out = ub;
}

}  // namespace nsw
}  // namespace tsqbx
