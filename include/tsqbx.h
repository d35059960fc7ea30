/*
 * include/tsqbx.h -- C ABI of the B200-native TSQBX near-field evaluator.
 *
 * Drop-in boundary for the reference's backend plugin protocol
 * (/root/reference/pkg/src/gigaqbx/_backend/__init__.py:7-41): every backend
 * module exposes
 *     ts_accum_laplace(variant, p, sources, weights, snormals, center, target, tnormal)
 *         -- _core.pyx:205-207, _backend/_ref.py:177, _backend/compiled.py:65-69
 *     ts_accum_helmholtz(variant, k, p, sources, weights, snormals, center, target, tnormal)
 *         -- _core.pyx:310-312, _backend/_ref.py:278, _backend/compiled.py:72-76
 * for ONE (center, target) over a batch of sources.  This ABI is the batched
 * form of the same call: many centers, each with a CSR row of near sources and
 * a contiguous run of targets.  A call with n_ctr = 1 and n_tgt = 1 is exactly
 * the reference function.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers, caller-owned; no hidden allocation.
 *     Scratch is passed in as `workspace` (size from the *_workspace_bytes query).
 *   - Complex numbers are interleaved (re, im) doubles (numpy complex128 layout).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All calls are
 *     stream-ordered and asynchronous unless stated otherwise.
 *   - Return value: TSQBX_OK or an error code; tsqbx_last_error() has the text.
 *   - Variant codes follow _backend/common.py:27-29 (0 = S, 1 = S', 2 = D);
 *     equations: 0 = Laplace, 1 = Helmholtz (kernels.py:26-28).
 *   - Validation (flag TSQBX_FLAG_VALIDATE) mirrors tsqbx._prep (tsqbx.py:38-53):
 *     a flagged problem leaves *err_key != INT64_MAX; tsqbx_validate() then
 *     locates the first offending (target, list position) exactly.
 */
#ifndef GIGAQBX_B200_TSQBX_H
#define GIGAQBX_B200_TSQBX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSQBX_ABI_VERSION 12

#define TSQBX_OK 0
#define TSQBX_ERR_SEPARATION 1   /* tsqbx.py:48-53  "separation violation for source i" */
#define TSQBX_ERR_COINCIDENT 2   /* tsqbx.py:44-47  "source i coincides with the expansion center" */
#define TSQBX_ERR_ARGUMENT 3
#define TSQBX_ERR_CUDA 4

#define TSQBX_EQ_LAPLACE 0
#define TSQBX_EQ_HELMHOLTZ 1

#define TSQBX_VARIANT_S 0
#define TSQBX_VARIANT_SPRIME 1
#define TSQBX_VARIANT_D 2

#define TSQBX_FLAG_VALIDATE 1u   /* cheap in-kernel screening, see tsqbx_validate */
#define TSQBX_FLAG_GENERIC 2u    /* force the runtime-p reference-order kernel */
#define TSQBX_FLAG_REAL_WEIGHTS 4u /* caller guarantees Im w == 0: skip the imaginary part */
#define TSQBX_FLAG_ONE_TARGET 8u   /* fast kernels: one target per pass (fewer registers) */
#define TSQBX_FLAG_PRECISE 16u     /* p2p: IEEE 1/sqrt (after a non-finite screen with no singular pair) */
/* eval: every row g owns targets [k g, k g + k) (tgt_ptr[g] == k g), k = (flags >> 8) & 0xff;
 * the SELL kernels then address a row's targets without loading tgt_ptr */
#define TSQBX_FLAG_UNIFORM_TARGETS 32u
/* Helmholtz: the caller guarantees k |s - c| <= pi/4 (NARROW) or <= pi/2 (WIDE)
 * for every near source of every row (e.g. k x the largest near radius):
 * the kernels then take one sin/cos series for every lane without a warp
 * vote.  Without either flag each warp picks the series its lanes need. */
#define TSQBX_FLAG_KR_NARROW 64u
#define TSQBX_FLAG_KR_WIDE 128u
/* a performance hint: the near lists are long (mean >~ 48 entries), pick the
 * kernel builds tuned for long rows (never changes results) */
#define TSQBX_FLAG_LONG_ROWS (1u << 16)
/* Laplace S with uniform target runs of 1 or 2 (TSQBX_FLAG_UNIFORM_TARGETS)
 * and the CSR entries (near_idx) given: evaluate with the short-list kernel
 * (a warp's 32 rows' entries split evenly over its lanes) instead of the
 * SELL thread-per-row kernel -- for near lists of a few dozen sources. */
#define TSQBX_FLAG_FLAT (1u << 17)
/* Laplace S on the SELL layout with uniform target runs and unsplit rows:
 * two rows per thread, the second row's loads in flight while the first
 * computes (short near lists: fewer waves of dependent-load chains). */
#define TSQBX_FLAG_TWO_ROWS (1u << 18)
/* Laplace S on a windowed SELL layout (tsqbx_sell_window; set by
 * tsqbx_eval_packed_win, rejected by tsqbx_eval_packed). */
#define TSQBX_FLAG_WINDOW (1u << 19)

#define TSQBX_MAX_ORDER 64

/* err_key encoding (int64, device scalar; INT64_MAX = no problem):
 *   (target << 32) | (kind << 31) | list_position,  kind 0 = coincident, 1 = separation.
 * After tsqbx_eval with TSQBX_FLAG_VALIDATE the key is only a screen
 * (TSQBX_ERR_KEY_SUSPECT); tsqbx_validate produces the exact key. */
#define TSQBX_ERR_KEY_NONE INT64_MAX
#define TSQBX_ERR_KEY_SUSPECT (INT64_MAX - 1)

int tsqbx_abi_version(void);
const char* tsqbx_last_error(void);
/* number of SMs and compute capability of the current device (host query) */
int tsqbx_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------------------
 * Source packing.  The evaluator reads sources in a packed, 32-byte aligned
 * layout: double4 {x, y, z, Re w} per source, then Im w per source, then (with
 * normals) double4 {nx, ny, nz, 0}, then 4 doubles of metadata (a device flag:
 * some Im w != 0, which lets the Laplace kernels skip the imaginary part).
 * packed[i] = source perm[i] (perm may be NULL).
 * ------------------------------------------------------------------------- */
int64_t tsqbx_packed_doubles(int64_t n_src, int with_normals);
int tsqbx_pack_sources(int64_t n_src, const double* xyz, const double* w, const double* nrm,
                       const int32_t* perm, double* packed, void* stream);

/* ---------------------------------------------------------------------------
 * Evaluation.  Every per-center array is in PROCESSING order (row g):
 *   packed      : tsqbx_pack_sources output (n_src sources)
 *   ctr_xyz     : n_ctr x 3 centers, row g
 *   near_ptr    : n_ctr + 1 row offsets into near_idx
 *   near_idx    : source indices into `packed`
 *   sell_ptr/idx: optional sliced-ELL copy of the same lists (tsqbx_sell_build);
 *                 when given, the thread-per-center kernels run on it (row ranges
 *                 must then start at a multiple of 32)
 *   tgt_xyz     : n_tgt x 3 targets grouped by row: the targets of row g are
 *                 tgt_ptr[g] .. tgt_ptr[g+1]-1
 *   tgt_nrm     : n_tgt x 3 (S' only, else NULL)
 *   tgt_out     : output slot of each target (NULL = identity); the value of
 *                 target t is written to out[(tgt_out ? tgt_out[t] : t) - out_offset]
 *   tgt_base    : with TSQBX_FLAG_UNIFORM_TARGETS (k = flags >> 8 & 255), row g
 *                 of the launch owns targets tgt_base + k g .. tgt_base + k g + k - 1
 *                 (no tgt_ptr load; a row range [g0, g1) passes k * g0); the
 *                 kernels that do not use the uniform form read tgt_ptr, so
 *                 tgt_ptr must hold the same runs; n_tgt >= tgt_base + k n_ctr
 *   out         : complex128 potentials
 *   err_key     : device int64 (see above); may be NULL when flags lacks VALIDATE
 *   group_lanes : CSR kernels: lanes per center (power of two <= 32, 0 = 8);
 *                 SELL layout (Laplace S): threads per row, 1, 2 or 4 (a row
 *                 split over lanes 32/S apart of one warp; 0 = 1)
 * A user CSR (rows by user center) is already in processing order (identity);
 * tsqbx_order_targets produces these arrays for a Morton order from
 * tsqbx_near_count.  A contiguous row range [g0, g1) of a problem is evaluated
 * by offsetting ctr_xyz / near_ptr / tgt_ptr by g0 (how ranks shard it).
 * ------------------------------------------------------------------------- */
int64_t tsqbx_eval_workspace_bytes(int equation, int variant, int p, int64_t n_tgt);
int tsqbx_eval_packed(int equation, int variant, double k, int p,
                      const double* packed, int64_t n_src, int with_normals,
                      const double* ctr_xyz, int64_t n_ctr,
                      const int64_t* near_ptr, const int32_t* near_idx,
                      const int64_t* sell_ptr, const int32_t* sell_idx,
                      const double* tgt_xyz, const double* tgt_nrm, const int64_t* tgt_ptr,
                      int64_t n_tgt, const int64_t* tgt_out, int64_t out_offset,
                      int64_t tgt_base, unsigned flags, int group_lanes, void* workspace,
                      int64_t ws_bytes, double* out, int64_t* err_key, void* stream);

/* Convenience forms with the reference's names: raw user-layout sources
 * (xyz n x 3, complex weights, optional normals), user-order CSR.  They pack
 * into `workspace` (size: tsqbx_user_workspace_bytes) and call tsqbx_eval_packed. */
int64_t tsqbx_user_workspace_bytes(int equation, int variant, int p, int64_t n_src,
                                   int64_t n_tgt);
int tsqbx_eval_laplace(int variant, int p,
                       const double* src_xyz, const double* src_w, const double* src_nrm,
                       int64_t n_src, const double* ctr_xyz, int64_t n_ctr,
                       const int64_t* near_ptr, const int32_t* near_idx,
                       const double* tgt_xyz, const double* tgt_nrm, const int64_t* tgt_ptr,
                       int64_t n_tgt, unsigned flags, void* workspace, int64_t ws_bytes,
                       double* out, int64_t* err_key, void* stream);
int tsqbx_eval_helmholtz(int variant, double k, int p,
                         const double* src_xyz, const double* src_w, const double* src_nrm,
                         int64_t n_src, const double* ctr_xyz, int64_t n_ctr,
                         const int64_t* near_ptr, const int32_t* near_idx,
                         const double* tgt_xyz, const double* tgt_nrm, const int64_t* tgt_ptr,
                         int64_t n_tgt, unsigned flags, void* workspace, int64_t ws_bytes,
                         double* out, int64_t* err_key, void* stream);

/* Exact validation in the reference's arithmetic (tsqbx.py:43-53): for every
 * (target, list position) computes R = |s - c|, r = |t - c| and writes into
 * *err_key the smallest key of a coincident (R == 0) or separated
 * (R * (1 + 1e-12) < r) pair; coincidence outranks separation within a target. */
int tsqbx_validate(const double* packed, int64_t n_src,
                   const double* ctr_xyz, int64_t n_ctr,
                   const int64_t* near_ptr, const int32_t* near_idx,
                   const double* tgt_xyz, const int64_t* tgt_ptr, int64_t n_tgt,
                   int64_t* err_key, void* stream);

/* ---------------------------------------------------------------------------
 * Radius-ball near lists on the device (no reference function: the reference
 * builds tree lists, driver.py:197-228 / ilists.py:93-218; BASELINE.json
 * defines radius balls).  member(s, c) iff ((dx*dx + dy*dy) + dz*dz) <= rad*rad
 * in round-to-nearest without contraction.
 *
 * Two phases sharing one caller-owned workspace.  Row order: processing
 * (Morton) order of the centers; entries in the order of the 27 neighbour
 * cells (dx, dy, dz), ascending within a cell.
 *
 * CSR mode (sell_ptr == NULL in count):
 *   tsqbx_near_count: Morton-sorts sources and centers, counts the members of
 *       every row exactly; writes src_perm (sorted position -> user source),
 *       ctr_order (processing position -> user center), near_ptr (n_ctr + 1)
 *       and totals[0] = n_pairs.
 *   tsqbx_near_fill : writes near_idx (indices into the sorted source order).
 * SELL mode (sell_ptr given to count, sell_idx to fill, near_idx NULL):
 *   tsqbx_near_count: as above, but instead of counting it bounds every row by
 *       its candidate count (no distance tests) and writes sell_ptr (SELL-32x4
 *       slice offsets, ceil(n_ctr/32) + 1 entries) and totals[1] = SELL slots
 *       (totals[0] = -1): one read-back sizes sell_idx.
 *   tsqbx_near_fill : writes every row straight into its slice (slots past a
 *       row's length are never read), then near_ptr and totals[0] = n_pairs.
 *       The CSR entries, when needed, come from tsqbx_sell_to_csr.
 * totals is a device int64[2].  tsqbx_near_count synchronises `stream` once,
 * after the bounding box, to radix-sort only the Morton key bits in use; the
 * rest of both phases is stream-ordered.
 * ------------------------------------------------------------------------- */
int64_t tsqbx_near_workspace_bytes(int64_t n_ctr, int64_t n_src);
int tsqbx_near_count(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                     const double* src_xyz, int64_t n_src,
                     void* workspace, int64_t ws_bytes,
                     int32_t* src_perm, int32_t* ctr_order, int64_t* near_ptr,
                     int64_t* sell_ptr, int64_t* totals, void* stream);
int tsqbx_near_fill(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                    const double* src_xyz, int64_t n_src,
                    void* workspace, int64_t ws_bytes,
                    const int32_t* ctr_order, int64_t* near_ptr, int32_t* near_idx,
                    const int64_t* sell_ptr, int32_t* sell_idx, int64_t* totals,
                    void* stream);
/* After a SELL-mode tsqbx_near_count (same workspace, no call in between but
 * tsqbx_sell_size): count every row exactly, reusing its sorts and cell hash,
 * into near_ptr (n_ctr + 1) and totals[0] = n_pairs -- the exact-size route
 * when the bound-sized SELL buffer would be too large.  No synchronisation. */
int tsqbx_near_recount(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                       int64_t n_src, void* workspace, int64_t ws_bytes,
                       const int32_t* ctr_order, int64_t* near_ptr, int64_t* totals,
                       void* stream);
/* The exact route with the member masks kept between its two sweeps: the
 * count writes one 32-bit word per (32-candidate group, center) into mask_ws
 * (tsqbx_near_mask_bytes(n_ctr, totals[1] of the SELL-mode tsqbx_near_count)
 * bytes, caller-owned), the SELL fill reads them back instead of staging and
 * testing every candidate a second time.  Same results, same call order as
 * tsqbx_near_recount / tsqbx_near_fill (sell_ptr from tsqbx_sell_size). */
int64_t tsqbx_near_mask_bytes(int64_t n_ctr, int64_t n_sell_bound);
int tsqbx_near_recount_masks(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                             int64_t n_src, void* workspace, int64_t ws_bytes,
                             const int32_t* ctr_order, int64_t* near_ptr, int64_t* totals,
                             void* mask_ws, int64_t mask_bytes, void* stream);
int tsqbx_near_fill_masks(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                          int64_t n_src, void* workspace, int64_t ws_bytes,
                          const int32_t* ctr_order, int64_t* near_ptr, const int64_t* sell_ptr,
                          int32_t* sell_idx, int64_t* totals, const void* mask_ws,
                          int64_t mask_bytes, void* stream);
/* The bounding box, Morton sorts (src_perm, ctr_order) and cell hash of
 * tsqbx_near_count without any sweep: the state tsqbx_eval_fused reads. */
int tsqbx_near_index(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                     const double* src_xyz, int64_t n_src, void* workspace, int64_t ws_bytes,
                     int32_t* src_perm, int32_t* ctr_order, void* stream);
/* One-shot near field (Laplace / Helmholtz S, compile-time p <= 16, uniform
 * target runs of 1 or 2 per center): every warp sweeps the near lists of 32
 * consecutive rows into a per-warp scratch slice and evaluates them at once;
 * no CSR is materialised.  After tsqbx_near_index on (ctr_user, radius,
 * sources) with `near_ws`; packed = tsqbx_pack_sources with src_perm;
 * ctr_proc / tgt_proc / tgt_out from tsqbx_order_targets.  flags:
 * TSQBX_FLAG_UNIFORM_TARGETS (| k << 8) required, VALIDATE / REAL_WEIGHTS /
 * KR_* as for tsqbx_eval_packed.  err: device int64[2] -- err[0] the
 * validation key, err[1] != 0 when a row had more than row_cap near sources
 * (the caller evaluates through tsqbx_near_count/fill + tsqbx_eval_packed
 * instead).  scratch: tsqbx_fused_scratch_bytes(equation, p, k, validate,
 * row_cap) bytes (sized by the resident CTAs of the current device). */
int64_t tsqbx_fused_scratch_bytes(int equation, int p, int targets_per_center, int validate,
                                  int row_cap);
int tsqbx_eval_fused(int equation, double k, int p, const double* packed, int64_t n_src,
                     const double* ctr_user, const double* radius, const int32_t* ctr_order,
                     void* near_ws, int64_t near_ws_bytes, const double* ctr_proc, int64_t n_ctr,
                     const double* tgt_proc, int64_t n_tgt, const int64_t* tgt_out,
                     unsigned flags, int row_cap, void* scratch, int64_t scratch_bytes,
                     double* out, int64_t* err, void* stream);
/* Rows g0..g1-1 of the processing order only (a rank's shard),
 * SELL mode: after tsqbx_near_count over ALL centers (CSR mode: exact row
 * lengths), the caller sizes the shard's slices from near_ptr[g0..g1] (e.g.
 * tsqbx_sell_size on the rebased offsets) and this call writes the shard's
 * rows into them, its exact offsets into near_ptr (g1 - g0 + 1 entries, from
 * 0) and its pair count into totals[0].  g0 must be a multiple of 32. */
int tsqbx_near_fill_rows(const double* ctr_xyz, const double* radius, int64_t n_ctr,
                         const double* src_xyz, int64_t n_src,
                         void* workspace, int64_t ws_bytes,
                         const int32_t* ctr_order, int64_t g0, int64_t g1, int64_t* near_ptr,
                         const int64_t* sell_ptr, int32_t* sell_idx, int64_t* totals,
                         void* stream);

/* Reorder centers and their targets into the processing order `ctr_order`
 * (user center ctr_order[g] becomes row g): writes ctr_out (n_ctr x 3),
 * tptr_out (n_ctr + 1), tgt_out / tnrm_out (n_tgt x 3; tnrm only if tgt_nrm)
 * and tgt_index (processing target -> user target; pass it as tgt_out of the
 * evaluation to write potentials in user order).  `bad` (device int64,
 * nullable) is set to 1 when tgt_ptr is malformed (tgt_ptr[0] != 0, a
 * decreasing entry, an entry past n_tgt, or tgt_ptr[n_ctr] != n_tgt), else 0;
 * malformed rows get no targets and tptr_out stays within [0, n_tgt], so a
 * later evaluation never leaves the target arrays (the caller reports *bad). */
int64_t tsqbx_order_workspace_bytes(int64_t n_ctr);
int tsqbx_order_targets(int64_t n_ctr, const int32_t* ctr_order, const double* ctr_xyz,
                        const int64_t* tgt_ptr, const double* tgt_xyz, const double* tgt_nrm,
                        int64_t n_tgt, void* workspace, int64_t ws_bytes,
                        double* ctr_out, int64_t* tptr_out, double* tgt_out, double* tnrm_out,
                        int64_t* tgt_index, int64_t* bad, void* stream);

/* Sliced-ELL (SELL-32x4) copy of a CSR: rows in slices of 32; a slice's width
 * is its longest row rounded up to 4, and entry (row r, column i) sits at
 * sell_ptr[r/32] + (i/4)*128 + (r%32)*4 + i%4 -- column blocks of 4 so that a
 * lane fetches 4 upcoming indices with one 16-byte load and a warp one 512-byte
 * run.  sell_ptr has ceil(n_rows/32) + 1 offsets (multiples of 128),
 * *n_entries (device) the total.
 * Two phases like the near lists: tsqbx_sell_size then tsqbx_sell_fill. */
int64_t tsqbx_sell_workspace_bytes(int64_t n_rows);
int tsqbx_sell_size(int64_t n_rows, const int64_t* near_ptr, void* workspace, int64_t ws_bytes,
                    int64_t* sell_ptr, int64_t* n_entries, void* stream);
int tsqbx_sell_fill(int64_t n_rows, const int64_t* near_ptr, const int32_t* near_idx,
                    const int64_t* sell_ptr, int32_t* sell_idx, void* stream);

/* tsqbx_eval_packed on a windowed SELL layout (TSQBX_FLAG_WINDOW implied):
 * sell_loc / win_src / win_len from tsqbx_sell_window, near_idx the plain CSR
 * entries (validation only).  Laplace S, p <= 16, uniform target runs,
 * group_lanes 1. */
int tsqbx_eval_packed_win(int equation, int variant, double k, int p, const double* packed,
                          int64_t n_src, int with_normals, const double* ctr_xyz, int64_t n_ctr,
                          const int64_t* near_ptr, const int32_t* near_idx,
                          const int64_t* sell_ptr, const int32_t* sell_loc,
                          const int32_t* win_src, const int32_t* win_len, const double* tgt_xyz,
                          const double* tgt_nrm, const int64_t* tgt_ptr, int64_t n_tgt,
                          const int64_t* tgt_out, int64_t out_offset, int64_t tgt_base,
                          unsigned flags, int group_lanes, void* workspace, int64_t ws_bytes,
                          double* out, int64_t* err_key, void* stream);
/* Windowed SELL for short near lists: for every 32-row slice its distinct
 * sources (at most TSQBX_WINDOW, win_src[s * TSQBX_WINDOW + i], count
 * win_len[s]) and loc_idx = the SELL entries as indices into that window
 * (same positions as sell_idx).  A slice with more distinct sources than
 * TSQBX_WINDOW keeps its global indices in loc_idx, gets win_len = -1 and is
 * counted in *overflow (device unsigned).  Evaluated with
 * TSQBX_FLAG_WINDOW: a warp stages its slice's window in shared memory once
 * and its rows read their sources from there. */
#define TSQBX_WINDOW 128
int tsqbx_sell_window(int64_t n_rows, const int64_t* near_ptr, const int64_t* sell_ptr,
                      const int32_t* sell_idx, int32_t* loc_idx, int32_t* win_src,
                      int32_t* win_len, unsigned* overflow, void* stream);

/* CSR entries (near_idx, rows by near_ptr) from a SELL-32x4 copy. */
/* Copy a SELL-32x4 layout into one with narrower slices (every slice of the
 * destination no wider than the source's; e.g. the bound-sized build output into
 * the exact widths of tsqbx_sell_size): a warp per slice copies its first
 * (sell_ptr_dst[s+1] - sell_ptr_dst[s]) entries. */
int tsqbx_sell_compact(int64_t n_rows, const int64_t* sell_ptr_src, const int32_t* sell_idx_src,
                       const int64_t* sell_ptr_dst, int32_t* sell_idx_dst, void* stream);
int tsqbx_sell_to_csr(int64_t n_rows, const int64_t* near_ptr, const int64_t* sell_ptr,
                      const int32_t* sell_idx, int32_t* near_idx, void* stream);

/* out[dest[i]] = src[i] for n complex128 values (dest NULL = copy); assembles
 * all-gathered shards into user target order. */
int tsqbx_scatter_c128(int64_t n, const int64_t* dest, const double* src, double* out,
                       void* stream);

/* ---------------------------------------------------------------------------
 * Single call: one (center, target) over a source batch -- the reference's
 * per-call protocol (_core.ts_accum_laplace / ts_accum_helmholtz,
 * _core.pyx:205-207, :310-312, and tsqbx.ts_accumulate, tsqbx.py:68-80): one
 * launch and a stream synchronisation; small batches (<= 256 KB staged) are
 * read from / written to the pinned host buffers in place, larger ones take one
 * H2D and one D2H copy through device_buf.
 * staged_host (pinned) holds tsqbx_one_staging_doubles(n, variant == D) doubles:
 *   [center(3) target(3) target_normal(3) |t-c| 0 x 6]   (|t-c| as the caller's
 *                                                       validation computed it)
 *   [x y z Re(w)] x n  [Im(w)] x n  [0 pad to a multiple of 4]  ([nx ny nz 0] x n for D)
 * device_buf holds at least that + 4 doubles.  result_host (pinned) receives
 * {Re, Im, err_key}: the reference's value and, with TSQBX_FLAG_VALIDATE, the
 * exact _prep key ((kind << 31) | position, kind 0 = coincident, 1 =
 * separation; TSQBX_ERR_KEY_NONE when valid), stored as int64 bits.
 * ------------------------------------------------------------------------- */
int64_t tsqbx_one_staging_doubles(int64_t n_src, int with_normals);
int tsqbx_eval_one(int equation, int variant, double k, int p, const double* staged_host,
                   int64_t n_src, unsigned flags, double* device_buf, int64_t device_doubles,
                   double* result_host, void* stream);

/* ---------------------------------------------------------------------------
 * Point-to-point direct interactions: replaces the
 * reference backends' laplace_p2p / helmholtz_p2p (_core.pyx:94-165), called by
 * kernels.direct_sum (kernels.py:114-136) and per target box by
 * driver.direct_stage (driver.py:187-210).
 *
 *   out[t] = sum_j w_j K(t, s_j),  K = 1/(4 pi r) | e^{ikr}/(4 pi r) (S),
 *            its target-normal (S') or source-normal (D) derivative.
 *
 * Dense (row_ptr NULL): every target sees every source.  Rows: row r's
 * targets [row_tgt[r], row_tgt[r+1]) (rows partition [0, n_tgt) in order) see
 * the packed sources row_idx[row_ptr[r] .. row_ptr[r+1]).
 * With TSQBX_FLAG_VALIDATE a non-finite result sets *err_key to
 * TSQBX_ERR_KEY_SUSPECT; tsqbx_p2p_find_singular then sets the exact key
 * (target << 32) | source of the first target-major pair with r2 == 0 (the
 * reference's "singular source/target pair: target i, source j"), or leaves
 * TSQBX_ERR_KEY_NONE, in which case the caller re-runs with TSQBX_FLAG_PRECISE.
 * ------------------------------------------------------------------------- */
int64_t tsqbx_p2p_workspace_bytes(int64_t n_src, int64_t n_tgt, int64_t n_rows, int dense);
int tsqbx_p2p_packed(int equation, int variant, double k, const double* packed, int64_t n_src,
                     int with_normals, int64_t n_rows, const int64_t* row_tgt,
                     const int64_t* row_ptr, const int32_t* row_idx, const double* tgt_xyz,
                     const double* tgt_nrm, int64_t n_tgt, unsigned flags, void* workspace,
                     int64_t ws_bytes, double* out, int64_t* err_key, void* stream);
int tsqbx_p2p_find_singular(const double* packed, int64_t n_src, int64_t n_rows,
                            const int64_t* row_tgt, const int64_t* row_ptr,
                            const int32_t* row_idx, const double* tgt_xyz, int64_t n_tgt,
                            int64_t* err_key, void* stream);
/* user layout (dense direct sum): sources xyz (n,3), weights complex128 (n,)
 * interleaved, normals (n,3) for D / (m,3) for S'; the workspace holds the
 * packed sources plus the chunk partial sums. */
int64_t tsqbx_p2p_user_workspace_bytes(int variant, int64_t n_src, int64_t n_tgt);
int tsqbx_p2p_laplace(int variant, const double* src_xyz, const double* src_w,
                      const double* src_nrm, int64_t n_src, const double* tgt_xyz,
                      const double* tgt_nrm, int64_t n_tgt, unsigned flags, void* workspace,
                      int64_t ws_bytes, double* out, int64_t* err_key, void* stream);
int tsqbx_p2p_helmholtz(int variant, double k, const double* src_xyz, const double* src_w,
                        const double* src_nrm, int64_t n_src, const double* tgt_xyz,
                        const double* tgt_nrm, int64_t n_tgt, unsigned flags, void* workspace,
                        int64_t ws_bytes, double* out, int64_t* err_key, void* stream);

/* ---------------------------------------------------------------------------
 * Box interaction lists -> row index lists: the gather of
 * driver.direct_stage (driver.py:197-217, _gather_sources :109-113) for all
 * target boxes at once.  Row r belongs to box row_box[r] (< 0: empty row); its
 * sources are the owned source ranges [box_start[d*stride], box_end[d*stride])
 * of the boxes d = lst_box[lst_ptr[b] .. lst_ptr[b+1]) concatenated in list
 * order (pass owned_start[:, SOURCES] with stride 3 for the reference Octree).
 * count: row_ptr (n_rows + 1) and *total (device scalar); fill: row_idx.
 * ------------------------------------------------------------------------- */
int64_t tsqbx_box_rows_workspace_bytes(int64_t n_rows);
int tsqbx_box_rows_count(int64_t n_rows, const int64_t* row_box, const int64_t* lst_ptr,
                         const int64_t* lst_box, const int64_t* box_start,
                         const int64_t* box_end, int64_t box_stride, void* workspace,
                         int64_t ws_bytes, int64_t* row_ptr, int64_t* total, void* stream);
int tsqbx_box_rows_fill(int64_t n_rows, const int64_t* row_box, const int64_t* lst_ptr,
                        const int64_t* lst_box, const int64_t* box_start, const int64_t* box_end,
                        int64_t box_stride, const int64_t* row_ptr, int32_t* row_idx,
                        void* stream);

/* ---------------------------------------------------------------------------
 * FP64 roofline probe: every thread runs 8 independent DFMA chains of `iters`
 * steps (16 * iters flops per thread); used by bench.py to measure the FP64
 * peak of the box (MEASURED_PEAKS.json has none).  out needs blocks*threads
 * doubles.
 * ------------------------------------------------------------------------- */
int tsqbx_fp64_probe(double* out, int64_t iters, int blocks, int threads, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU helper: after each rank evaluated its contiguous block of targets,
 * one NCCL all-gather assembles every target's potential on every rank
 * (implemented in Python over torch.distributed/NCCL; see
 * paper_1811_01110_b200/distributed.py).  Nothing to export here.
 * ------------------------------------------------------------------------- */

#ifdef __cplusplus
}
#endif
#endif
