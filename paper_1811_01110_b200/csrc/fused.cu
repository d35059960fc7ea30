// fused.cu -- one-shot near field: the near-list sweep and the TSQBX S
// evaluation in one kernel, the lists never written to HBM as a CSR.
//
// The one-shot path (near_field_potentials: geometry -> potentials) otherwise
// builds the lists (count or bound pass, fill, compaction: C5 dense 17 ms,
// 6.8 GB of indices written and read back) and then evaluates them.  Here a
// warp takes 32 consecutive rows (processing order), runs the builder's sweep
// (near_sweep.cuh: union region, FFMA2 membership test) writing its members
// into a per-warp scratch slice in the SELL-32x4 layout, and evaluates the
// same 32 rows from it right away with the stand-alone kernels' row bodies
// (eval_bodies.cuh).  The scratch slice belongs to a resident CTA slot of the
// SM (claimed at CTA start, released at exit), so the scratch is sized by the
// resident warps, not by the problem: ~100 MB that stays mostly in L2.  While
// some warps of an SM sweep (FP32 / integer pipes) others evaluate (FP64
// pipe).  A row longer than the slice capacity (row_cap) sets err[1]; the
// caller then takes the two-step path.
//
// Reference: _core.pyx:205-307 (Laplace S) and :310-398 (Helmholtz S) for the
// per-pair sums; the membership of the device near-list builder (near.cu).
#include "eval_bodies.cuh"
#include "near_sweep.cuh"

namespace tsqbx {
namespace {

constexpr int kFusedBlock = kSellBlock;   // 8 warps = 8 slices of 32 rows

struct FusedArgs {
  nsw::SweepIn in;
  int32_t* scratch;          // [slots][8 warps][32 rows x row_cap] ints, SELL-32x4 per warp
  unsigned* lock;            // [n_smid][slots_per_sm]: 1 = slot in use
  int slots_per_sm;
  int row_cap;               // entries per row a slice holds (multiple of 4)
  unsigned long long* overflow;
};

template <int EQ, int P, int NT, bool VAL>
__global__ void __launch_bounds__(kFusedBlock, EQ == TSQBX_EQ_LAPLACE ? 3 : 2)
    fused_kernel(const EvalParams a, const FusedArgs f) {
  __shared__ nsw::SweepSmem sm[kFusedBlock / 32];
  __shared__ int4 ring[kSlots * kSellBlock];
  __shared__ int slot_s;
  if (threadIdx.x == 0) {
    // a free scratch slot of this SM (at most slots_per_sm CTAs are resident)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned* mine = f.lock + (size_t)smid * f.slots_per_sm;
    int s = -1;
    while (s < 0)
      for (int i = 0; i < f.slots_per_sm && s < 0; ++i)
        if (atomicCAS(mine + i, 0u, 1u) == 0u) s = (int)(smid * f.slots_per_sm + i);
    slot_s = s;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kFusedBlock + threadIdx.x;
  const int64_t g_warp = g - lane;
  const int64_t soff = ((int64_t)slot_s * (kFusedBlock / 32) + w) * 32 * f.row_cap;
  if (g_warp < a.n_ctr) {
    int k = 0;
    int64_t ub = 0;
    nsw::sweep_warp<1>(f.in, sm[w], g, g < a.n_ctr ? f.scratch + soff + 4 * lane : nullptr,
                       f.row_cap, k, ub);
    if (k > f.row_cap) atomicOr(f.overflow, 1ull);
    __syncwarp();
    __threadfence_block();      // the lane's scratch stores before its cp.async reads
    if (g < a.n_ctr) {
      const int len = min(k, f.row_cap);
      if (EQ == TSQBX_EQ_LAPLACE) {
        RowHead h;
        h.soff = soff;
        h.len = len;
        h.t0 = a.tbase + g * NT;
        h.t1 = h.t0 + NT;
        h.cx = a.ctr[3 * g];
        h.cy = a.ctr[3 * g + 1];
        h.cz = a.ctr[3 * g + 2];
        const bool realw = a.real_w || *a.imag_flag == 0u;
        if (realw) laplace_sell_body<P, NT, VAL, true, 1>(a, g, h, ring);
        else laplace_sell_body<P, NT, VAL, false, 1>(a, g, h, ring);
      } else {
        helmholtz_sell_row<P, NT, VAL, NT, 1>(a, g, soff, len, nullptr, ring);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(f.lock + slot_s, 0u);
  }
}

template <int P>
struct FusedLaunch {
  template <int EQ, int NT, bool VAL>
  static const void* fn() {
    return reinterpret_cast<const void*>(&fused_kernel<EQ, P, NT, VAL>);
  }
  static const void* pick(int eq, int nt, bool val) {
    if (eq == TSQBX_EQ_LAPLACE) {
      if (nt >= 2) return val ? fn<TSQBX_EQ_LAPLACE, 2, true>() : fn<TSQBX_EQ_LAPLACE, 2, false>();
      return val ? fn<TSQBX_EQ_LAPLACE, 1, true>() : fn<TSQBX_EQ_LAPLACE, 1, false>();
    }
    if (nt >= 2) return val ? fn<TSQBX_EQ_HELMHOLTZ, 2, true>() : fn<TSQBX_EQ_HELMHOLTZ, 2, false>();
    return val ? fn<TSQBX_EQ_HELMHOLTZ, 1, true>() : fn<TSQBX_EQ_HELMHOLTZ, 1, false>();
  }
  static void go(int eq, int nt, bool val, const void** out) { *out = pick(eq, nt, val); }
};

template <template <int> class F, int... Ps>
struct FusedOrders {
  template <class... Args>
  static bool run(int p, Args&&... args) {
    bool done = false;
    ((p == Ps ? (F<Ps>::go(args...), done = true) : false), ...);
    return done;
  }
};

const void* fused_fn(int eq, int p, int nt, bool val) {
  const void* fn = nullptr;
  FusedOrders<FusedLaunch, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>::run(
      p, eq, nt, val, &fn);
  return fn;
}

__global__ void fused_err_init(int64_t* err) {
  err[0] = TSQBX_ERR_KEY_NONE;
  err[1] = 0;
}

__global__ void nsmid_kernel(unsigned* out) {
  unsigned v;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
  *out = v;
}

// SM identifiers of the current device (%nsmid: may exceed the SM count)
int device_nsmid() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
  if (cache[dev] > 0) return cache[dev];
  unsigned* d = nullptr;
  unsigned h = 0;
  if (cudaMalloc(&d, sizeof(unsigned)) != cudaSuccess) return -1;
  nsmid_kernel<<<1, 1>>>(d);
  const bool ok = cudaMemcpy(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(d);
  if (!ok || h == 0) return -1;
  cache[dev] = (int)h;
  return cache[dev];
}

struct FusedPlan {
  const void* fn;
  int slots_per_sm, nsmid;
  int64_t slice_ints, lock_bytes, scratch_bytes;
};

int fused_plan(int eq, int p, int nt, bool val, int row_cap, FusedPlan& pl) {
  if (p < 0 || p > 16) return set_error(TSQBX_ERR_ARGUMENT, "fused: order p=%d outside [0, 16]", p);
  if (row_cap <= 0 || (row_cap & 3))
    return set_error(TSQBX_ERR_ARGUMENT, "fused: row_cap must be a positive multiple of 4");
  pl.fn = fused_fn(eq, p, nt, val);
  if (!pl.fn) return set_error(TSQBX_ERR_ARGUMENT, "fused: no kernel for p=%d", p);
  int blocks = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, pl.fn, kFusedBlock, 0);
  if (e != cudaSuccess) return check_cuda(e, "fused occupancy");
  pl.slots_per_sm = std::max(1, blocks);
  pl.nsmid = device_nsmid();
  if (pl.nsmid <= 0) return set_error(TSQBX_ERR_CUDA, "fused: cannot read %%nsmid");
  pl.slice_ints = 32LL * row_cap;
  const int64_t slots = (int64_t)pl.nsmid * pl.slots_per_sm;
  pl.lock_bytes = nsw::align256(slots * sizeof(unsigned));
  pl.scratch_bytes = pl.lock_bytes + 256 + slots * (kFusedBlock / 32) * pl.slice_ints * 4;
  return TSQBX_OK;
}

}  // namespace
}  // namespace tsqbx

using namespace tsqbx;

extern "C" {

int64_t tsqbx_fused_scratch_bytes(int equation, int p, int targets_per_center, int validate,
                                  int row_cap) {
  FusedPlan pl{};
  if (fused_plan(equation, p, targets_per_center, validate != 0, row_cap, pl) != TSQBX_OK)
    return -1;
  return pl.scratch_bytes;
}

int tsqbx_eval_fused(int equation, double k, int p, const double* packed, int64_t n_src,
                     const double* ctr_user, const double* radius, const int32_t* ctr_order,
                     void* near_ws, int64_t near_ws_bytes, const double* ctr_proc, int64_t n_ctr,
                     const double* tgt_proc, int64_t n_tgt, const int64_t* tgt_out,
                     unsigned flags, int row_cap, void* scratch, int64_t scratch_bytes,
                     double* out, int64_t* err, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (equation != TSQBX_EQ_LAPLACE && equation != TSQBX_EQ_HELMHOLTZ)
    return set_error(TSQBX_ERR_ARGUMENT, "bad equation %d", equation);
  if (equation == TSQBX_EQ_HELMHOLTZ && !(k > 0.0))
    return set_error(TSQBX_ERR_ARGUMENT, "Helmholtz requires k > 0");
  if (n_ctr < 0 || n_src < 0 || n_src > INT32_MAX - 64 || n_ctr > INT32_MAX - 64)
    return set_error(TSQBX_ERR_ARGUMENT, "fused: bad sizes");
  const int tuni = (flags & TSQBX_FLAG_UNIFORM_TARGETS) ? (int)((flags >> 8) & 0xffu) : 0;
  if (tuni < 1 || tuni > 2 || n_tgt != (int64_t)tuni * n_ctr)
    return set_error(TSQBX_ERR_ARGUMENT,
                     "fused: needs uniform target runs of 1 or 2 (n_tgt = k n_ctr)");
  if (!err) return set_error(TSQBX_ERR_ARGUMENT, "fused: err (int64[2]) required");
  const nsw::NearLayout L = nsw::near_layout(n_ctr, n_src);
  if (!near_ws || near_ws_bytes < (int64_t)L.total)
    return set_error(TSQBX_ERR_ARGUMENT, "fused: near workspace too small (need %lld)",
                     (long long)L.total);
  if (n_ctr > 0 && (!packed || !ctr_user || !radius || !ctr_order || !ctr_proc || !tgt_proc || !out))
    return set_error(TSQBX_ERR_ARGUMENT, "fused: null array");
  const bool val = (flags & TSQBX_FLAG_VALIDATE) != 0;
  FusedPlan pl{};
  int rc = fused_plan(equation, p, tuni, val, row_cap, pl);
  if (rc != TSQBX_OK) return rc;
  if (!scratch || scratch_bytes < pl.scratch_bytes)
    return set_error(TSQBX_ERR_ARGUMENT, "fused: scratch too small (need %lld)",
                     (long long)pl.scratch_bytes);
  cudaError_t e = cudaMemsetAsync(scratch, 0, pl.lock_bytes, st);
  if (e != cudaSuccess) return check_cuda(e, "fused memset");
  fused_err_init<<<1, 1, 0, st>>>(err);
  if (n_ctr == 0) return TSQBX_OK;

  char* ws = static_cast<char*>(near_ws);
  EvalParams a{};
  a.sp = reinterpret_cast<const double4*>(packed);
  a.swi = packed + 4 * n_src;
  a.snrm = nullptr;
  a.imag_flag = reinterpret_cast<const unsigned*>(packed + packed_meta_offset(n_src, 0));
  a.ctr = ctr_proc;
  a.sell_idx = reinterpret_cast<const int32_t*>(static_cast<char*>(scratch) + pl.lock_bytes + 256);
  a.tgt = tgt_proc;
  a.tout = tgt_out;
  a.out = reinterpret_cast<double2*>(out);
  a.err = reinterpret_cast<unsigned long long*>(err);
  a.n_ctr = n_ctr;
  a.p = p;
  a.G = 1;
  a.validate = val ? 1 : 0;
  a.real_w = (flags & TSQBX_FLAG_REAL_WEIGHTS) ? 1 : 0;
  a.tuni = tuni;
  a.tbase = 0;
  a.k = k;
  a.sc = kSincCos;
  a.series = (flags & TSQBX_FLAG_KR_NARROW) ? 1 : (flags & TSQBX_FLAG_KR_WIDE) ? 2 : 0;
  a.long_rows = 1;
  FusedArgs f{};
  f.in = nsw::SweepIn{ctr_user, radius, n_ctr, ctr_order,
                      reinterpret_cast<const double*>(ws + L.off_prm),
                      reinterpret_cast<const double4*>(ws + L.off_sxyz),
                      reinterpret_cast<const unsigned long long*>(ws + L.off_hkey),
                      reinterpret_cast<const int32_t*>(ws + L.off_hst),
                      reinterpret_cast<const int32_t*>(ws + L.off_hen), L.cap};
  f.scratch = const_cast<int32_t*>(a.sell_idx);
  f.lock = static_cast<unsigned*>(scratch);
  f.slots_per_sm = pl.slots_per_sm;
  f.row_cap = row_cap;
  f.overflow = reinterpret_cast<unsigned long long*>(err + 1);
  const unsigned grid = (unsigned)((n_ctr + kFusedBlock - 1) / kFusedBlock);
  void* args[] = {&a, &f};
  e = cudaLaunchKernel(pl.fn, dim3(grid), dim3(kFusedBlock), args, 0, st);
  if (e != cudaSuccess) return check_cuda(e, "fused launch");
  return TSQBX_OK;
}

}  // extern "C"
