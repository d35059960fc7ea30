// boxes.cu -- box interaction lists -> per-row source index lists.
//
// The reference's direct stages (driver.py:197-228) walk the target boxes one
// by one: the sources of box b's list (List 1, 3close or 4close; ilists.py
// CSR `starts/flat`) are the concatenated owned source ranges of the listed
// boxes (_gather_sources, driver.py:109-113), and every center / conventional
// target owned by b is evaluated against them.  On the GPU that walk becomes
// one batched evaluation over rows: row r (a center, or a target box for the
// p2p rows) belongs to box row_box[r] and its index list is that expansion,
// written here by two kernels (count + scan, then fill; a warp per row writes
// each owned range as a coalesced run of consecutive indices).
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace tsqbx {
namespace {

struct BoxArgs {
  const int64_t* __restrict__ row_box;   // box of row r (< 0: empty row)
  const int64_t* __restrict__ lst_ptr;   // list CSR over boxes (n_boxes + 1)
  const int64_t* __restrict__ lst_box;
  const int64_t* __restrict__ box_start; // owned source range of box d:
  const int64_t* __restrict__ box_end;   //   [box_start[d*stride], box_end[d*stride])
  int64_t stride;
  int64_t n_rows;
};

__global__ void box_count_kernel(BoxArgs a, int64_t* __restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > a.n_rows) return;
  int64_t n = 0;
  if (r < a.n_rows) {
    const int64_t b = a.row_box[r];
    if (b >= 0) {
      for (int64_t q = a.lst_ptr[b]; q < a.lst_ptr[b + 1]; ++q) {
        const int64_t d = a.lst_box[q];
        n += a.box_end[d * a.stride] - a.box_start[d * a.stride];
      }
    }
  }
  cnt[r] = n;   // cnt[n_rows] = 0: the exclusive scan's last entry is the total
}

__global__ void box_fill_kernel(BoxArgs a, const int64_t* __restrict__ row_ptr,
                                int32_t* __restrict__ row_idx) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= a.n_rows) return;
  const int64_t b = a.row_box[r];
  if (b < 0) return;
  int64_t out = row_ptr[r];
  for (int64_t q = a.lst_ptr[b]; q < a.lst_ptr[b + 1]; ++q) {
    const int64_t d = a.lst_box[q];
    const int64_t s0 = a.box_start[d * a.stride], s1 = a.box_end[d * a.stride];
    for (int64_t s = s0 + lane; s < s1; s += 32) row_idx[out + (s - s0)] = (int32_t)s;
    out += s1 - s0;
  }
}

size_t scan_bytes(int64_t n_rows) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n_rows + 1));
  return t;
}

}  // namespace
}  // namespace tsqbx

using namespace tsqbx;

extern "C" {

int64_t tsqbx_box_rows_workspace_bytes(int64_t n_rows) {
  const int64_t cnt = ((n_rows + 1) * (int64_t)sizeof(int64_t) + 255) / 256 * 256;
  return cnt + (int64_t)scan_bytes(n_rows) + 256;
}

int tsqbx_box_rows_count(int64_t n_rows, const int64_t* row_box, const int64_t* lst_ptr,
                         const int64_t* lst_box, const int64_t* box_start,
                         const int64_t* box_end, int64_t box_stride, void* workspace,
                         int64_t ws_bytes, int64_t* row_ptr, int64_t* total, void* stream) {
  if (n_rows < 0 || n_rows >= INT32_MAX || !row_ptr || !total || box_stride < 1 ||
      (n_rows > 0 && (!row_box || !lst_ptr || !box_start || !box_end)))
    return set_error(TSQBX_ERR_ARGUMENT, "box_rows_count: bad arguments");
  if (!workspace || ws_bytes < tsqbx_box_rows_workspace_bytes(n_rows))
    return set_error(TSQBX_ERR_ARGUMENT, "box_rows_count: workspace too small");
  const cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);
  int64_t* cnt = reinterpret_cast<int64_t*>(ws);
  const int64_t off = ((n_rows + 1) * (int64_t)sizeof(int64_t) + 255) / 256 * 256;
  BoxArgs a{row_box, lst_ptr, lst_box, box_start, box_end, box_stride, n_rows};
  box_count_kernel<<<(unsigned)((n_rows + 1 + 255) / 256), 256, 0, st>>>(a, cnt);
  size_t tb = scan_bytes(n_rows);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(ws + off, tb, cnt, row_ptr, (int)(n_rows + 1), st);
  if (e != cudaSuccess) return check_cuda(e, "box_rows scan");
  e = cudaMemcpyAsync(total, row_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return check_cuda(e, "box_rows total");
  return check_cuda(cudaGetLastError(), "box_rows_count launch");
}

int tsqbx_box_rows_fill(int64_t n_rows, const int64_t* row_box, const int64_t* lst_ptr,
                        const int64_t* lst_box, const int64_t* box_start, const int64_t* box_end,
                        int64_t box_stride, const int64_t* row_ptr, int32_t* row_idx,
                        void* stream) {
  if (n_rows < 0 || box_stride < 1 || (n_rows > 0 && (!row_box || !lst_ptr || !box_start ||
                                                      !box_end || !row_ptr)))
    return set_error(TSQBX_ERR_ARGUMENT, "box_rows_fill: bad arguments");
  if (n_rows == 0) return TSQBX_OK;
  BoxArgs a{row_box, lst_ptr, lst_box, box_start, box_end, box_stride, n_rows};
  box_fill_kernel<<<(unsigned)((n_rows * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      a, row_ptr, row_idx);
  return check_cuda(cudaGetLastError(), "box_rows_fill launch");
}

}  // extern "C"
