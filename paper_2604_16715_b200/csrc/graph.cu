// Graph preparation on the device (plan time): transposed pattern A^T and index remaps.
//
// A^T is needed by the backward column pass (dK = dS^T Q and dV = U^T dY are
// SpMMs over A^T).  CSC is built by a stable LSD radix sort of the entries keyed by column with
// the source row as value; the input is in CSR order (rows ascending), so stability leaves rows
// ascending within each column -> the canonical CSC, unique given the edge set (bit-exact vs
// the oracle's counting-sort transpose).  The sort carries the CSR entry index, so the same pass
// yields the CSC -> CSR entry map through which the column pass reads the row pass's (P, dS).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gt_internal.h"

namespace gt {
namespace {

__global__ void expand_rows_kernel(const int64_t* row_ptr, int64_t n, int32_t* rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw)
    for (int64_t e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) rows[e] = (int32_t)i;
}

__global__ void iota_kernel(int32_t* x, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] = (int32_t)e;
}

// CSC position p holds CSR entry src[p]: row[p] = rows_of_entry[src[p]]
__global__ void gather_rows_kernel(const int32_t* src, const int32_t* rows_of_entry, int64_t n, int32_t* row) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    row[p] = rows_of_entry[src[p]];
}

// out[p - p_lo] = src[p] - e_lo when that CSR entry is in [e_lo, e_hi) (an owned row), else -1
__global__ void local_src_kernel(const int32_t* src, int64_t p_lo, int64_t p_hi, int64_t e_lo, int64_t e_hi,
                                 int32_t* out) {
  for (int64_t p = p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p_hi;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = src[p];
    out[p - p_lo] = (e >= e_lo && e < e_hi) ? (int32_t)(e - e_lo) : -1;
  }
}

__global__ void count_cols_kernel(const int32_t* col, int64_t nnz, unsigned long long* cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[e], 1ull);
}

}  // namespace

gt_status build_csc_device(const int64_t* d_row_ptr, const int32_t* d_col, int64_t n, int64_t nnz,
                           int64_t* d_col_ptr, int32_t* d_row, int32_t* d_src, cudaStream_t st) {
  DevBuf rows_in, keys_out, cnt, tmp, ids, src_own;
  GT_TRY(cnt.alloc((size_t)(n + 1) * sizeof(unsigned long long)));
  GT_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, (size_t)(n + 1) * sizeof(unsigned long long), st));
  if (nnz > 0) {
    // sort (column, CSR entry index) pairs: stable, so entries (rows) stay ascending within a column
    GT_TRY(rows_in.alloc((size_t)nnz * sizeof(int32_t)));
    GT_TRY(keys_out.alloc((size_t)nnz * sizeof(int32_t)));
    GT_TRY(ids.alloc((size_t)nnz * sizeof(int32_t)));
    int32_t* src = d_src;
    if (!src) {
      GT_TRY(src_own.alloc((size_t)nnz * sizeof(int32_t)));
      src = src_own.as<int32_t>();
    }
    expand_rows_kernel<<<1184, 256, 0, st>>>(d_row_ptr, n, rows_in.as<int32_t>());
    iota_kernel<<<1184, 256, 0, st>>>(ids.as<int32_t>(), nnz);
    count_cols_kernel<<<1184, 256, 0, st>>>(d_col, nnz, cnt.as<unsigned long long>());
    int end_bit = 1;
    while ((1ll << end_bit) < n) ++end_bit;
    size_t tb = 0;
    GT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)d_col, keys_out.as<uint32_t>(),
                                                ids.as<int32_t>(), src, (int)nnz, 0, end_bit, st));
    size_t tb2 = 0;
    GT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb2, (const int64_t*)cnt.p, d_col_ptr, (int)(n + 1), st));
    GT_TRY(tmp.alloc(std::max(tb, tb2)));
    GT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tb, (const uint32_t*)d_col, keys_out.as<uint32_t>(),
                                                ids.as<int32_t>(), src, (int)nnz, 0, end_bit, st));
    GT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, (const int64_t*)cnt.p, d_col_ptr, (int)(n + 1), st));
    gather_rows_kernel<<<1184, 256, 0, st>>>(src, rows_in.as<int32_t>(), nnz, d_row);
    GT_CUDA_TRY(cudaGetLastError());
  } else {
    GT_CUDA_TRY(cudaMemsetAsync(d_col_ptr, 0, (size_t)(n + 1) * sizeof(int64_t), st));
  }
  GT_CUDA_TRY(cudaStreamSynchronize(st));
  return GT_OK;
}

gt_status build_local_src(const int32_t* d_src, int64_t p_lo, int64_t p_hi, int64_t e_lo, int64_t e_hi,
                          int32_t* d_out, cudaStream_t st) {
  if (p_hi > p_lo) {
    local_src_kernel<<<1184, 256, 0, st>>>(d_src, p_lo, p_hi, e_lo, e_hi, d_out);
    GT_CUDA_TRY(cudaGetLastError());
  }
  GT_CUDA_TRY(cudaStreamSynchronize(st));
  return GT_OK;
}

}  // namespace gt
