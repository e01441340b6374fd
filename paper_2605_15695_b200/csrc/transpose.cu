// (f3) CSR transpose on the device: the adjacency of A^T, whose PCSR gives the
// backward SpMM of a GNN layer, dL/dB = A^T . dL/dC (PAPER.md P:21-23, P:449-460
// GCN/GIN training).  A stable radix sort of the nonzeros by
// column keeps rows ascending inside every column, so the result is canonical
// CSR and bit-for-bit deterministic.
#include <cub/cub.cuh>

#include "common.cuh"

namespace pspmm {
namespace {

// row index of every nonzero (CSR -> COO rows), one warp per row
__global__ void expand_rows_kernel(int64_t n_rows, const int32_t *__restrict__ rowptr,
                                   int32_t *__restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows;
       i += warps)
    for (int p = rowptr[i] + lane; p < rowptr[i + 1]; p += 32) rows[p] = (int32_t)i;
}

__global__ void iota_kernel(int64_t n, int32_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

// t_rowptr[c] = first position of column c among the sorted keys
__global__ void bounds_kernel(int64_t nnz, int64_t n_cols, const int32_t *__restrict__ keys,
                              int32_t *__restrict__ t_rowptr) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = p == 0 ? -1 : keys[p - 1];
    const int64_t hi = p == nnz ? n_cols : keys[p];
    for (int64_t c = lo + 1; c <= hi; ++c) t_rowptr[c] = (int32_t)p;
  }
}

__global__ void gather_kernel(int64_t nnz, const int32_t *__restrict__ perm,
                              const int32_t *__restrict__ rows, const float *__restrict__ val,
                              int32_t *__restrict__ t_colidx, float *__restrict__ t_val) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = perm[p];
    t_colidx[p] = rows[q];
    t_val[p] = val[q];
  }
}

int grid(int64_t items) {
  int64_t b = (items + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

pspmm_status csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                           const int32_t *d_colidx, const float *d_val, int32_t *d_t_rowptr,
                           int32_t *d_t_colidx, float *d_t_val, cudaStream_t stream) {
  if (!d_t_rowptr || (nnz > 0 && (!d_t_colidx || !d_t_val || !d_val)))
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "csr_transpose: null output");
  pspmm_status st = validate_csr(n_rows, n_cols, nnz, d_rowptr, d_colidx, stream);
  if (st != PSPMM_OK) return st;
  if (nnz == 0) {
    PSPMM_CUDA_TRY(cudaMemsetAsync(d_t_rowptr, 0, (size_t)(n_cols + 1) * sizeof(int32_t), stream));
    PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
    return PSPMM_OK;
  }
  int32_t *rows = nullptr, *idx = nullptr, *keys_out = nullptr, *perm = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  PSPMM_CUDA_TRY(cudaMallocAsync(&rows, nnz * sizeof(int32_t), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&idx, nnz * sizeof(int32_t), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&keys_out, nnz * sizeof(int32_t), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&perm, nnz * sizeof(int32_t), stream));
  expand_rows_kernel<<<grid(n_rows * 32), 256, 0, stream>>>(n_rows, d_rowptr, rows);
  iota_kernel<<<grid(nnz), 256, 0, stream>>>(nnz, idx);
  PSPMM_CUDA_TRY(cudaGetLastError());
  int end_bit = 1;
  while (end_bit < 32 && (int64_t(1) << end_bit) < n_cols) ++end_bit;
  // stable LSD radix sort of (col, original position) pairs
  PSPMM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_colidx, keys_out, idx, perm,
                                                 (int)nnz, 0, end_bit, stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes > 0 ? tmp_bytes : 16, stream));
  PSPMM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, d_colidx, keys_out, idx, perm,
                                                 (int)nnz, 0, end_bit, stream));
  bounds_kernel<<<grid(nnz + 1), 256, 0, stream>>>(nnz, n_cols, keys_out, d_t_rowptr);
  gather_kernel<<<grid(nnz), 256, 0, stream>>>(nnz, perm, rows, d_val, d_t_colidx, d_t_val);
  PSPMM_CUDA_TRY(cudaGetLastError());
  PSPMM_CUDA_TRY(cudaFreeAsync(tmp, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(rows, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(idx, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(keys_out, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(perm, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  return PSPMM_OK;
}

}  // namespace pspmm
