// (f1) Applying a node permutation on the device: A' = P A P^T (row i of A
// becomes row perm[i], column j becomes perm[j]; columns re-sorted per row)
// and the matching row permutation of the dense B / C (B' = P B, C = P^T C').
// Then SpMM(A', B') = P SpMM(A, B), so a reordered graph can be
// used in every layer and only the final output is un-permuted.
#include <cub/cub.cuh>

#include "common.cuh"

namespace pspmm {
namespace {

int grid(int64_t items) {
  int64_t b = (items + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

__global__ void new_degree_kernel(int64_t n, const int32_t *__restrict__ rowptr,
                                  const int32_t *__restrict__ perm, int32_t *__restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (i < n)
      deg[perm[i]] = rowptr[i + 1] - rowptr[i];
    else
      deg[n] = 0;
}

// one warp per old row: relabel the columns into the new row's slot
__global__ void scatter_kernel(int64_t n, const int32_t *__restrict__ rowptr,
                               const int32_t *__restrict__ colidx, const float *__restrict__ val,
                               const int32_t *__restrict__ perm,
                               const int32_t *__restrict__ new_rowptr,
                               int32_t *__restrict__ out_col, float *__restrict__ out_val) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int h = rowptr[i], t = rowptr[i + 1];
    const int64_t base = new_rowptr[perm[i]];
    for (int p = h + lane; p < t; p += 32) {
      out_col[base + (p - h)] = perm[colidx[p]];
      out_val[base + (p - h)] = val[p];
    }
  }
}

__global__ void permute_rows_kernel(int64_t n, int32_t K, const float *__restrict__ in, int64_t ldi,
                                    const int32_t *__restrict__ perm, float *__restrict__ out,
                                    int64_t ldo, int inverse) {
  const int64_t total = n * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / K, k = t % K;
    if (inverse)
      out[i * ldo + k] = in[(int64_t)perm[i] * ldi + k];  // C[i] = C'[perm[i]]
    else
      out[(int64_t)perm[i] * ldo + k] = in[i * ldi + k];  // B'[perm[i]] = B[i]
  }
}

}  // namespace

pspmm_status csr_permute(int64_t n, int64_t nnz, const int32_t *d_rowptr, const int32_t *d_colidx,
                         const float *d_val, const int32_t *d_perm, int32_t *d_out_rowptr,
                         int32_t *d_out_colidx, float *d_out_val, cudaStream_t stream) {
  if (!d_perm || !d_out_rowptr || (nnz > 0 && (!d_out_colidx || !d_out_val || !d_val)))
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "csr_permute: null argument");
  pspmm_status st = validate_csr(n, n, nnz, d_rowptr, d_colidx, stream);
  if (st != PSPMM_OK) return st;
  int32_t *deg = nullptr, *tmp_col = nullptr;
  float *tmp_val = nullptr;
  void *tmp = nullptr;
  size_t bytes = 0;
  PSPMM_CUDA_TRY(cudaMallocAsync(&deg, (n + 1) * sizeof(int32_t), stream));
  new_degree_kernel<<<grid(n + 1), 256, 0, stream>>>(n, d_rowptr, d_perm, deg);
  PSPMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg, d_out_rowptr, (int)(n + 1),
                                               stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&tmp, bytes > 0 ? bytes : 16, stream));
  PSPMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, bytes, deg, d_out_rowptr, (int)(n + 1), stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(tmp, stream));
  if (nnz > 0) {
    PSPMM_CUDA_TRY(cudaMallocAsync(&tmp_col, nnz * sizeof(int32_t), stream));
    PSPMM_CUDA_TRY(cudaMallocAsync(&tmp_val, nnz * sizeof(float), stream));
    scatter_kernel<<<grid(n * 32), 256, 0, stream>>>(n, d_rowptr, d_colidx, d_val, d_perm,
                                                     d_out_rowptr, tmp_col, tmp_val);
    PSPMM_CUDA_TRY(cudaGetLastError());
    // columns ascending inside every new row (they are distinct, so any sort is canonical)
    bytes = 0;
    PSPMM_CUDA_TRY(cub::DeviceSegmentedSort::SortPairs(
        nullptr, bytes, tmp_col, d_out_colidx, tmp_val, d_out_val, (int)nnz, (int)n,
        d_out_rowptr, d_out_rowptr + 1, stream));
    PSPMM_CUDA_TRY(cudaMallocAsync(&tmp, bytes > 0 ? bytes : 16, stream));
    PSPMM_CUDA_TRY(cub::DeviceSegmentedSort::SortPairs(
        tmp, bytes, tmp_col, d_out_colidx, tmp_val, d_out_val, (int)nnz, (int)n, d_out_rowptr,
        d_out_rowptr + 1, stream));
    PSPMM_CUDA_TRY(cudaFreeAsync(tmp, stream));
    PSPMM_CUDA_TRY(cudaFreeAsync(tmp_col, stream));
    PSPMM_CUDA_TRY(cudaFreeAsync(tmp_val, stream));
  }
  PSPMM_CUDA_TRY(cudaFreeAsync(deg, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  return PSPMM_OK;
}

pspmm_status permute_rows(int64_t n, int32_t K, const float *d_in, int64_t ldi,
                          const int32_t *d_perm, float *d_out, int64_t ldo, int32_t inverse,
                          cudaStream_t stream) {
  if (!d_in || !d_out || !d_perm || d_in == d_out)
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "permute_rows: null or aliased arguments");
  if (K < 1 || ldi < K || ldo < K) PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "permute_rows: bad K / ld");
  permute_rows_kernel<<<grid(n * K), 256, 0, stream>>>(n, K, d_in, ldi, d_perm, d_out, ldo,
                                                       inverse);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
