// (a1) CSR intake check — the canonical-CSR preconditions of the boundary
// ("traversal range of i-th row is (rowPtr[i], rowPtr[i+1])";
// SPEC S:33-34 invariants).  One warp per row, grid-stride; any violation
// raises a device flag that the host reads after one stream sync.
#include "common.cuh"

namespace pspmm {
namespace {

enum : unsigned { kBadRowptr = 1u, kBadColRange = 2u, kNotSorted = 4u, kBadEnds = 8u };

__global__ void __launch_bounds__(256) validate_kernel(int64_t n_rows, int64_t n_cols,
                                                       int64_t nnz,
                                                       const int32_t *__restrict__ rowptr,
                                                       const int32_t *__restrict__ colidx,
                                                       unsigned *__restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned bad = 0;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w == 0 && lane == 0) {
    if (rowptr[0] != 0 || (int64_t)rowptr[n_rows] != nnz) bad |= kBadEnds;
  }
  for (int64_t i = w; i < n_rows; i += warps) {
    const int64_t head = rowptr[i], tail = rowptr[i + 1];
    if (head > tail || head < 0 || tail > nnz) {
      bad |= kBadRowptr;
      continue;
    }
    for (int64_t p = head + lane; p < tail; p += 32) {
      const int32_t c = colidx[p];
      if (c < 0 || (int64_t)c >= n_cols) bad |= kBadColRange;
      if (p + 1 < tail && colidx[p + 1] <= c) bad |= kNotSorted;
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0 && bad) atomicOr(flag, bad);
}

}  // namespace

pspmm_status validate_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                          const int32_t *d_colidx, cudaStream_t stream) {
  if (n_rows < 1 || n_cols < 1 || nnz < 0 || !d_rowptr || (nnz > 0 && !d_colidx))
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "validate: bad sizes or null pointer");
  if (n_rows >= INT32_MAX || n_cols >= INT32_MAX || nnz >= INT32_MAX)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "validate: sizes need int64 indices");
  unsigned *d_flag = nullptr;
  PSPMM_CUDA_TRY(cudaMallocAsync(&d_flag, sizeof(unsigned), stream));
  PSPMM_CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(unsigned), stream));
  int64_t blocks = (n_rows + 7) / 8;
  int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  validate_kernel<<<(unsigned)blocks, 256, 0, stream>>>(n_rows, n_cols, nnz, d_rowptr,
                                                          d_colidx, d_flag);
  PSPMM_CUDA_TRY(cudaGetLastError());
  unsigned h_flag = 0;
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&h_flag, d_flag, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                 stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(d_flag, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  if (h_flag) {
    std::string why = "CSR not canonical:";
    if (h_flag & kBadEnds) why += " rowPtr[0]!=0 or rowPtr[n]!=nnz;";
    if (h_flag & kBadRowptr) why += " rowPtr decreasing or out of range;";
    if (h_flag & kBadColRange) why += " column index out of range;";
    if (h_flag & kNotSorted) why += " columns not strictly increasing in a row;";
    PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, why);
  }
  return PSPMM_OK;
}

}  // namespace pspmm
