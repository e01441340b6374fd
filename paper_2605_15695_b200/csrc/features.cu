// (a2) Table 3 features on the device.  Readings:
// degree = row nnz (c-22); CV population std over all n rows, CV^ over the
// non-empty rows (c-20); row bandwidth = last col - first col (P:329
// footnote), 0 for empty rows (c-21); SR_i / PR_i with V = i (c-19).
//
// Degree and bandwidth statistics are exact integer reductions (sum of
// degree^2 in 64-bit), so the host can form the variance from exact
// integers: var = (n S2 - S1^2) / n^2 with one rounding.
#include "common.cuh"

namespace pspmm {
namespace {

struct RowStats {
  unsigned long long n_hat, s2, b_sum, d_max, b_max;
};

__global__ void row_stats_kernel(int64_t n, const int32_t *__restrict__ rowptr,
                                 const int32_t *__restrict__ colidx, RowStats *__restrict__ out) {
  unsigned long long n_hat = 0, s2 = 0, b_sum = 0, d_max = 0, b_max = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int h = rowptr[i], t = rowptr[i + 1];
    const unsigned long long d = (unsigned long long)(t - h);
    if (d) {
      n_hat += 1;
      s2 += d * d;
      const unsigned long long bw = (unsigned long long)(colidx[t - 1] - colidx[h]);
      b_sum += bw;
      b_max = bw > b_max ? bw : b_max;
      d_max = d > d_max ? d : d_max;
    }
  }
  // warp reductions, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    n_hat += __shfl_xor_sync(0xffffffffu, n_hat, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    b_sum += __shfl_xor_sync(0xffffffffu, b_sum, o);
    unsigned long long x = __shfl_xor_sync(0xffffffffu, d_max, o);
    d_max = x > d_max ? x : d_max;
    x = __shfl_xor_sync(0xffffffffu, b_max, o);
    b_max = x > b_max ? x : b_max;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out->n_hat, n_hat);
    atomicAdd(&out->s2, s2);
    atomicAdd(&out->b_sum, b_sum);
    atomicMax(&out->d_max, d_max);
    atomicMax(&out->b_max, b_max);
  }
}

// Panel statistics for V in {1, 2}: sum of L, non-empty panels (pass 1), or
// the chunk count sum max(1, ceil(L/SG)) (pass 2, SG > 0).
__global__ void panel_stats_kernel(int64_t n, int V, const int32_t *__restrict__ rowptr,
                                   const int32_t *__restrict__ L2, int64_t SG,
                                   unsigned long long *__restrict__ out /* [sumL, nonempty, chunks] */) {
  const int64_t P = (n + V - 1) / V;
  unsigned long long sum = 0, ne = 0, ch = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const long long L = V == 1 ? (long long)(rowptr[p + 1] - rowptr[p]) : (long long)L2[p];
    sum += (unsigned long long)L;
    ne += L > 0 ? 1ull : 0ull;
    if (SG > 0) ch += L == 0 ? 1ull : (unsigned long long)((L + SG - 1) / SG);
  }
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    ne += __shfl_xor_sync(0xffffffffu, ne, o);
    ch += __shfl_xor_sync(0xffffffffu, ch, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], sum);
    atomicAdd(&out[1], ne);
    atomicAdd(&out[2], ch);
  }
}

}  // namespace

pspmm_status compute_features(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                              const int32_t *d_colidx, int32_t omega, cudaStream_t stream,
                              pspmm_features *out) {
  if (!out || omega < 1) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "features: bad output or omega");
  pspmm_status st = validate_csr(n, n, nnz, d_rowptr, d_colidx, stream);
  if (st != PSPMM_OK) return st;
  if (nnz == 0) PSPMM_FAIL(PSPMM_ERR_EMPTY, "features: undefined for nnz == 0 (S:279)");

  const int64_t P2 = (n + 1) / 2;
  RowStats *d_rs = nullptr;
  unsigned long long *d_ps = nullptr;  // [V=1: 3][V=2: 3]
  int32_t *d_L2 = nullptr;
  PSPMM_CUDA_TRY(cudaMallocAsync(&d_rs, sizeof(RowStats), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&d_ps, 6 * sizeof(unsigned long long), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&d_L2, (size_t)(P2 + 1) * sizeof(int32_t), stream));
  PSPMM_CUDA_TRY(cudaMemsetAsync(d_rs, 0, sizeof(RowStats), stream));
  PSPMM_CUDA_TRY(cudaMemsetAsync(d_ps, 0, 6 * sizeof(unsigned long long), stream));
  const int blocks = num_sms() * 8;
  row_stats_kernel<<<blocks, 256, 0, stream>>>(n, d_rowptr, d_colidx, d_rs);
  PSPMM_CUDA_TRY(cudaGetLastError());
  st = panel_counts_v2(n, d_rowptr, d_colidx, d_L2, stream);
  if (st != PSPMM_OK) return st;
  panel_stats_kernel<<<blocks, 256, 0, stream>>>(n, 1, d_rowptr, d_L2, 0, d_ps);
  panel_stats_kernel<<<blocks, 256, 0, stream>>>(n, 2, d_rowptr, d_L2, 0, d_ps + 3);
  PSPMM_CUDA_TRY(cudaGetLastError());
  RowStats rs;
  unsigned long long ps[6];
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&rs, d_rs, sizeof(rs), cudaMemcpyDeviceToHost, stream));
  PSPMM_CUDA_TRY(cudaMemcpyAsync(ps, d_ps, sizeof(ps), cudaMemcpyDeviceToHost, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));

  // Eq. 3 for V = 1 and V = 2 (integer form, c-3a)
  const int64_t nnz1 = (int64_t)ps[0], ne1 = (int64_t)ps[1];
  const int64_t nnz2 = (int64_t)ps[3], ne2 = (int64_t)ps[4];
  const int64_t SG1 = ((nnz1 + ne1 * omega - 1) / (ne1 * omega)) * omega;
  const int64_t SG2 = ((nnz2 + ne2 * omega - 1) / (ne2 * omega)) * omega;
  PSPMM_CUDA_TRY(cudaMemsetAsync(d_ps, 0, 6 * sizeof(unsigned long long), stream));
  panel_stats_kernel<<<blocks, 256, 0, stream>>>(n, 1, d_rowptr, d_L2, SG1, d_ps);
  panel_stats_kernel<<<blocks, 256, 0, stream>>>(n, 2, d_rowptr, d_L2, SG2, d_ps + 3);
  PSPMM_CUDA_TRY(cudaGetLastError());
  PSPMM_CUDA_TRY(cudaMemcpyAsync(ps, d_ps, sizeof(ps), cudaMemcpyDeviceToHost, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(d_rs, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(d_ps, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(d_L2, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t ch1 = (int64_t)ps[2], ch2 = (int64_t)ps[5];
  const int64_t P1 = n;

  const double dn = (double)n, dnnz = (double)nnz, dnh = (double)rs.n_hat;
  out->n = dn;
  out->n_hat = dnh;
  out->nnz = dnnz;
  out->delta = dnh / dn;
  out->d = dnnz / dn;
  out->d_hat = dnnz / dnh;
  out->d_max = (double)rs.d_max;
  // exact integer numerators of the variances (S1 = nnz, S2 = sum d^2)
  const __int128 S1 = nnz, S2 = (__int128)rs.s2;
  const __int128 num = (__int128)n * S2 - S1 * S1;
  const __int128 num_hat = (__int128)rs.n_hat * S2 - S1 * S1;
  const double var = (double)num / (dn * dn);
  const double var_hat = (double)num_hat / (dnh * dnh);
  out->cv = __builtin_sqrt(var) / out->d;
  out->cv_hat = __builtin_sqrt(var_hat) / out->d_hat;
  out->sr1 = (double)(ch1 + 1) / (double)(P1 + 1);
  out->sr2 = (double)(ch2 + 1) / (double)(P2 + 1);
  out->rho = dnnz / (dn * dn);
  out->b = (double)rs.b_sum / dn;
  out->b_max = (double)rs.b_max;
  out->pr1 = 1.0 - dnnz / ((double)nnz1 * 1.0);
  out->pr2 = 1.0 - dnnz / ((double)nnz2 * 2.0);
  return PSPMM_OK;
}

}  // namespace pspmm
