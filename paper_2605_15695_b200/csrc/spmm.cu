// (a6, a7) Host dispatch of the ParamSpMM computing engine (Alg. 2,
// P:215-267) and its two helper kernels.  The kernel template and its
// design notes are in spmm_kernel.cuh.
#include <algorithm>

#include "spmm_kernel.cuh"

namespace pspmm {
namespace {
using namespace detail;

// Zero the C rows of panels that own more than one chunk (S = 1, c-12).
__global__ void zero_split_kernel(const int32_t *__restrict__ split, int64_t num_split, int V,
                                  int64_t n_rows, int32_t K, float *__restrict__ C, int64_t ldc) {
  const int64_t per = (int64_t)V * K;
  const int64_t total = num_split * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / per, r = t % per;
    const int64_t row = (int64_t)split[s] * V + r / K;
    if (row < n_rows) C[row * ldc + r % K] = 0.f;
  }
}

// C = 0 (nnz_V == 0).
__global__ void zero_all_kernel(int64_t n_rows, int32_t K, float *__restrict__ C, int64_t ldc) {
  const int64_t total = n_rows * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    C[(t / K) * ldc + t % K] = 0.f;
}

KernelFn pick_kernel(int V, int S, bool vec, int F, int G) {
  if (V == 1) return S ? pick_v1s1(vec, F, G) : pick_v1s0(vec, F, G);
  return S ? pick_v2s1(vec, F, G) : pick_v2s0(vec, F, G);
}

bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

int ceil_pow2(int64_t x) {
  int p = 1;
  while (p < x && p < 32) p <<= 1;
  return p;
}

}  // namespace

pspmm_status run_spmm(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K, float *d_C,
                      int64_t ldc, const pspmm_config &cfg, cudaStream_t stream) {
  if (!A || !d_B || !d_C) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run: null handle or pointer");
  if (K < 1 || ldb < K || ldc < K)
    PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "spmm_run: need K >= 1, ldb >= K, ldc >= K");
  if (cfg.V != A->V || cfg.S != A->S || cfg.omega != A->omega)
    PSPMM_FAIL(PSPMM_ERR_CONFIG_MISMATCH, "spmm_run: cfg.V/S/omega differ from the PCSR handle");
  if (cfg.mode != 0 && cfg.mode != 2)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: mode must be 0 (LDG engine) or 2 (TMA gather)");
  if (!(cfg.W == 1 || cfg.W == 2 || cfg.W == 4 || cfg.W == 8))
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: W must be 1, 2, 4 or 8");
  if (cfg.W * 32 > PSPMM_MAX_THREADS)
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: W exceeds this build's launch bounds");
  if (cfg.F < 1 || cfg.F > 8)
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: F must be in 1..8 (float4 units)");
  if (cfg.G != 0 && !(pow2(cfg.G) && cfg.G <= 32))
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: G must be 0 or a power of two <= 32");

  const int64_t n_rows = A->n_rows;
  if (A->nnz_v == 0) {
    int64_t total = n_rows * K;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    zero_all_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(n_rows, K, d_C, ldc);
    PSPMM_CUDA_TRY(cudaGetLastError());
    return PSPMM_OK;
  }

  const bool vec = (K % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(d_B) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(d_C) & 15) == 0);
  int F = cfg.F, G = cfg.G, cols_per_pass;
  if (vec) {
    if (G == 0) G = ceil_pow2((K / 4 + F - 1) / F);
    cols_per_pass = 4 * G * F;
  } else {
    // masked scalar variant: one column per lane, G = min(32, pow2 >= K)
    F = 1;
    G = ceil_pow2(K);
    cols_per_pass = G;
  }
  KernelFn fn = nullptr;
  if (cfg.mode == 2) {
    if (!tma_supported(K, ldb, ldc, d_B, d_C))
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
                 "spmm_run mode 2: needs K % 32 == 0, ld % 4 == 0 and 16-B aligned B and C");
  } else {
    fn = pick_kernel(A->V, A->S, vec, F, G);
    if (!fn) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: no kernel instance for this config");
  }

  if (A->S == 1 && A->num_split > 0) {
    int64_t total = A->num_split * A->V * (int64_t)K;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    zero_split_kernel<<<blocks, 256, 0, stream>>>(A->d_split, A->num_split, A->V, n_rows, K, d_C,
                                                   ldc);
    PSPMM_CUDA_TRY(cudaGetLastError());
  }
  if (cfg.mode == 2) return run_spmm_tma(A, d_B, ldb, K, d_C, ldc, cfg, stream);

  SpmmArgs args;
  args.rowptr = A->d_rowptr;
  args.colidx = A->d_colidx;
  args.val = A->d_val;
  args.trow = A->d_trow;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.n_rows = (int32_t)n_rows;
  args.units = (int32_t)A->num_chunks;
  args.K = K;
  const int threads = cfg.W * 32;
  const int64_t groups_per_block = threads / G;
  // groups loop over units (grid-stride): cap the grid at PSPMM_WAVES waves of
  // resident blocks so each group pipelines several units
  int64_t bx = (A->num_chunks + groups_per_block - 1) / groups_per_block;
  const int64_t resident = std::min<int64_t>(32, (PSPMM_MAX_THREADS * PSPMM_MIN_BLOCKS) / threads);
  if (PSPMM_WAVES > 0) bx = std::min<int64_t>(bx, (int64_t)num_sms() * resident * PSPMM_WAVES);
  const int64_t by = (K + cols_per_pass - 1) / cols_per_pass;
  if ((uint64_t)ldb * 4 >= (1ull << 32))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: ldb * 4 bytes must be < 2^32");
  if (bx > 0x7fffffff || by > 65535)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: grid too large for this config");
  fn<<<dim3((unsigned)bx, (unsigned)by), threads, 0, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
