// cuSPARSE SpMM baseline (include/pspmm_baseline.h).  Built into a separate
// library (libpspmm_cusparse.so) that the product never loads.
#include <cuda_runtime.h>
#include <cusparse.h>

#include <new>

#include "pspmm_baseline.h"

struct pspmm_cusparse_plan_s {
  cusparseHandle_t h = nullptr;
  cusparseSpMatDescr_t A = nullptr;
  cusparseDnMatDescr_t B = nullptr, C = nullptr;
  cusparseSpMMAlg_t alg = CUSPARSE_SPMM_ALG_DEFAULT;
  void *buf = nullptr;
  float alpha = 1.f, beta = 0.f;
};

#define CS_TRY(x)                                    \
  do {                                               \
    cusparseStatus_t _s = (x);                       \
    if (_s != CUSPARSE_STATUS_SUCCESS) {             \
      pspmm_cusparse_destroy(p);                     \
      return (int)_s;                                \
    }                                                \
  } while (0)

extern "C" {

void pspmm_cusparse_destroy(pspmm_cusparse_plan p) {
  if (!p) return;
  if (p->A) cusparseDestroySpMat(p->A);
  if (p->B) cusparseDestroyDnMat(p->B);
  if (p->C) cusparseDestroyDnMat(p->C);
  if (p->h) cusparseDestroy(p->h);
  if (p->buf) cudaFree(p->buf);
  delete p;
}

int pspmm_cusparse_create(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                          const int32_t *d_colidx, const float *d_val, const float *d_B,
                          int64_t ldb, int32_t K, float *d_C, int64_t ldc, int32_t alg,
                          void *stream, pspmm_cusparse_plan *out) {
  *out = nullptr;
  pspmm_cusparse_plan p = new (std::nothrow) pspmm_cusparse_plan_s();
  if (!p) return 2000;
  switch (alg) {
    case 1: p->alg = CUSPARSE_SPMM_CSR_ALG1; break;
    case 2: p->alg = CUSPARSE_SPMM_CSR_ALG2; break;
    case 3: p->alg = CUSPARSE_SPMM_CSR_ALG3; break;
    default: p->alg = CUSPARSE_SPMM_ALG_DEFAULT; break;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CS_TRY(cusparseCreate(&p->h));
  CS_TRY(cusparseSetStream(p->h, s));
  CS_TRY(cusparseCreateCsr(&p->A, n_rows, n_cols, nnz, (void *)d_rowptr, (void *)d_colidx,
                           (void *)d_val, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                           CUSPARSE_INDEX_BASE_ZERO, CUDA_R_32F));
  CS_TRY(cusparseCreateDnMat(&p->B, n_cols, K, ldb, (void *)d_B, CUDA_R_32F, CUSPARSE_ORDER_ROW));
  CS_TRY(cusparseCreateDnMat(&p->C, n_rows, K, ldc, (void *)d_C, CUDA_R_32F, CUSPARSE_ORDER_ROW));
  size_t bytes = 0;
  CS_TRY(cusparseSpMM_bufferSize(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                 CUSPARSE_OPERATION_NON_TRANSPOSE, &p->alpha, p->A, p->B, &p->beta,
                                 p->C, CUDA_R_32F, p->alg, &bytes));
  if (bytes) {
    cudaError_t e = cudaMalloc(&p->buf, bytes);
    if (e != cudaSuccess) {
      pspmm_cusparse_destroy(p);
      return 1000 + (int)e;
    }
  }
  CS_TRY(cusparseSpMM_preprocess(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                 CUSPARSE_OPERATION_NON_TRANSPOSE, &p->alpha, p->A, p->B, &p->beta,
                                 p->C, CUDA_R_32F, p->alg, p->buf));
  *out = p;
  return 0;
}

int pspmm_cusparse_run(pspmm_cusparse_plan p, void *stream) {
  if (!p) return 2001;
  cusparseStatus_t s = cusparseSetStream(p->h, reinterpret_cast<cudaStream_t>(stream));
  if (s != CUSPARSE_STATUS_SUCCESS) return (int)s;
  s = cusparseSpMM(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE,
                   &p->alpha, p->A, p->B, &p->beta, p->C, CUDA_R_32F, p->alg, p->buf);
  return (int)s;
}

}  // extern "C"
