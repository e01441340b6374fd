/*
 * pspmm_baseline.h — cuSPARSE SpMM baseline (libpspmm_cusparse.so).
 *
 * NOT part of the product path: bench.py and the tests use it to time the
 * vendor library on the same box and data (SURVEY §8(d)
 * "cuSPARSE baseline").  Generic cusparseSpMM with a CSR descriptor (int32
 * indices, fp32 values), row-major dense B and C, alpha = 1, beta = 0.
 * bufferSize and SpMM_preprocess run in create (not timed); run issues
 * exactly one cusparseSpMM on `stream`.
 *
 * alg: 0 = CUSPARSE_SPMM_ALG_DEFAULT, 1 = CSR_ALG1, 2 = CSR_ALG2,
 *      3 = CSR_ALG3.  Returns 0 on success, otherwise the cusparseStatus_t
 *      (or 1000 + cudaError_t) of the failing call.
 */
#ifndef PSPMM_BASELINE_H
#define PSPMM_BASELINE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct pspmm_cusparse_plan_s *pspmm_cusparse_plan;

int pspmm_cusparse_create(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                          const int32_t *d_colidx, const float *d_val, const float *d_B,
                          int64_t ldb, int32_t K, float *d_C, int64_t ldc, int32_t alg,
                          void *stream, pspmm_cusparse_plan *out);
int pspmm_cusparse_run(pspmm_cusparse_plan plan, void *stream);
void pspmm_cusparse_destroy(pspmm_cusparse_plan plan);

#ifdef __cplusplus
}
#endif
#endif
