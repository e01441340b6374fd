// extern "C" entry points of libpspmm.so (declared in include/pspmm.h).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "common.cuh"

namespace pspmm {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) {
  try {
    g_last_error = msg;
  } catch (...) {  // never throws: the message is best-effort
  }
}

void set_error_cstr(const char *where, const char *what) noexcept {
  try {
    g_last_error = std::string(where) + ": " + what;
  } catch (...) {
  }
}

pspmm_status cuda_status(cudaError_t e, const char *where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // clear sticky-free errors
  return e == cudaErrorMemoryAllocation ? PSPMM_ERR_OOM : PSPMM_ERR_CUDA;
}

// cuMemGetAddressRange through the runtime's driver entry point (the library
// does not link libcuda directly)
static PFN_cuMemGetAddressRange_v3020 get_address_range() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

}  // namespace pspmm

using namespace pspmm;

extern "C" {

const char *pspmm_status_string(pspmm_status s) {
  switch (s) {
    case PSPMM_OK: return "PSPMM_OK";
    case PSPMM_ERR_INVALID_ARG: return "PSPMM_ERR_INVALID_ARG";
    case PSPMM_ERR_NOT_CANONICAL: return "PSPMM_ERR_NOT_CANONICAL";
    case PSPMM_ERR_DIM_MISMATCH: return "PSPMM_ERR_DIM_MISMATCH";
    case PSPMM_ERR_CONFIG: return "PSPMM_ERR_CONFIG";
    case PSPMM_ERR_CONFIG_MISMATCH: return "PSPMM_ERR_CONFIG_MISMATCH";
    case PSPMM_ERR_EMPTY: return "PSPMM_ERR_EMPTY";
    case PSPMM_ERR_UNSUPPORTED: return "PSPMM_ERR_UNSUPPORTED";
    case PSPMM_ERR_OOM: return "PSPMM_ERR_OOM";
    case PSPMM_ERR_CUDA: return "PSPMM_ERR_CUDA";
  }
  return "PSPMM_UNKNOWN_STATUS";
}

const char *pspmm_last_error(void) { return g_last_error.c_str(); }

const char *pspmm_version(void) { return "pspmm 0.1 sm_100a"; }

pspmm_status pspmm_csr_validate_rect(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                     const int32_t *d_rowptr, const int32_t *d_colidx,
                                     void *stream) {
  return pspmm::guarded("csr_validate_rect", [&]() -> pspmm_status {
    return validate_csr(n_rows, n_cols, nnz, d_rowptr, d_colidx, as_stream(stream));
  });
}

pspmm_status pspmm_csr_validate(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                                const int32_t *d_colidx, void *stream) {
  return pspmm::guarded("csr_validate", [&]() -> pspmm_status {
    return validate_csr(n, n, nnz, d_rowptr, d_colidx, as_stream(stream));
  });
}

pspmm_status pspmm_pcsr_build_rect(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                   const int32_t *d_rowptr, const int32_t *d_colidx,
                                   const float *d_val, int32_t V, int32_t S, int32_t omega,
                                   int32_t sg_override, void *stream, pspmm_pcsr *out) {
  return pspmm::guarded("pcsr_build_rect", [&]() -> pspmm_status {
    if (!out) {
      set_error("pcsr_build: null out");
      return PSPMM_ERR_INVALID_ARG;
    }
    *out = nullptr;
    pspmm_pcsr_s *A = new (std::nothrow) pspmm_pcsr_s();
    if (!A) {
      set_error("pcsr_build: host allocation failed");
      return PSPMM_ERR_OOM;
    }
    pspmm_status st = build_pcsr(n_rows, n_cols, nnz, d_rowptr, d_colidx, d_val, V, S, omega,
                                 sg_override, as_stream(stream), A);
    if (st != PSPMM_OK) {
      pspmm_pcsr_destroy(A);
      return st;
    }
    *out = A;
    return PSPMM_OK;
  });
}

pspmm_status pspmm_pcsr_build(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                              const int32_t *d_colidx, const float *d_val, int32_t V, int32_t S,
                              int32_t omega, int32_t sg_override, void *stream, pspmm_pcsr *out) {
  return pspmm::guarded("pcsr_build", [&]() -> pspmm_status {
    return pspmm_pcsr_build_rect(n, n, nnz, d_rowptr, d_colidx, d_val, V, S, omega, sg_override,
                                 stream, out);
  });
}

pspmm_status pspmm_pcsr_get_info(pspmm_pcsr A, pspmm_pcsr_info *out) {
  return pspmm::guarded("pcsr_get_info", [&]() -> pspmm_status {
    if (!A || !out) {
      set_error("pcsr_get_info: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    std::memset(out, 0, sizeof(*out));
    out->n = A->n_rows;
    out->num_panels = A->num_panels;
    out->nnz = A->nnz;
    out->nnz_v = A->nnz_v;
    out->num_chunks = A->num_chunks;
    out->sg = A->sg;
    out->V = A->V;
    out->S = A->S;
    out->omega = A->omega;
    out->pr = A->pr;
    out->sr = A->sr;
    return PSPMM_OK;
  });
}

pspmm_status pspmm_pcsr_export(pspmm_pcsr A, int32_t *h_rowptr, int32_t *h_colidx, float *h_val,
                               int32_t *h_trow) {
  return pspmm::guarded("pcsr_export", [&]() -> pspmm_status {
    if (!A) {
      set_error("pcsr_export: null handle");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (h_rowptr)
      PSPMM_CUDA_TRY(cudaMemcpy(h_rowptr, A->d_rowptr, (size_t)A->rowptr_len * sizeof(int32_t),
                                cudaMemcpyDeviceToHost));
    if (h_colidx && A->nnz_v)
      PSPMM_CUDA_TRY(cudaMemcpy(h_colidx, A->d_colidx, (size_t)A->nnz_v * sizeof(int32_t),
                                cudaMemcpyDeviceToHost));
    if (h_val && A->nnz_v)
      PSPMM_CUDA_TRY(cudaMemcpy(h_val, A->d_val, (size_t)A->nnz_v * A->V * sizeof(float),
                                cudaMemcpyDeviceToHost));
    if (h_trow && A->S == 1 && A->num_chunks)
      PSPMM_CUDA_TRY(cudaMemcpy(h_trow, A->d_trow, (size_t)A->num_chunks * sizeof(int32_t),
                                cudaMemcpyDeviceToHost));
    return PSPMM_OK;
  });
}

void pspmm_pcsr_destroy(pspmm_pcsr A) {
  if (!A) return;  // (nothing below allocates or throws: CUDA frees and delete)
  cudaFree(A->d_rowptr);
  cudaFree(A->d_colidx);
  cudaFree(A->d_val);
  cudaFree(A->d_trow);
  cudaFree(A->d_split);
  cudaFree(A->d_order);
  if (A->copy_stream) {
    cudaStreamSynchronize(A->copy_stream);
    cudaStreamDestroy(A->copy_stream);
    for (int k = 0; k < kSlices; ++k)
      if (A->slice_done[k]) cudaEventDestroy(A->slice_done[k]);
  }
  for (cudaStream_t s : {A->h2d_stream, A->d2h_stream})
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t e : {A->h2d_done[b], A->comp_done[b], A->d2h_done[b]})
      if (e) cudaEventDestroy(e);
  if (A->batch_start) cudaEventDestroy(A->batch_start);
  destroy_dense(A->dense);
  destroy_blocks(A->blocks);
  destroy_band(A->band);
  delete A;
}

pspmm_status pspmm_spmm_run(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K, float *d_C,
                            int64_t ldc, pspmm_config cfg, void *stream) {
  return pspmm::guarded("spmm_run", [&]() -> pspmm_status {
    return run_spmm(A, d_B, ldb, K, d_C, ldc, cfg, as_stream(stream));
  });
}

pspmm_status pspmm_spmm_accumulate(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K,
                                   float *d_C, int64_t ldc, pspmm_config cfg, void *stream) {
  return pspmm::guarded("spmm_accumulate", [&]() -> pspmm_status {
    return run_spmm(A, d_B, ldb, K, d_C, ldc, cfg, as_stream(stream), 1);
  });
}

pspmm_status pspmm_spmm_run_fanout(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K,
                                   float *d_C, int64_t ldc, float *const *h_peers, int32_t npeers,
                                   pspmm_config cfg, void *stream) {
  return pspmm::guarded("spmm_run_fanout", [&]() -> pspmm_status {
    if (npeers < 0 || npeers > PSPMM_MAX_PEERS || (npeers > 0 && !h_peers)) {
      set_error("spmm_run_fanout: npeers must be in 0..PSPMM_MAX_PEERS with a peer array");
      return PSPMM_ERR_INVALID_ARG;
    }
    Fanout fan{};
    fan.n = npeers;
    for (int d = 0; d < npeers; ++d) fan.peer[d] = h_peers[d];
    return run_spmm(A, d_B, ldb, K, d_C, ldc, cfg, as_stream(stream), 0, &fan);
  });
}

pspmm_status pspmm_spmm_run_multicast(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K,
                                      float *d_C, int64_t ldc, float *d_C_mc, pspmm_config cfg,
                                      void *stream) {
  return pspmm::guarded("spmm_run_multicast", [&]() -> pspmm_status {
    if (!d_C_mc) {
      set_error("spmm_run_multicast: null multicast address");
      return PSPMM_ERR_INVALID_ARG;
    }
    if ((reinterpret_cast<uintptr_t>(d_C_mc) & 15) != (reinterpret_cast<uintptr_t>(d_C) & 15)) {
      set_error("spmm_run_multicast: multicast address alignment differs from C's");
      return PSPMM_ERR_INVALID_ARG;
    }
    Fanout fan{};
    fan.n = 1;
    fan.mc = 1;
    fan.peer[0] = d_C_mc;
    return run_spmm(A, d_B, ldb, K, d_C, ldc, cfg, as_stream(stream), 0, &fan);
  });
}

pspmm_status pspmm_ipc_get_handle(const void *d_ptr, void *h_handle, int64_t *offset) {
  return pspmm::guarded("ipc_get_handle", [&]() -> pspmm_status {
    if (!d_ptr || !h_handle || !offset) {
      set_error("ipc_get_handle: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    CUdeviceptr base = 0;
    size_t size = 0;
    auto range = get_address_range();
    if (!range) {
      set_error("ipc_get_handle: cuMemGetAddressRange unavailable");
      return PSPMM_ERR_CUDA;
    }
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) {
      set_error("ipc_get_handle: not a device allocation");
      return PSPMM_ERR_INVALID_ARG;
    }
    cudaIpcMemHandle_t h;
    PSPMM_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
    memcpy(h_handle, &h, sizeof(h));
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return PSPMM_OK;
  });
}

pspmm_status pspmm_ipc_open(const void *h_handle, void **d_base) {
  return pspmm::guarded("ipc_open", [&]() -> pspmm_status {
    if (!h_handle || !d_base) {
      set_error("ipc_open: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, h_handle, sizeof(h));
    PSPMM_CUDA_TRY(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
    return PSPMM_OK;
  });
}

pspmm_status pspmm_ipc_close(void *d_base) {
  return pspmm::guarded("ipc_close", [&]() -> pspmm_status {
    if (!d_base) return PSPMM_OK;
    PSPMM_CUDA_TRY(cudaIpcCloseMemHandle(d_base));
    return PSPMM_OK;
  });
}

pspmm_status pspmm_spmm_run_host(pspmm_pcsr A, const float *h_B, int64_t ldb, int32_t K,
                                 float *h_C, int64_t ldc, pspmm_config cfg, float *d_Bbuf,
                                 float *d_Cbuf, void *stream) {
  return pspmm::guarded("spmm_run_host", [&]() -> pspmm_status {
    if (!A || !h_B || !h_C || !d_Bbuf || !d_Cbuf) {
      set_error("spmm_run_host: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (K < 1 || ldb < K || ldc < K) {
      set_error("spmm_run_host: need K >= 1, ldb >= K, ldc >= K");
      return PSPMM_ERR_DIM_MISMATCH;
    }
    return run_spmm_host(A, h_B, ldb, K, h_C, ldc, cfg, d_Bbuf, d_Cbuf, as_stream(stream));
  });
}

pspmm_status pspmm_spmm_run_host_batch(pspmm_pcsr A, const float *const *h_B, int64_t ldb,
                                       int32_t K, float *const *h_C, int64_t ldc, int32_t count,
                                       pspmm_config cfg, float *const *d_B, float *const *d_C,
                                       void *stream) {
  return pspmm::guarded("spmm_run_host_batch", [&]() -> pspmm_status {
    if (!A || !h_B || !h_C || !d_B || !d_C || count < 0) {
      set_error("spmm_run_host_batch: null argument or negative count");
      return PSPMM_ERR_INVALID_ARG;
    }
    for (int32_t i = 0; i < count; ++i)
      if (!h_B[i] || !h_C[i]) {
        set_error("spmm_run_host_batch: null host matrix");
        return PSPMM_ERR_INVALID_ARG;
      }
    for (int b = 0; b < 2; ++b)
      if (!d_B[b] || !d_C[b]) {
        set_error("spmm_run_host_batch: null device buffer");
        return PSPMM_ERR_INVALID_ARG;
      }
    if (K < 1 || ldb < K || ldc < K) {
      set_error("spmm_run_host_batch: need K >= 1, ldb >= K, ldc >= K");
      return PSPMM_ERR_DIM_MISMATCH;
    }
    return run_spmm_host_batch(A, h_B, ldb, K, h_C, ldc, count, cfg, d_B, d_C, as_stream(stream));
  });
}

pspmm_status pspmm_dense_gemm(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                              const float *d_W, int64_t ldw, float *d_T, int64_t ldt,
                              void *stream) {
  return pspmm::guarded("dense_gemm", [&]() -> pspmm_status {
    return dense_gemm(n, Ki, Ko, d_X, ldx, d_W, ldw, d_T, ldt, as_stream(stream));
  });
}

pspmm_status pspmm_gnn_layer(pspmm_pcsr A, const float *d_X, int64_t ldx, int32_t Ki,
                             const float *d_W, int64_t ldw, int32_t Ko, float *d_T, int64_t ldt,
                             float *d_Y, int64_t ldy, pspmm_config cfg, void *stream) {
  return pspmm::guarded("gnn_layer", [&]() -> pspmm_status {
    if (!A || !d_X || !d_W || !d_T || !d_Y) {
      set_error("gnn_layer: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (Ki < 1 || Ko < 1 || ldx < Ki || ldw < Ko || ldy < Ko || ldt < std::min(Ki, Ko)) {
      set_error("gnn_layer: need Ki, Ko >= 1, ldx >= Ki, ldw >= Ko, ldy >= Ko, ldt >= min(Ki, Ko)");
      return PSPMM_ERR_DIM_MISMATCH;
    }
    cudaStream_t s = as_stream(stream);
    pspmm_status st;
    if (Ko <= Ki) {  // T = X . W (n_cols x Ko), Y = A . T: the SpMM runs on Ko columns
      st = dense_gemm(A->n_cols, Ki, Ko, d_X, ldx, d_W, ldw, d_T, ldt, s);
      if (st != PSPMM_OK) return st;
      return run_spmm(A, d_T, ldt, Ko, d_Y, ldy, cfg, s);
    }
    // T = A . X (n x Ki), Y = T . W: the SpMM runs on Ki columns
    st = run_spmm(A, d_X, ldx, Ki, d_T, ldt, cfg, s);
    if (st != PSPMM_OK) return st;
    return dense_gemm(A->n_rows, Ki, Ko, d_T, ldt, d_W, ldw, d_Y, ldy, s);
  });
}

pspmm_status pspmm_csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                 const int32_t *d_rowptr, const int32_t *d_colidx,
                                 const float *d_val, int32_t *d_t_rowptr, int32_t *d_t_colidx,
                                 float *d_t_val, void *stream) {
  return pspmm::guarded("csr_transpose", [&]() -> pspmm_status {
    return csr_transpose(n_rows, n_cols, nnz, d_rowptr, d_colidx, d_val, d_t_rowptr, d_t_colidx,
                         d_t_val, as_stream(stream));
  });
}

pspmm_status pspmm_csr_permute(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                               const int32_t *d_colidx, const float *d_val, const int32_t *d_perm,
                               int32_t *d_out_rowptr, int32_t *d_out_colidx, float *d_out_val,
                               void *stream) {
  return pspmm::guarded("csr_permute", [&]() -> pspmm_status {
    return csr_permute(n, nnz, d_rowptr, d_colidx, d_val, d_perm, d_out_rowptr, d_out_colidx,
                       d_out_val, as_stream(stream));
  });
}

pspmm_status pspmm_permute_rows(int64_t n, int32_t K, const float *d_in, int64_t ldi,
                                const int32_t *d_perm, float *d_out, int64_t ldo, int32_t inverse,
                                void *stream) {
  return pspmm::guarded("permute_rows", [&]() -> pspmm_status {
    return permute_rows(n, K, d_in, ldi, d_perm, d_out, ldo, inverse, as_stream(stream));
  });
}

pspmm_status pspmm_features_compute(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                                    const int32_t *d_colidx, int32_t omega, void *stream,
                                    pspmm_features *out) {
  return pspmm::guarded("features_compute", [&]() -> pspmm_status {
    return compute_features(n, nnz, d_rowptr, d_colidx, omega, as_stream(stream), out);
  });
}

pspmm_status pspmm_pcsr_attach_dense(pspmm_pcsr A, const int32_t *d_rowptr,
                                     const int32_t *d_colidx, const float *d_val,
                                     double min_density, int32_t k_max, void *stream,
                                     int64_t *out_tiles) {
  return pspmm::guarded("pcsr_attach_dense", [&]() -> pspmm_status {
    return attach_dense(A, d_rowptr, d_colidx, d_val, min_density, k_max, as_stream(stream),
                        out_tiles);
  });
}

pspmm_status pspmm_decide_dense(pspmm_pcsr A, int32_t K, double min_frac, pspmm_config *cfg) {
  return pspmm::guarded("decide_dense", [&]() -> pspmm_status {
    if (!A || !cfg || K < 1 || !(min_frac >= 0.0 && min_frac <= 1.0)) {
      set_error("decide_dense: null argument, K < 1 or min_frac outside [0, 1]");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (A->dense && A->dense->num_tiles > 0 && K % 16 == 0 && K <= A->dense->k_max && A->nnz > 0 &&
        (double)A->dense->nnz_dense >= min_frac * (double)A->nnz) {
      cfg->mode = 1;
      // the rest is its own sparse matrix: the decider's mode-0 knobs for its
      // features (a TMA-gather label, mode 2, has no W / F / G for mode 0)
      pspmm_config rc{};
      if (A->dense->rest_f_ok && pspmm_decide_config(&A->dense->rest_f, K, &rc) == PSPMM_OK &&
          rc.mode != 2 && rc.F >= 1) {
        cfg->W = rc.W;
        cfg->F = rc.F;
        cfg->G = rc.G;
        cfg->order = rc.order;
      }
    } else if (cfg->mode == 1)
      cfg->mode = 0;
    return PSPMM_OK;
  });
}

pspmm_status pspmm_pcsr_dense_info(pspmm_pcsr A, int64_t *num_panels, int64_t *num_tiles,
                                   int64_t *nnz_dense) {
  return pspmm::guarded("pcsr_dense_info", [&]() -> pspmm_status {
    if (!A || !num_panels || !num_tiles || !nnz_dense) {
      set_error("pcsr_dense_info: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    *num_panels = A->dense ? A->dense->num_panels : 0;
    *num_tiles = A->dense ? A->dense->num_tiles : 0;
    *nnz_dense = A->dense ? A->dense->nnz_dense : 0;
    return PSPMM_OK;
  });
}

pspmm_status pspmm_block_reuse(pspmm_pcsr A, void *stream, double *reuse) {
  return pspmm::guarded("block_reuse", [&]() -> pspmm_status {
    return block_reuse(A, as_stream(stream), reuse, nullptr);
  });
}

pspmm_status pspmm_pcsr_attach_blocks(pspmm_pcsr A, void *stream, int64_t *out_windows) {
  return pspmm::guarded("pcsr_attach_blocks", [&]() -> pspmm_status {
    pspmm_status st = attach_blocks(A, as_stream(stream));
    if (st == PSPMM_OK && out_windows) *out_windows = A->blocks->num_windows;
    return st;
  });
}

pspmm_status pspmm_block_info(pspmm_pcsr A, int32_t *block_rows, int64_t *windows) {
  return pspmm::guarded("block_info", [&]() -> pspmm_status {
    if (!A || !block_rows || !windows) {
      set_error("block_info: null argument");
      return PSPMM_ERR_INVALID_ARG;
    }
    *block_rows = A->blocks ? A->blocks->nw * A->blocks->rw : 0;
    *windows = A->blocks ? A->blocks->num_windows : 0;
    return PSPMM_OK;
  });
}

pspmm_status pspmm_pcsr_attach_band(pspmm_pcsr A, int32_t k_max, void *stream,
                                    double *staged_frac) {
  return pspmm::guarded("pcsr_attach_band", [&]() -> pspmm_status {
    return attach_band(A, k_max, as_stream(stream), staged_frac);
  });
}

pspmm_status pspmm_decide_blocks(pspmm_pcsr A, int32_t K, double min_reuse, pspmm_config *cfg) {
  return pspmm::guarded("decide_blocks", [&]() -> pspmm_status {
    if (!A || !cfg || K < 1 || !(min_reuse >= 0.0)) {
      set_error("decide_blocks: null argument, K < 1 or min_reuse < 0");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (A->blocks && A->V == 1 && A->S == 0 && K % 128 == 0 && A->nnz > 0 &&
        A->blocks->reuse >= min_reuse)
      cfg->mode = 5;
    else if (cfg->mode == 5)
      cfg->mode = 0;
    return PSPMM_OK;
  });
}

}  // extern "C"
