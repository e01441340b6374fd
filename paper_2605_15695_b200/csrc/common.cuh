// Internal declarations of libpspmm.so (not part of the ABI; see include/pspmm.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "guard.h"
#include "pspmm.h"

// The PCSR handle: rowPtr / colIdx / val / TRow on the device, plus
// derived data that is NOT part of the bit-exact PCSR contract:
//   d_split  = ids of panels that own more than one chunk (S = 1); their C
//              rows are zeroed before the chunks accumulate into them.
//   slice_*  = kSlices + 1 unit / row bounds at panel boundaries, used by the
//              host entry to overlap the D2H copy of C with the engine.
constexpr int kSlices = 8;
struct pspmm_pcsr_s;
// Engine mode 1 (spmm_dense.cu): the dense 128 x 32 tiles of A and a PCSR of
// the remaining nonzeros, attached by pspmm_pcsr_attach_dense.
struct DenseTiles {
  int64_t num_panels = 0, num_tiles = 0, nnz_dense = 0, kgroups = 0;
  int32_t k_max = 0;
  float *d_tiles = nullptr;        // num_tiles x (TF32 hi 4096, lo 4096), smem image order
  float4 *d_bhi = nullptr;         // kgroups x k_max: per-run TF32 hi / lo images of B
  float4 *d_blo = nullptr;
  int32_t *d_panel_ptr = nullptr;  // num_panels + 1
  int32_t *d_panel = nullptr;      // num_panels: 128-row panel index
  int32_t *d_tile_col = nullptr;   // num_tiles: first column of the tile
  pspmm_pcsr_s *rest = nullptr;    // A minus the dense tiles (same V, S, omega)
  pspmm_features rest_f{};         // Table-3 features of the rest
  bool rest_f_ok = false;
};
// Engine mode 5 (spmm_block.cu): rows in blocks of nw x rw rows (nw
// consumer warps of rw rows: 23 x 8 by default, 19 x 8, 15 x 8 or 15 x 16
// for A/B); each block's touched windows of
// kBlockWindow B rows, split into "virtual windows" of at most
// kBlockMaxPairs nonzeros; per virtual window its nonzeros packed warp by
// warp, slot by slot (one bulk copy stages them), attached by
// pspmm_pcsr_attach_blocks.  Derived data, not part of the PCSR contract.
constexpr int kBlockWindow = 128;     // B rows per staged window
constexpr int kBlockRw = 8;           // default rows per consumer warp
constexpr int kBlockNw = 23;          // default consumer warps (8 x 23 = 184-row blocks)
constexpr int kBlockMaxPairs = 1408;  // nonzeros staged per virtual window (11 KB)
constexpr int kReuseRows = 128;       // row-block height of the reuse feature
struct RowBlocks {
  int64_t num_blocks = 0, num_windows = 0, num_virtual = 0;
  int32_t rw = 8;                  // rows per consumer warp
  int32_t nw = 23;                 // consumer warps; block rows = nw * rw
  double reuse = 0.0;              // nnz / (touched windows x kBlockWindow)
  int32_t *d_win_ptr = nullptr;    // num_blocks + 1: virtual-window range of each block
  int32_t *d_win_c0 = nullptr;     // num_virtual: first B row of the window
  int64_t *d_win_pbase = nullptr;  // num_virtual + 1: first packed pair (even: 16-B aligned)
  uint8_t *d_win_cnt = nullptr;    // num_virtual x nw x rw: per (window, warp, slot) count
  uint16_t *d_win_woff = nullptr;  // num_virtual x nw: a warp's first pair in the window
  int2 *d_pairs = nullptr;         // (column - window start, value bits), windows padded to even
  int16_t *d_rowmap = nullptr;     // num_blocks x nw x rw: local row of a slot, -1 = none
};
// Engine mode 6 (spmm_band.cu): rows in blocks of 128 / 64 / 32 / 16 (by k_max);
// per block a descriptor, the contiguous ranges of B rows it touches (staged
// by bulk copies) and every nonzero's (band slot, value) pair, attached by
// pspmm_pcsr_attach_band.  Derived data, not part of the PCSR contract.
constexpr int kBandBytes = 32 * 1024;  // staged band budget per block (6 CTAs per SM)
constexpr int kBandMaxK = 128;
struct Band {
  int64_t num_blocks = 0;
  int32_t k_max = 0, rows = 0;      // rows per block
  double staged_frac = 0.0;         // non-empty blocks whose band fits the budget
  int4 *d_desc = nullptr;           // num_blocks: {first range, ranges, p0, p1}
  int32_t *d_staged = nullptr;      // num_blocks: staged rows (-1 over budget, 0 empty)
  int4 *d_rng = nullptr;            // ranges: {first B row, rows, band slot, 0}
  int2 *d_pairs = nullptr;          // nnz + 2: (band slot or column, value bits)
  int32_t *d_rowptr = nullptr;      // n + 65: padded copy of rowPtr
};
struct pspmm_pcsr_s {
  int64_t n_rows = 0, n_cols = 0, num_panels = 0, nnz = 0, nnz_v = 0, num_chunks = 0;
  int64_t sg = 0, rowptr_len = 0, num_split = 0;
  int32_t V = 1, S = 0, omega = 32;
  double pr = 0.0, sr = 1.0;
  int32_t *d_rowptr = nullptr;  // rowptr_len
  int32_t *d_colidx = nullptr;  // nnz_v
  float *d_val = nullptr;       // nnz_v * V
  int32_t *d_trow = nullptr;    // num_chunks (S = 1)
  int32_t *d_split = nullptr;   // num_split (S = 1)
  int32_t *d_order = nullptr;   // num_chunks unit ids by descending vector count (engine schedule)
  int64_t slice_units[kSlices + 1] = {};
  int64_t slice_rows[kSlices + 1] = {};
  cudaStream_t copy_stream = nullptr;  // created lazily by pspmm_spmm_run_host
  cudaEvent_t slice_done[kSlices] = {};
  int64_t max_unit_len = 0;            // vectors of the longest unit (load-balance check)
  // pspmm_spmm_run_host_batch: copy-in / copy-out streams and per-buffer events
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t h2d_done[2] = {}, comp_done[2] = {}, d2h_done[2] = {}, batch_start = nullptr;
  DenseTiles *dense = nullptr;         // engine mode 1 (pspmm_pcsr_attach_dense)
  RowBlocks *blocks = nullptr;         // engine mode 5 (pspmm_pcsr_attach_blocks)
  Band *band = nullptr;                // engine mode 6 (pspmm_pcsr_attach_band)
};

namespace pspmm {

void set_error(const std::string &msg);
pspmm_status cuda_status(cudaError_t e, const char *where);

#define PSPMM_CUDA_TRY(expr)                                      \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return ::pspmm::cuda_status(_e, #expr); \
  } while (0)

#define PSPMM_FAIL(code, msg)          \
  do {                                 \
    ::pspmm::set_error(msg);           \
    return code;                       \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

inline int64_t l2_bytes() {
  static int64_t l2 = 0;
  if (!l2) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
    l2 = v > 0 ? v : (int64_t)126 << 20;
  }
  return l2;
}

// validate.cu
pspmm_status validate_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                          const int32_t *d_colidx, cudaStream_t stream);

// pcsr_build.cu
pspmm_status build_pcsr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                        const int32_t *d_colidx, const float *d_val, int32_t V, int32_t S,
                        int32_t omega, int32_t sg_override, cudaStream_t stream,
                        pspmm_pcsr_s *P);
// engine schedule: d_order = unit ids by descending vector count (derived)
pspmm_status build_unit_order(pspmm_pcsr_s *A, cudaStream_t stream);
// per-panel vector counts |union_p| for V = 2 (shared with features.cu)
pspmm_status panel_counts_v2(int64_t n_rows, const int32_t *d_rowptr, const int32_t *d_colidx,
                             int32_t *d_L, cudaStream_t stream);

// Output fan-out (f2, pspmm_spmm_run_fanout): every C element the engine
// writes is also written, at the same offset, to each peer buffer (device
// pointers this device can store to, e.g. CUDA-IPC-mapped peer memory), and
// each CTA ends with a system-scope fence.  Passed by value in kernel args.
constexpr int kMaxPeers = PSPMM_MAX_PEERS;
struct Fanout {
  float *peer[kMaxPeers];
  int32_t n;
  // mc = 1 (NVLS, f2 i): peer[0] is the multicast address of C (NVLink
  // SHARP / NVSwitch multicast object every rank's copy is bound to) and
  // n = 1: each C write is ONE multimem store (or reduction) that the switch
  // delivers to every bound copy, the local one included, instead of the
  // local write plus n unicast peer stores.
  int32_t mc;
};
#ifdef __CUDACC__
__device__ __forceinline__ void mc_st(float *p, const float4 &v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_st(float *p, const float &v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void mc_red(float *p, const float4 &v) {
  asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_red(float *p, const float &v) {
  asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// The store epilogue of the row-owning engines (modes 3, 5, 6): C[off] = v
// (v already includes C's old value when accumulating), fanned out.
__device__ __forceinline__ void fan_store4(float *C, const Fanout &fan, int64_t off,
                                           const float4 &v) {
  if (fan.mc) {
    mc_st(fan.peer[0] + off, v);
    return;
  }
  __stcs(reinterpret_cast<float4 *>(C + off), v);
#pragma unroll 1
  for (int d = 0; d < fan.n; ++d) __stcs(reinterpret_cast<float4 *>(fan.peer[d] + off), v);
}
#endif

// spmm_dense.cu (engine mode 1)
bool dense_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                     const float *d_C);
pspmm_status run_spmm_dense(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                            int32_t accumulate);
pspmm_status attach_dense(pspmm_pcsr_s *A, const int32_t *d_rowptr, const int32_t *d_colidx,
                          const float *d_val, double min_density, int32_t k_max,
                          cudaStream_t stream, int64_t *out_tiles);
void destroy_dense(DenseTiles *D);

// spmm_block.cu (engine mode 5)
pspmm_status block_reuse(const pspmm_pcsr_s *A, cudaStream_t stream, double *reuse,
                         int64_t *touched);
pspmm_status attach_blocks(pspmm_pcsr_s *A, cudaStream_t stream);
void destroy_blocks(RowBlocks *B);
bool block_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc,
                     const float *d_B, const float *d_C);
pspmm_status run_spmm_block(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, cudaStream_t stream, int32_t accumulate,
                            const Fanout &fan);

// spmm_band.cu (engine mode 6)
void destroy_band(Band *D);
pspmm_status attach_band(pspmm_pcsr_s *A, int32_t k_max, cudaStream_t stream, double *staged_frac);
bool band_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                    const float *d_C);
pspmm_status run_spmm_band(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                           float *d_C, int64_t ldc, cudaStream_t stream, int32_t accumulate,
                           const Fanout &fan);

// spmm.cu
pspmm_status run_spmm(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K, float *d_C,
                      int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                      int32_t accumulate = 0, const Fanout *fan = nullptr);

// spmm_tma.cu (engine mode 2)
bool tma_supported(int32_t K, int64_t ldb, int64_t ldc, const float *d_B, const float *d_C);
pspmm_status run_spmm_tma(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                          float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                          int64_t u0, int64_t u1, int32_t accumulate, const Fanout &fan);
// spmm_short.cu (engine mode 3)
bool short_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                     const float *d_C, const pspmm_config &cfg);
pspmm_status run_spmm_short(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                            int64_t u0, int64_t u1, int32_t accumulate, const Fanout &fan);
// host entry: H2D(B), engine in kSlices unit slices, D2H of each slice's C
// rows on a second stream as soon as the slice is done
pspmm_status run_spmm_host(pspmm_pcsr_s *A, const float *h_B, int64_t ldb, int32_t K, float *h_C,
                           int64_t ldc, const pspmm_config &cfg, float *d_Bbuf, float *d_Cbuf,
                           cudaStream_t stream);
// host batch entry: count independent B -> C products through two device
// buffer sets, H2D of i + 1 and D2H of i - 1 overlapping the engine on i
pspmm_status run_spmm_host_batch(pspmm_pcsr_s *A, const float *const *h_B, int64_t ldb, int32_t K,
                                 float *const *h_C, int64_t ldc, int32_t count,
                                 const pspmm_config &cfg, float *const *d_B, float *const *d_C,
                                 cudaStream_t stream);

// gnn_layer.cu (f3: the dense product of a GNN layer)
// spmm_block.cu: cuTensorMapEncodeTiled (PFN_cuTensorMapEncodeTiled_v12000),
// nullptr when the driver lacks it
void *tensor_map_encoder();
// gemm_tc.cu (f3 dense product on tcgen05, 3xTF32)
bool gemm_tc_supported(int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx, const float *d_W,
                       int64_t ldw, const float *d_T, int64_t ldt);
pspmm_status gemm_tc(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                     const float *d_W, int64_t ldw, float *d_T, int64_t ldt, cudaStream_t stream);
pspmm_status dense_gemm(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                        const float *d_W, int64_t ldw, float *d_T, int64_t ldt,
                        cudaStream_t stream);

// transpose.cu (f3: backward SpMM operand)
pspmm_status csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                           const int32_t *d_colidx, const float *d_val, int32_t *d_t_rowptr,
                           int32_t *d_t_colidx, float *d_t_val, cudaStream_t stream);

// permute.cu (f1: applying a reordering)
pspmm_status csr_permute(int64_t n, int64_t nnz, const int32_t *d_rowptr, const int32_t *d_colidx,
                         const float *d_val, const int32_t *d_perm, int32_t *d_out_rowptr,
                         int32_t *d_out_colidx, float *d_out_val, cudaStream_t stream);
pspmm_status permute_rows(int64_t n, int32_t K, const float *d_in, int64_t ldi,
                          const int32_t *d_perm, float *d_out, int64_t ldo, int32_t inverse,
                          cudaStream_t stream);

// features.cu
pspmm_status compute_features(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                              const int32_t *d_colidx, int32_t omega, cudaStream_t stream,
                              pspmm_features *out);

}  // namespace pspmm
