/*
 * pspmm.h — C ABI of the B200-native ParamSpMM hot path (libpspmm.so).
 *
 * The operation is the paper's SpMM  A_{n x n} . B_{n x dim} = C_{n x dim}
 * (arXiv 2605.15695) with A held in Parameterized CSR
 * (PCSR) and computed by a parametric engine configured by
 * <W, F, V, S> (Alg. 2).  The three-phase workflow of P:192
 * maps onto the calls below:
 *   phase 1  configuration prediction : pspmm_features_compute + pspmm_decide_config
 *   phase 2  PCSR generation          : pspmm_pcsr_build
 *   phase 3  SpMM computing           : pspmm_spmm_run
 * plus the row-shard helpers of the multi-GPU path.
 *
 * Conventions (apply to every call):
 *  - Every call returns pspmm_status (0 == PSPMM_OK); no C++ exception ever
 *    crosses the ABI.  pspmm_last_error() returns a thread-local message for
 *    the most recent failure on the calling thread.
 *  - "d_" pointers are CUDA device pointers (global memory of the current
 *    device); "h_" pointers are host pointers.  `stream` is a cudaStream_t
 *    passed as void* (NULL = the legacy default stream).
 *  - Sparse matrices at the boundary are canonical CSR:
 *    int32 rowPtr[n+1] with rowPtr[0] = 0, rowPtr[n] = nnz, non-decreasing;
 *    int32 colIdx[nnz] strictly increasing inside each row, 0 <= col < n;
 *    fp32 val[nnz].  A is square.
 *  - Dense matrices are fp32 row-major with a leading dimension (ld >= K).
 *    B is n x K (ldb), C is n x K (ldc).  The 128-bit path needs K % 4 == 0,
 *    ld % 4 == 0 and 16-byte aligned B and C; otherwise the same engine runs
 *    a masked scalar variant (correct, slower).  There is no CPU fallback.
 *  - Memory passed in is caller-owned; the library never frees it.  A PCSR
 *    handle owns its own device arrays until pspmm_pcsr_destroy.
 *  - Indices are int32: n, nnz and nnz_V must be < 2^31 (else
 *    PSPMM_ERR_UNSUPPORTED).
 */
#ifndef PSPMM_H
#define PSPMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PSPMM_OK = 0,
  PSPMM_ERR_INVALID_ARG = 1,     /* null pointer, negative size, bad omega ... */
  PSPMM_ERR_NOT_CANONICAL = 2,   /* CSR violates the preconditions above */
  PSPMM_ERR_DIM_MISMATCH = 3,    /* K < 1 or ld < K */
  PSPMM_ERR_CONFIG = 4,          /* config outside its domain */
  PSPMM_ERR_CONFIG_MISMATCH = 5, /* cfg.V / cfg.S / cfg.omega differ from the handle's */
  PSPMM_ERR_EMPTY = 6,           /* features / SG undefined because nnz == 0 */
  PSPMM_ERR_UNSUPPORTED = 7,     /* sizes beyond int32 indexing, unsupported mode */
  PSPMM_ERR_OOM = 8,             /* device allocation failed */
  PSPMM_ERR_CUDA = 9             /* any other CUDA runtime error */
} pspmm_status;

/*
 * <W, F, V, S> of P:173 plus the build-specific knobs.
 *  W  warps per CTA: 1, 2, 4 or 8.
 *  F  thread-coarsening factor, in B200 units: the number of
 *     128-bit (4 x fp32) accumulators a lane keeps per output row, i.e. a
 *     row group covers 4.G.F columns of C per pass.  1 .. 8.
 *  V  vector size of vectorized blocking: 1 or 2.
 *  S  workload balancing flag: 0 or 1.
 *  omega  warp width used by Eq. 3; 32 on the device.  Other
 *     values are accepted (>= 1) so small traces can be reproduced.
 *  sg_override  0 = Split Granularity from Eq. 3; > 0 forces SG (c-18).
 *  G  lanes per row group (1, 2, 4, 8, 16, 32); 0 = derived from K and F
 *     as the smallest power of two with 4.G.F >= K (capped at 32).
 *  mode  0 = CUDA-core engine, B rows gathered with 128-bit loads into
 *     registers (any K, any layout; W, F, G apply);
 *     2 = CUDA-core engine, B rows gathered by TMA tile::gather4 into a
 *     shared-memory ring per warp (needs K % 32 == 0, ld % 4 == 0, 16-B
 *     aligned B and C, else PSPMM_ERR_UNSUPPORTED; only W applies);
 *     3 = short-row pipeline for low-degree graphs (V = 1, S = 0, F in
 *     {1, 2, 4}, 128-bit layout; W, F, G apply);
 *     (4: retired in round 2 -- a cp.async short-row stream that was slower
 *     than mode 3 on every workload and never selected; PSPMM_ERR_UNSUPPORTED)
 *     5 = row blocks with shared-memory B reuse (pspmm_pcsr_attach_blocks;
 *     V = 1, S = 0, K % 128 == 0; W, F, G, order do not apply);
 *     1 = dense-panel tensor-core path: the dense 128 x 32 tiles attached by
 *     pspmm_pcsr_attach_dense run on tcgen05 (kind::tf32, 3xTF32 split,
 *     fp32 accumulators in TMEM), the remaining nonzeros on the mode-0
 *     engine (W, F, G, order apply to it); needs an attached split (else
 *     PSPMM_ERR_UNSUPPORTED), K % 16 == 0, ld % 4 == 0, 16-B aligned B and
 *     C; not with the fan-out entry (the host entries run it whole,
 *     without slices).
 *  order  mode 0 only: 1 = visit units by descending vector count (a
 *     schedule built with the PCSR; helps skewed, shuffled graphs, hurts
 *     locality-ordered ones), 0 = in storage order.
 * For pspmm_pcsr_build only V, S, omega and sg_override matter.
 */
typedef struct {
  int32_t W, F, V, S;
  int32_t omega;
  int32_t sg_override;
  int32_t G;
  int32_t mode;
  int32_t order;
} pspmm_config;

typedef struct pspmm_pcsr_s *pspmm_pcsr; /* opaque, immutable after build */

/* PCSR sizes and the metrics of Eq. 2 / Eq. 4. */
typedef struct {
  int64_t n;          /* rows of A (and of B, C) */
  int64_t num_panels; /* ceil(n / V) */
  int64_t nnz;        /* nonzeros of A */
  int64_t nnz_v;      /* nonzero vectors (len(colIdx)); len(val) = nnz_v * V */
  int64_t num_chunks; /* S = 1: chunks = len(TRow) = len(rowPtr) - 1; S = 0: num_panels */
  int64_t sg;         /* split granularity used (S = 1), else 0 */
  int32_t V, S, omega, reserved;
  double pr;          /* PR_V = 1 - nnz / (nnz_V V)   (Eq. 2); NaN when nnz_v == 0 */
  double sr;          /* SR = (chunks + 1) / (panels + 1)  (Eq. 4, c-4a); 1 when S = 0 */
} pspmm_pcsr_info;

/* The 16 Table-3 features, readings c-19 .. c-22 of DESIGN.md §3. */
typedef struct {
  double n, n_hat, nnz, delta, d, d_hat, d_max, cv, cv_hat, sr1, sr2, rho, b, b_max, pr1, pr2;
} pspmm_features;

/* Human-readable name of a status code (static storage). */
const char *pspmm_status_string(pspmm_status s);

/* Message of the last failing call on this thread ("" if none). */
const char *pspmm_last_error(void);

/* Library version string, e.g. "pspmm 0.1 sm_100a". */
const char *pspmm_version(void);

/*
 * (a1) CSR intake check on the device: the canonical-CSR preconditions
 * listed above.  Synchronises `stream` once to read the verdict.
 * Returns PSPMM_OK or PSPMM_ERR_NOT_CANONICAL (or INVALID_ARG / CUDA).
 */
pspmm_status pspmm_csr_validate(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                                const int32_t *d_colidx, void *stream);

/* Same check for an n_rows x n_cols CSR (0 <= col < n_cols). */
pspmm_status pspmm_csr_validate_rect(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                     const int32_t *d_rowptr, const int32_t *d_colidx,
                                     void *stream);

/*
 * (a4, a5) PCSR generation: vectorized blocking of A into
 * ceil(n/V) panels of V x 1 nonzero vectors (ascending column order,
 * +0.0f padding), then, if S == 1, the nonzero-split
 * balancing of Eq. 3 (each panel's run cut into max(1, ceil(L/SG)) chunks,
 * rowPtr reassigned, TRow[c] = source panel).  The integer arrays and the
 * copied values are bit-identical to the oracle's (oracle/oracle.c).
 * Validates the CSR first (pspmm_csr_validate).  V in {1, 2}; S in {0, 1};
 * omega >= 1; sg_override >= 0 (0 = Eq. 3).  nnz == 0 with S == 1 and
 * sg_override == 0 returns PSPMM_ERR_EMPTY (SG undefined).
 * Allocates the handle's device arrays; synchronises `stream` (sizes).
 * On success *out holds a new handle; on failure *out is NULL.
 */
pspmm_status pspmm_pcsr_build(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                              const int32_t *d_colidx, const float *d_val, int32_t V,
                              int32_t S, int32_t omega, int32_t sg_override, void *stream,
                              pspmm_pcsr *out);

/*
 * Same as pspmm_pcsr_build for a rectangular n_rows x n_cols CSR (columns
 * checked against n_cols).  Used for the row shards of the multi-GPU path,
 * whose columns index the all-gathered B (pspmm_shard_extract).  B then has
 * n_cols rows and C has n_rows rows.
 */
pspmm_status pspmm_pcsr_build_rect(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                   const int32_t *d_rowptr, const int32_t *d_colidx,
                                   const float *d_val, int32_t V, int32_t S, int32_t omega,
                                   int32_t sg_override, void *stream, pspmm_pcsr *out);

/* Sizes and metrics of a handle. */
pspmm_status pspmm_pcsr_get_info(pspmm_pcsr A, pspmm_pcsr_info *out);

/*
 * Copy the four PCSR arrays to host memory (for bit-exact checks).
 * h_rowptr: num_chunks + 1 int32 (S = 1) or num_panels + 1 (S = 0);
 * h_colidx: nnz_v int32; h_val: nnz_v * V fp32; h_trow: num_chunks int32
 * (S = 1 only; may be NULL when S = 0).  Any pointer may be NULL to skip
 * that array.  Synchronous.
 */
pspmm_status pspmm_pcsr_export(pspmm_pcsr A, int32_t *h_rowptr, int32_t *h_colidx,
                               float *h_val, int32_t *h_trow);

/*
 * (f4) PCSR binary file: little-endian; header = magic "PCSR",
 * u32 version (1), u64 n, u64 numPanels, u64 nnzV, u8 V, u8 S, u16 omega —
 * the SPEC's fields in its order — then the version-1 extension u32 0,
 * u64 numChunks, u64 SG, u64 nnz, u64 nCols (72-byte header), then rowPtr
 * u64[numChunks + 1], colIdx u32[nnzV], val f32[nnzV * V] and, iff S = 1,
 * TRow u32[numChunks].  Byte offsets in csrc/pcsr_io.cu.
 * save: copies the handle's arrays to the host and writes `path`
 * (synchronous).  load: reads, validates every PCSR invariant (rowPtr
 * monotone 0..nnzV, ascending in-range columns per panel, TRow covering each
 * panel in order, chunks <= SG cut at multiples of SG) and builds a handle
 * usable by pspmm_spmm_run (the engine's derived data is rebuilt on
 * `stream`).  Errors: INVALID_ARG (I/O, magic, header), UNSUPPORTED (other
 * version), NOT_CANONICAL (array invariants), OOM / CUDA.
 */
pspmm_status pspmm_pcsr_save(pspmm_pcsr A, const char *path);
pspmm_status pspmm_pcsr_load(const char *path, void *stream, pspmm_pcsr *out);

/* Release a handle and its device arrays (NULL is a no-op). */
void pspmm_pcsr_destroy(pspmm_pcsr A);

/*
 * (a6, a7) C = A . B (beta = 0) with the computing engine of Alg. 2
 * configured by cfg: every output row of C is overwritten.
 * cfg.V / cfg.S / cfg.omega must equal the handle's (else
 * PSPMM_ERR_CONFIG_MISMATCH).  Asynchronous on `stream`; allocates nothing,
 * so it can be captured in a CUDA graph.  With S = 1 the rows of split
 * panels are zeroed by a small pre-kernel and accumulated with vector
 * atomics (the accumulation order is then non-deterministic, c-23).
 * Any K >= 1.  nnz_v == 0 writes zeros.
 */
pspmm_status pspmm_spmm_run(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K, float *d_C,
                            int64_t ldc, pspmm_config cfg, void *stream);

/*
 * C += A . B (beta = 1): same engines and config rules as pspmm_spmm_run,
 * but every C element is read and accumulated (sole-owner stores read
 * first; split-panel chunks accumulate with vector atomics as usual and
 * nothing is zeroed).  Used by the multi-GPU path to add the remote-column
 * block of a row shard onto its local-column block.
 * Asynchronous; allocates nothing.
 */
pspmm_status pspmm_spmm_accumulate(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K,
                                   float *d_C, int64_t ldc, pspmm_config cfg, void *stream);

/*
 * (a6, conditional: SURVEY §8 a6 "dense-panel variant") Split A for engine
 * mode 1.  The paper's blocking groups rows into panels so a
 * B row serves several rows; where a 128-row panel is dense over a column
 * range the product is a real dense contraction.  (d_rowptr, d_colidx,
 * d_val) must be the CSR A was built from (device, caller-owned, read
 * only; validated, and nnz must match).  Every 128 x 32 tile (rows
 * [128p, 128p + 128), columns [32t, 32t + 32)) holding at least
 * ceil(min_density * 4096) nonzeros is stored densely inside the handle;
 * the other nonzeros get a PCSR of their own (the handle's V, S, omega;
 * SG from Eq. 3).  The split also holds scratch for the per-run TF32
 * images of B (2 x 16 bytes x n_cols x k_max, rounded up), so mode-1 runs
 * allocate nothing; they accept K <= k_max.  Replaces a previous split;
 * freed by pspmm_pcsr_destroy.  min_density in (0, 1] and k_max a positive
 * multiple of 16, else INVALID_ARG.  *out_tiles (may be NULL) =
 * number of dense tiles.  Runs on the host; synchronises `stream`.  The
 * bit-exact PCSR arrays of A are untouched.
 */
pspmm_status pspmm_pcsr_attach_dense(pspmm_pcsr A, const int32_t *d_rowptr,
                                     const int32_t *d_colidx, const float *d_val,
                                     double min_density, int32_t k_max, void *stream,
                                     int64_t *out_tiles);

/*
 * Mode-1 decision (host, pure given the handle): cfg->mode = 1 iff a split
 * is attached, it has dense tiles, K % 16 == 0 and the tiles hold at least
 * min_frac of A's nonzeros; otherwise a mode of 1 is reset to 0 and any
 * other mode is left alone.  When it switches to mode 1 it also sets the
 * knobs the rest runs with (W, F, G, order) to pspmm_decide_config's pick
 * for the rest's own Table-3 features (computed by pspmm_pcsr_attach_dense;
 * kept as given when unavailable or when that pick is a mode-2 label).
 * min_frac in [0, 1] else INVALID_ARG.
 */
pspmm_status pspmm_decide_dense(pspmm_pcsr A, int32_t K, double min_frac, pspmm_config *cfg);

/*
 * (a6: the paper's blocking "to exploit B's data reuse through registers or
 * shared memory", §3.1) Engine mode 5: row blocks with
 * shared-memory B reuse.  Rows are grouped in blocks of nw x rw rows (nw
 * consumer warps of rw rows each; 23 x 8 = 184 rows by default); each block's
 * columns are cut into windows of 128 B rows, and a CTA stages every window
 * its block touches (128 B rows x 128 columns of B, one 2-D TMA copy) into
 * shared memory once, then all the block's nonzeros in that window read it
 * there instead of gathering their B row from L2.
 *
 * pspmm_block_reuse: the reuse that staging would capture, a graph feature
 * computed on the device from A's CSR order (V = 1, S = 0 handle, else
 * UNSUPPORTED) on fixed 128-row blocks: *reuse = nnz / (sum over 128-row
 * blocks of touched windows x 128), i.e. how many nonzeros read each staged
 * B row.  Synchronises `stream`.
 *
 * pspmm_pcsr_attach_blocks: build the mode-5 pack (host pass over A's CSR,
 * then uploaded; 8 B per nonzero + ~0.2 KB per touched window): per row
 * block a degree-balanced assignment of its rows to nw warps x rw slots, the
 * touched windows (split into virtual windows of at most 1408 nonzeros), and
 * the nonzeros reordered window by window, warp by warp, slot by slot (runs
 * padded to an even length).  Derived data: A's PCSR arrays are untouched; replaces a
 * previous pack; freed by pspmm_pcsr_destroy.  *out_windows (may be NULL) =
 * touched (block, window) pairs.  Synchronises `stream`.  UNSUPPORTED unless
 * V = 1, S = 0.
 *
 * pspmm_block_info: the attached pack's block height (rows per block) and
 * touched (block, window) pairs; zeros when no pack is attached.
 *
 * pspmm_decide_blocks (host, pure given the handle): cfg->mode = 5 iff a
 * pack is attached, K % 128 == 0 and its reuse >= min_reuse; otherwise a
 * mode of 5 is reset to 0 and any other mode is left alone.
 *
 * Mode-5 runs (pspmm_spmm_run / _accumulate / _fanout / the host entries,
 * which run it whole) need the pack, K % 128 == 0, ld % 4 == 0 and 16-B
 * aligned B and C, else PSPMM_ERR_UNSUPPORTED; W, F, G and order do not
 * apply.  Every C element has one writer (no atomics), so results are
 * deterministic run to run.
 */
pspmm_status pspmm_block_reuse(pspmm_pcsr A, void *stream, double *reuse);
pspmm_status pspmm_pcsr_attach_blocks(pspmm_pcsr A, void *stream, int64_t *out_windows);
pspmm_status pspmm_decide_blocks(pspmm_pcsr A, int32_t K, double min_reuse, pspmm_config *cfg);
pspmm_status pspmm_block_info(pspmm_pcsr A, int32_t *block_rows, int64_t *windows);

/*
 * (a6 on locality-ordered graphs: the paper's reordering step, P:271-272
 * §4.4, and its locality argument for blocking) Engine mode 6:
 * staged bands.  Rows are grouped in blocks of 128 / 64 / 32 / 16 rows
 * (k_max <= 16 / 32 / 64 / 128); each block's distinct
 * columns are merged into contiguous ranges of B rows (gaps of <= 8 rows
 * included), and a CTA stages the whole band with one 1-D bulk copy per
 * range into shared memory before any row is computed, while its rows'
 * (slot, value) pairs load into registers; every nonzero then reads its B
 * row from shared memory.  No per-nonzero dependent global gather remains
 * on the critical path.
 *
 * pspmm_pcsr_attach_band: build the pack (host pass over A's CSR, then
 * uploaded; 4 B per nonzero + 8 B per range): per block the ranges and each
 * nonzero's row slot in the band.  k_max (multiple of 4, 4..128) bounds the
 * K and the B row pitch (ldb) of later runs: a block is staged when its band
 * fits 32 KB at k_max columns; other blocks keep the column and gather from
 * global memory.  *staged_frac (may be NULL) = staged / non-empty blocks.
 * Replaces a previous pack; freed by pspmm_pcsr_destroy.  Synchronises
 * `stream`.  UNSUPPORTED unless V = 1, S = 0; INVALID_ARG for a bad k_max.
 *
 * Mode-6 runs (pspmm_spmm_run / _accumulate / _fanout / the host entries,
 * which run it whole) need the pack, K % 4 == 0, K <= ldb <= k_max,
 * ldc % 4 == 0 and 16-B aligned B and C, else PSPMM_ERR_UNSUPPORTED; W, F, G
 * and order do not apply.  One writer per C element (deterministic).
 */
pspmm_status pspmm_pcsr_attach_band(pspmm_pcsr A, int32_t k_max, void *stream,
                                    double *staged_frac);


/* Sizes of the attached split (zeros when none): 128-row panels with dense
 * tiles, dense tiles, nonzeros inside them. */
pspmm_status pspmm_pcsr_dense_info(pspmm_pcsr A, int64_t *num_panels, int64_t *num_tiles,
                                   int64_t *nnz_dense);

/*
 * End-to-end variant for host-resident B and C (bench.py "e2e"): copies
 * h_B (n x K, ldb) into the caller's device staging buffer d_Bbuf (same
 * layout), runs the engine into d_Cbuf (ldc) in 8 slices of units cut at
 * panel boundaries, copies each slice's rows of C back into h_C on an
 * internal second stream as soon as that slice is done (so the D2H copy
 * overlaps the remaining compute), and synchronises `stream`.  h_B / h_C
 * should be pinned for the copies to be asynchronous.  The first call on a
 * handle creates its copy stream and events (released by destroy).
 */
pspmm_status pspmm_spmm_run_host(pspmm_pcsr A, const float *h_B, int64_t ldb, int32_t K,
                                 float *h_C, int64_t ldc, pspmm_config cfg, float *d_Bbuf,
                                 float *d_Cbuf, void *stream);

/*
 * Host batch entry (serving / a stream of feature matrices through one A):
 * count independent products C_i = A . B_i with host-resident h_B[i]
 * (n_cols x K, ldb) and h_C[i] (n x K, ldc), host ARRAYS of count host
 * pointers each.  Two caller-owned device buffer sets d_B[0..1] / d_C[0..1]
 * (host arrays of 2 device pointers, same layouts) rotate, so the H2D copy
 * of B_{i+1} and the D2H copy of C_{i-1} run on internal copy streams while
 * the engine computes product i on `stream` (whole matrix, unit order
 * honoured).  Synchronises `stream` at the end.  h_B / h_C should be pinned.
 * The first call on a handle creates its copy streams and events (released
 * by destroy).  Errors as pspmm_spmm_run, plus INVALID_ARG for null
 * pointers or count < 0.
 */
pspmm_status pspmm_spmm_run_host_batch(pspmm_pcsr A, const float *const *h_B, int64_t ldb,
                                       int32_t K, float *const *h_C, int64_t ldc, int32_t count,
                                       pspmm_config cfg, float *const *d_B, float *const *d_C,
                                       void *stream);

/*
 * (f2 (i): the all-gather fused into the SpMM epilogue)
 * C = A . B exactly as pspmm_spmm_run, and every C element the engine writes
 * (stores, split-panel atomics, the zeroing of split rows) is also written at
 * the same offset relative to each of d_peers[0 .. npeers) — device pointers
 * this device can store to (peer memory mapped with pspmm_ipc_open over
 * NVLink, or any other device buffer), each addressed with ldc like d_C.  In
 * the sharded layer chain d_C is this rank's slot of its own
 * next-layer B_full and d_peers are the same slot in every peer's B_full, so
 * the transfer is spread over the kernel's lifetime instead of following it.
 * Each CTA ends with a system-scope fence; the caller orders the peers'
 * subsequent reads with a barrier (stream-ordered, e.g. a one-element NCCL
 * all-reduce).  h_peers is a HOST array of npeers device pointers,
 * 0 <= npeers <= PSPMM_MAX_PEERS (else PSPMM_ERR_INVALID_ARG).  Asynchronous.
 */
#define PSPMM_MAX_PEERS 7
pspmm_status pspmm_spmm_run_fanout(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K,
                                   float *d_C, int64_t ldc, float *const *h_peers, int32_t npeers,
                                   pspmm_config cfg, void *stream);

/*
 * (f2 (i) over NVLS: SURVEY §8(f) f2 "NVLS multicast (multimem.st via
 * symmetric memory) fusing the allgather into the SpMM epilogue")
 * C = A . B with every C write issued as ONE multimem store (split-panel
 * atomics: one multimem reduction, their zeroing: multimem stores of 0) to
 * d_C_mc, the multicast address of d_C: an address of an NVSwitch multicast
 * object every rank's copy of the gathered next-layer buffer is bound to
 * (e.g. torch.distributed._symmetric_memory's multicast_ptr plus d_C's
 * offset in the buffer).  The switch delivers the value to every bound copy,
 * d_C's own memory included, so no separate local store and no per-peer
 * unicast stores are issued.  d_C is read only when the engine needs C's old
 * value (never for C = A.B).  Engine modes 0, 3, 5 and 6 (mode 1, 2:
 * PSPMM_ERR_UNSUPPORTED); same fences and barrier contract as
 * pspmm_spmm_run_fanout.  INVALID_ARG for a null d_C_mc or an alignment
 * differing from d_C's.  Asynchronous.
 */
pspmm_status pspmm_spmm_run_multicast(pspmm_pcsr A, const float *d_B, int64_t ldb, int32_t K,
                                      float *d_C, int64_t ldc, float *d_C_mc, pspmm_config cfg,
                                      void *stream);

/*
 * CUDA IPC plumbing for the fan-out (f2): export a device allocation made
 * with cudaMalloc (or any sub-range of one, as caching allocators hand out) as a 64-byte
 * handle, open a peer process's handle (peer access enabled lazily) and
 * close it.  pspmm_ipc_get_handle writes 64 bytes to h_handle and the byte
 * offset of d_ptr inside its allocation to *offset (the handle names the
 * whole allocation); the opener adds that offset.  A handle cannot be opened
 * in the process that exported it (CUDA IPC rule) -> PSPMM_ERR_CUDA.
 */
pspmm_status pspmm_ipc_get_handle(const void *d_ptr, void *h_handle, int64_t *offset);
pspmm_status pspmm_ipc_open(const void *h_handle, void **d_base);
pspmm_status pspmm_ipc_close(void *d_base);

/*
 * (f3) CSR of A^T on the device, for the backward SpMM of a GNN layer
 * (dL/dB = A^T . dL/dC).  A is n_rows x n_cols
 * canonical CSR; the outputs are caller-allocated device arrays:
 * d_t_rowptr[n_cols + 1], d_t_colidx[nnz], d_t_val[nnz].  Rows of A^T hold
 * A's row indices in ascending order (a stable sort by column), so the
 * result is canonical and deterministic.  Validates A first; synchronises
 * `stream`.
 */
pspmm_status pspmm_csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                 const int32_t *d_rowptr, const int32_t *d_colidx,
                                 const float *d_val, int32_t *d_t_rowptr, int32_t *d_t_colidx,
                                 float *d_t_val, void *stream);

/*
 * (f3) Dense product of a GNN layer: T = X . W, fp32 in and out.  X: n x Ki
 * (ldx), W: Ki x Ko (ldw), T: n x Ko (ldt), all row-major device fp32.
 * When Ki % 32 == 0, Ko % 16 == 0, ld % 4 == 0 and X / W / T are 16-B
 * aligned it runs on the tcgen05 tensor cores (kind::tf32 "3xTF32": x = hi
 * + lo, Xhi.Whi + Xhi.Wlo + Xlo.Whi accumulated in fp32 in TMEM; the dropped
 * terms are < 2^-20 relative per product), in output-column blocks of at
 * most 256 when W's TF32 image does not fit shared memory whole; otherwise
 * on CUDA cores with sequential fp32 accumulation over Ki (Ki <= 800, else
 * PSPMM_ERR_UNSUPPORTED).  Both stay within 1e-5 sum |x||w| of the exact
 * product.  Asynchronous on `stream`.
 */
pspmm_status pspmm_dense_gemm(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                              const float *d_W, int64_t ldw, float *d_T, int64_t ldt,
                              void *stream);

/*
 * (f3) One GCN / GIN-style layer H' = A . H . W (PAPER.md P:21-23,
 * P:449-460): Y = A . (X . W) when Ko <= Ki, else (A . X) . W, so the SpMM
 * always runs on min(Ki, Ko) columns; `cfg` is the engine config for that
 * K (e.g. pspmm_decide_config(features, min(Ki, Ko))).  X: n x Ki, W:
 * Ki x Ko, Y: n x Ko; T is a caller-owned n x min(Ki, Ko) workspace (ldt).
 * Errors as pspmm_spmm_run and pspmm_dense_gemm.  Asynchronous.
 */
pspmm_status pspmm_gnn_layer(pspmm_pcsr A, const float *d_X, int64_t ldx, int32_t Ki,
                             const float *d_W, int64_t ldw, int32_t Ko, float *d_T, int64_t ldt,
                             float *d_Y, int64_t ldy, pspmm_config cfg, void *stream);

/*
 * (f1) Locality reordering (§4.4; Rabbit itself is not
 * reimplemented).  Host function over host CSR arrays; writes
 * perm[old] = new for all n nodes (a bijection).  strategy 0 = identity,
 * 1 = BFS / Cuthill-McKee (components by descending size, pseudo-peripheral
 * start, neighbours by ascending degree; the pattern is symmetrised),
 * 2 = descending degree (stable).  Deterministic.
 */
pspmm_status pspmm_reorder(int64_t n, const int32_t *h_rowptr, const int32_t *h_colidx,
                           int32_t strategy, int32_t *h_perm);

/*
 * (f1) A' = P A P^T on the device: row i of A becomes row perm[i], column j
 * becomes perm[j], columns re-sorted ascending per row (canonical).  d_perm
 * is a device int32 bijection of [0, n).  Outputs are caller-allocated:
 * d_out_rowptr[n + 1], d_out_colidx[nnz], d_out_val[nnz].  Validates A;
 * synchronises `stream`.
 */
pspmm_status pspmm_csr_permute(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                               const int32_t *d_colidx, const float *d_val, const int32_t *d_perm,
                               int32_t *d_out_rowptr, int32_t *d_out_colidx, float *d_out_val,
                               void *stream);

/*
 * (f1) Row permutation of a dense fp32 matrix (K columns) on the device,
 * for i < n (n = entries of d_perm):
 * inverse == 0: out[perm[i]] = in[i]   (B' = P B before the SpMM)
 * inverse != 0: out[i] = in[perm[i]]   (C = P^T C' after it; also the
 *               row gather that packs halo rows for the multi-GPU path)
 * in and out must not alias.  Asynchronous on `stream`.
 */
pspmm_status pspmm_permute_rows(int64_t n, int32_t K, const float *d_in, int64_t ldi,
                                const int32_t *d_perm, float *d_out, int64_t ldo, int32_t inverse,
                                void *stream);

/*
 * (a2) Table 3 features of a CSR matrix on the device.  Degree
 * and bandwidth statistics are exact integer reductions; SR_1, SR_2, PR_1,
 * PR_2 use the PCSR counting kernels with the given omega.  Synchronises
 * `stream`.  nnz == 0 -> PSPMM_ERR_EMPTY.
 */
pspmm_status pspmm_features_compute(int64_t n, int64_t nnz, const int32_t *d_rowptr,
                                    const int32_t *d_colidx, int32_t omega, void *stream,
                                    pspmm_features *out);

/*
 * (a3) SpMM-decider stand-in: a pure host function of
 * (features, K) returning a valid <W, F, V, S> (+ G, engine mode, unit
 * order) for K.  The model is a random forest trained on this repo's own
 * B200 autotune sweep, compiled in.
 */
pspmm_status pspmm_decide_config(const pspmm_features *f, int32_t K, pspmm_config *out);

/*
 * (e) nnz-balanced contiguous row partition for P ranks (host).
 * bounds[g] = min{ r : rowptr[r] >= ceil(g nnz / P) } rounded up to a
 * multiple of `align` (>= 1) and clamped to n; bounds[0] = 0, bounds[P] = n.
 * bounds must hold P + 1 entries.
 */
pspmm_status pspmm_shard_plan(int64_t n, const int32_t *h_rowptr, int32_t P, int32_t align,
                              int64_t *bounds);

/*
 * (e) Local CSR of rank r's row shard with columns remapped into the padded
 * all-gather layout of B: col' = owner(col) * n_max + (col - bounds[owner]),
 * n_max = max_g (bounds[g+1] - bounds[g]).  Host arrays; h_lrowptr holds
 * (bounds[r+1] - bounds[r] + 1) entries, h_lcolidx / h_lval hold
 * rowptr[bounds[r+1]] - rowptr[bounds[r]] entries.  Columns stay strictly
 * increasing per row (the remap is monotone).  *n_max_out receives n_max.
 */
pspmm_status pspmm_shard_extract(int64_t n, const int32_t *h_rowptr, const int32_t *h_colidx,
                                 const float *h_val, int32_t P, const int64_t *bounds,
                                 int32_t r, int32_t *h_lrowptr, int32_t *h_lcolidx,
                                 float *h_lval, int64_t *n_max_out);

#ifdef __cplusplus
}
#endif

#endif /* PSPMM_H */
