// (a6, conditional) Engine mode 1: dense-panel tensor-core path.
//
// "Dense-panel variant (conditional): densify a 128-row panel
// tile in SMEM, gather its union B rows, run tcgen05 kind::tf32 3xTF32 into
// TMEM."  The paper's blocking groups rows into panels so
// that one B row serves several rows of A; where a panel's rows share most
// of a column range the panel tile is a real dense contraction and belongs
// on the tensor cores.
//
// Split (pspmm_pcsr_attach_dense, host, once per graph): A = A_dense +
// A_rest.  A_dense is the set of 128 x 32 tiles (rows [128p, 128p + 128),
// columns [32t, 32t + 32)) holding at least min_density * 4096 nonzeros,
// stored densely (fp32, +0.0f where A has no entry) in the shared-memory
// image order below; A_rest (every other nonzero) gets its own PCSR with
// the handle's (V, S, omega), run by the mode-0 engine.
//
// Run (cfg.mode = 1): C = A_rest.B (mode-0 engine, cfg's W / F / G / order),
// then C += A_dense.B by dense_tc_kernel, one CTA per (dense panel, N pass of
// up to 256 columns):
//  - per tile, the 256 threads stage A (from the image) and the 32 B rows
//    [32t, 32t + 32) x [n0, n0 + N) into shared memory, split into TF32 hi
//    and lo parts (x = hi + lo, both rounded to nearest TF32), in the
//    no-swizzle K-major core-matrix layout the UMMA descriptors describe;
//    two stages, so staging tile i overlaps the MMAs of tile i - 1;
//  - one thread issues tcgen05.mma.cta_group::1.kind::tf32, M = 128,
//    N = 16..256, K = 8 per instruction, three products per K step
//    (hi.hi + hi.lo + lo.hi: "3xTF32", fp32-level accuracy; lo.lo is below
//    2^-22 relative) into one fp32 accumulator in TMEM (N columns);
//    tcgen05.commit on a per-stage mbarrier frees the stage;
//  - epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32w..32w+31 =
//    rows of the panel), C[row, n0 + c] += acc.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kTM = 128;                             // tile rows (MMA M)
constexpr int kTK = 32;                              // tile columns of A (contraction)
constexpr int kNmax = 256;                           // MMA N per pass
constexpr int kABytes = kTM * kTK * 4;               // one A part (hi or lo): 16 KB
constexpr int kBBytes = kNmax * kTK * 4;             // one B part: 32 KB
constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;  // 96 KB
constexpr int kStages = 2;
constexpr int kDenseThreads = 128;                   // 4 warps: producer, MMA, epilogue
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 64 /*barriers, TMEM slot*/;

#ifndef PSPMM_DENSE_DESC_SWAP
#define PSPMM_DENSE_DESC_SWAP 0  // A/B of the LBO / SBO reading (1 = swapped)
#endif

struct DenseArgs {
  const float *__restrict__ tiles;      // num_tiles x (hi 4096, lo 4096), image order
  const float4 *__restrict__ bhi, *__restrict__ blo;  // split_b_kernel images
  const int32_t *__restrict__ panel_ptr;  // dense panel -> its tiles
  const int32_t *__restrict__ panel;      // dense panel -> panel index p
  const int32_t *__restrict__ tile_col;   // tile -> first column 32t
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t n_rows, n_cols, K;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, no swizzle, K-major: core matrices of
// 8 rows x 16 B (8 x 4 TF32) stored as 128 contiguous bytes; `lbo` = bytes
// between core matrices adjacent along K, `sbo` = bytes between core
// matrices adjacent along M / N; version 1 (sm_100) at bit 46.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
#if PSPMM_DENSE_DESC_SWAP
  const uint32_t t = lbo;
  lbo = sbo;
  sbo = t;
#endif
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // base offset 0, layout type 0 (SWIZZLE_NONE)
}

// Instruction descriptor, kind::tf32: D fp32, A and B TF32, both K-major.
__device__ __forceinline__ uint32_t umma_idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kTM >> 4) << 24);
}

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void split4(const float4 &x, float4 &hi, float4 &lo) {
  hi.x = tf32_rn(x.x);
  hi.y = tf32_rn(x.y);
  hi.z = tf32_rn(x.z);
  hi.w = tf32_rn(x.w);
  lo.x = tf32_rn(x.x - hi.x);
  lo.y = tf32_rn(x.y - hi.y);
  lo.z = tf32_rn(x.z - hi.z);
  lo.w = tf32_rn(x.w - hi.w);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// Pre-pass of every mode-1 run: B (row-major, n_cols x K) -> the TF32 hi /
// lo images the tiles copy from.  bimg[kb][n] (float4) = B rows 4kb .. 4kb+3
// at column n (zeros past n_cols), so the 8 K groups of a tile's B operand
// are 8 contiguous runs of N float4: one bulk copy each.
__global__ void split_b_kernel(const float *__restrict__ B, int64_t ldb, int32_t n_cols,
                               int32_t K, int64_t kgroups, float4 *__restrict__ hi,
                               float4 *__restrict__ lo) {
  const int64_t total = kgroups * K;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kb = q / K;
    const int n = (int)(q - kb * K);
    const int64_t r0 = 4 * kb;
    const float *bp = B + r0 * ldb + n;
    float4 x;
    x.x = r0 + 0 < n_cols ? __ldg(bp) : 0.f;
    x.y = r0 + 1 < n_cols ? __ldg(bp + ldb) : 0.f;
    x.z = r0 + 2 < n_cols ? __ldg(bp + 2 * ldb) : 0.f;
    x.w = r0 + 3 < n_cols ? __ldg(bp + 3 * ldb) : 0.f;
    float4 h, l;
    split4(x, h, l);
    hi[q] = h;
    lo[q] = l;
  }
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One CTA per (dense panel, N pass).  Warp 0 lane 0: producer (bulk copies
// of the A hi / lo image and the 2 x 8 B runs of each tile into a stage);
// warp 1 lane 0: MMA issuer; all four warps: epilogue.
__global__ void __launch_bounds__(kDenseThreads, 1) dense_tc_kernel(const DenseArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  // barriers: full[0..1] (copies landed), empty[0..1] (MMAs done), acc
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
  uint64_t *full = bar, *empty = bar + 2, *accb = bar + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 6);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int dp = blockIdx.x;
  const int panel = a.panel[dp];
  const int t0 = a.panel_ptr[dp], t1 = a.panel_ptr[dp + 1];
  const int n0 = blockIdx.y * kNmax;
  const int N = min(kNmax, a.K - n0);  // multiple of 16 (checked on the host)

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kNmax));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t bytes_b = (uint32_t)N * 16;  // one K group of B (N float4)

  if (tid == 0) {  // producer
    for (int t = t0; t < t1; ++t) {
      const int i = t - t0, s = i & 1;
      if (i >= 2) mbar_wait(&empty[s], ((i - 2) >> 1) & 1);
      uint8_t *st = smem + s * kStageBytes;
      mbar_expect_tx(&full[s], 2u * kABytes + 2u * (kTK / 4) * bytes_b);
      const float4 *ai = reinterpret_cast<const float4 *>(a.tiles) + (int64_t)t * (2 * kTM * kTK / 4);
      bulk_g2s(st, ai, kABytes, &full[s]);                              // A hi
      bulk_g2s(st + kABytes, ai + kTM * kTK / 4, kABytes, &full[s]);    // A lo
      const int64_t kb0 = a.tile_col[t] / 4;
#pragma unroll 1
      for (int kb = 0; kb < kTK / 4; ++kb) {
        const int64_t off = (kb0 + kb) * a.K + n0;
        bulk_g2s(st + 2 * kABytes + kb * bytes_b, a.bhi + off, bytes_b, &full[s]);
        bulk_g2s(st + 2 * kABytes + kBBytes + kb * bytes_b, a.blo + off, bytes_b, &full[s]);
      }
    }
  } else if (tid == 32) {  // MMA issuer
    const uint32_t idesc = umma_idesc(N);
    for (int t = t0; t < t1; ++t) {
      const int i = t - t0, s = i & 1;
      mbar_wait(&full[s], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = smem_u32(smem + s * kStageBytes);
      const uint32_t a_lo = a_hi + kABytes, b_hi = a_hi + 2 * kABytes, b_lo = b_hi + kBBytes;
#pragma unroll
      for (int ks = 0; ks < kTK / 8; ++ks) {  // K = 8 TF32 = two core matrices per MMA
        const uint32_t oa = ks * 2 * (kTM * 16), ob = ks * 2 * bytes_b;
        const uint64_t dah = umma_desc(a_hi + oa, kTM * 16, 128);
        const uint64_t dal = umma_desc(a_lo + oa, kTM * 16, 128);
        const uint64_t dbh = umma_desc(b_hi + ob, bytes_b, 128);
        const uint64_t dbl = umma_desc(b_lo + ob, bytes_b, 128);
        umma_tf32(tmem, dah, dbh, idesc, (i > 0 || ks > 0) ? 1u : 0u);
        umma_tf32(tmem, dah, dbl, idesc, 1u);
        umma_tf32(tmem, dal, dbh, idesc, 1u);
      }
      umma_commit(&empty[s]);
    }
    // every MMA of this CTA has completed once this commit arrives
    umma_commit(accb);
  }
  __syncwarp();
  mbar_wait(accb, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // warp w reads TMEM lanes 32 w .. 32 w + 31 = rows of the panel
  const int64_t row = (int64_t)panel * kTM + warp * 32 + lane;
  const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tbase + c, v);
    if (row < a.n_rows) {
      float4 *cp = reinterpret_cast<float4 *>(a.C + row * a.ldc + n0 + c);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4 o = cp[j];
        o.x += v[4 * j];
        o.y += v[4 * j + 1];
        o.z += v[4 * j + 2];
        o.w += v[4 * j + 3];
        cp[j] = o;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kNmax));
}

}  // namespace

bool dense_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                     const float *d_C) {
  return A->dense != nullptr && K % 16 == 0 && K <= A->dense->k_max && ldb % 4 == 0 &&
         ldc % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0;
}

// C (+)= A.B with cfg.mode = 1: the rest through the mode-0 engine, then the
// dense tiles on the tensor cores (same stream, so the RMW sees the rest).
pspmm_status run_spmm_dense(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                            int32_t accumulate) {
  if (!A || !d_B || !d_C) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run: null handle or pointer");
  if (K < 1 || ldb < K || ldc < K)
    PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "spmm_run: need K >= 1, ldb >= K, ldc >= K");
  if (!A->dense)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run mode 1: no dense tiles attached (pspmm_pcsr_attach_dense)");
  if (!dense_supported(A, K, ldb, ldc, d_B, d_C))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run mode 1: needs K % 16 == 0, K <= the split's k_max, ld % 4 == 0, "
               "16-B aligned B and C");
  pspmm_config rc = cfg;
  rc.mode = 0;
  // no dense tiles: the rest is A itself (not duplicated)
  const DenseTiles &D = *A->dense;
  pspmm_status st =
      run_spmm(D.rest ? D.rest : A, d_B, ldb, K, d_C, ldc, rc, stream, accumulate);
  if (st != PSPMM_OK) return st;
  if (D.num_panels == 0) return PSPMM_OK;
  static bool attr = false;
  if (!attr) {
    PSPMM_CUDA_TRY(cudaFuncSetAttribute(dense_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kSmemBytes));
    attr = true;
  }
  const int64_t total = D.kgroups * K;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  split_b_kernel<<<blocks, 256, 0, stream>>>(d_B, ldb, (int32_t)A->n_cols, K, D.kgroups, D.d_bhi,
                                             D.d_blo);
  PSPMM_CUDA_TRY(cudaGetLastError());
  DenseArgs args;
  args.tiles = D.d_tiles;
  args.bhi = D.d_bhi;
  args.blo = D.d_blo;
  args.panel_ptr = D.d_panel_ptr;
  args.panel = D.d_panel;
  args.tile_col = D.d_tile_col;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.n_cols = (int32_t)A->n_cols;
  args.K = K;
  const unsigned by = (unsigned)((K + kNmax - 1) / kNmax);
  dense_tc_kernel<<<dim3((unsigned)D.num_panels, by), kDenseThreads, kSmemBytes, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

void destroy_dense(DenseTiles *D) {
  if (!D) return;
  cudaFree(D->d_tiles);
  cudaFree(D->d_panel_ptr);
  cudaFree(D->d_panel);
  cudaFree(D->d_tile_col);
  cudaFree(D->d_bhi);
  cudaFree(D->d_blo);
  pspmm_pcsr_destroy(D->rest);
  delete D;
}

// Round to the nearest TF32 (ties away from zero), like cvt.rna.tf32.f32:
// the A image is split on the host once per graph (finite values).
float tf32_rn_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Host-side split of the CSR A was built from into dense 128 x 32 tiles and
// the rest (one pass over the nonzeros per panel, a touched-list counter per
// 32-column tile).  Synchronises `stream` (sizes, copies).
pspmm_status attach_dense(pspmm_pcsr_s *A, const int32_t *d_rowptr, const int32_t *d_colidx,
                          const float *d_val, double min_density, int32_t k_max,
                          cudaStream_t stream, int64_t *out_tiles) {
  if (!A || !d_rowptr || (A->nnz > 0 && (!d_colidx || !d_val)))
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_attach_dense: null handle or CSR pointer");
  if (!(min_density > 0.0 && min_density <= 1.0))
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_attach_dense: min_density must be in (0, 1]");
  if (k_max < 16 || k_max % 16 != 0)
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_attach_dense: k_max must be a positive multiple of 16");
  pspmm_status st = validate_csr(A->n_rows, A->n_cols, A->nnz, d_rowptr, d_colidx, stream);
  if (st != PSPMM_OK) return st;
  const int64_t n = A->n_rows, nnz = A->nnz;
  std::vector<int32_t> rp(n + 1), ci(nnz), rest_rp(n + 1);
  std::vector<float> vl(nnz);
  PSPMM_CUDA_TRY(cudaMemcpyAsync(rp.data(), d_rowptr, (n + 1) * 4, cudaMemcpyDeviceToHost, stream));
  if (nnz) {
    PSPMM_CUDA_TRY(cudaMemcpyAsync(ci.data(), d_colidx, nnz * 4, cudaMemcpyDeviceToHost, stream));
    PSPMM_CUDA_TRY(cudaMemcpyAsync(vl.data(), d_val, nnz * 4, cudaMemcpyDeviceToHost, stream));
  }
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  if (rp[n] != nnz) PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "pcsr_attach_dense: nnz differs from A's");

  const int64_t T = (A->n_cols + kTK - 1) / kTK;
  const int64_t P = (n + kTM - 1) / kTM;
  const int32_t thr = std::max<int32_t>(1, (int32_t)(min_density * kTM * kTK + 0.999999));
  std::vector<int32_t> cnt(T, 0), tid_of(T, -1), touched;
  std::vector<int32_t> panel_ptr(1, 0), panel_ids, tile_col;
  std::vector<float> tiles;
  std::vector<int32_t> rest_ci;
  std::vector<float> rest_vl;
  rest_ci.reserve(nnz);
  rest_vl.reserve(nnz);
  rest_rp[0] = 0;
  for (int64_t p = 0; p < P; ++p) {
    const int64_t r0 = p * kTM, r1 = std::min(n, r0 + kTM);
    touched.clear();
    for (int64_t e = rp[r0]; e < rp[r1]; ++e) {
      const int32_t t = ci[e] / kTK;
      if (cnt[t]++ == 0) touched.push_back(t);
    }
    std::sort(touched.begin(), touched.end());
    const int64_t first = (int64_t)tile_col.size();
    for (int32_t t : touched)
      if (cnt[t] >= thr) {
        tid_of[t] = (int32_t)tile_col.size();
        tile_col.push_back(t * kTK);
      }
    const int64_t added = (int64_t)tile_col.size() - first;
    if (added) {
      tiles.resize(tile_col.size() * (size_t)(2 * kTM * kTK), 0.f);
      panel_ids.push_back((int32_t)p);
      panel_ptr.push_back((int32_t)tile_col.size());
    }
    for (int64_t r = r0; r < r1; ++r) {
      for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        const int32_t c = ci[e], t = c / kTK;
        if (tid_of[t] >= 0) {
          // image order: float4 q = kb * 128 + (r - r0), element c % 4; the
          // TF32 hi part, then the lo part 4096 floats later
          const int k = c - t * kTK;
          const size_t at =
              (size_t)tid_of[t] * (2 * kTM * kTK) + ((size_t)(k / 4) * kTM + (r - r0)) * 4 + k % 4;
          const float hi = tf32_rn_host(vl[e]);
          tiles[at] = hi;
          tiles[at + kTM * kTK] = tf32_rn_host(vl[e] - hi);
        } else {
          rest_ci.push_back(c);
          rest_vl.push_back(vl[e]);
        }
      }
      rest_rp[r + 1] = (int32_t)rest_ci.size();
    }
    for (int32_t t : touched) {
      cnt[t] = 0;
      tid_of[t] = -1;
    }
  }

  DenseTiles *D = new (std::nothrow) DenseTiles();
  if (!D) PSPMM_FAIL(PSPMM_ERR_OOM, "pcsr_attach_dense: host allocation failed");
  D->num_panels = (int64_t)panel_ids.size();
  D->num_tiles = (int64_t)tile_col.size();
  D->nnz_dense = nnz - (int64_t)rest_ci.size();
  D->k_max = k_max;
  D->kgroups = ((A->n_cols + kTK - 1) / kTK) * (kTK / 4);
  int32_t *d_rrp = nullptr, *d_rci = nullptr;
  float *d_rvl = nullptr;
  const int64_t rn = (int64_t)rest_ci.size();
  auto fail = [&](cudaError_t e, const char *w) {
    cudaFree(d_rrp);
    cudaFree(d_rci);
    cudaFree(d_rvl);
    destroy_dense(D);
    return cuda_status(e, w);
  };
  cudaError_t e = cudaSuccess;
  if (D->num_tiles) {
    if ((e = cudaMalloc(&D->d_tiles, tiles.size() * 4)) != cudaSuccess ||
        (e = cudaMalloc(&D->d_panel_ptr, panel_ptr.size() * 4)) != cudaSuccess ||
        (e = cudaMalloc(&D->d_panel, panel_ids.size() * 4)) != cudaSuccess ||
        (e = cudaMalloc(&D->d_tile_col, tile_col.size() * 4)) != cudaSuccess ||
        (e = cudaMalloc(&D->d_bhi, (size_t)D->kgroups * k_max * 16)) != cudaSuccess ||
        (e = cudaMalloc(&D->d_blo, (size_t)D->kgroups * k_max * 16)) != cudaSuccess)
      return fail(e, "pcsr_attach_dense: cudaMalloc");
    if ((e = cudaMemcpy(D->d_tiles, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess ||
        (e = cudaMemcpy(D->d_panel_ptr, panel_ptr.data(), panel_ptr.size() * 4,
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(D->d_panel, panel_ids.data(), panel_ids.size() * 4,
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(D->d_tile_col, tile_col.data(), tile_col.size() * 4,
                        cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(e, "pcsr_attach_dense: cudaMemcpy");
  }
  if (D->num_tiles == 0) {  // nothing dense: mode 1 runs A itself on the mode-0 engine
    destroy_dense(A->dense);
    A->dense = D;
    if (out_tiles) *out_tiles = 0;
    return PSPMM_OK;
  }
  if ((e = cudaMalloc(&d_rrp, (n + 1) * 4)) != cudaSuccess ||
      (e = cudaMalloc(&d_rci, std::max<int64_t>(rn, 1) * 4)) != cudaSuccess ||
      (e = cudaMalloc(&d_rvl, std::max<int64_t>(rn, 1) * 4)) != cudaSuccess)
    return fail(e, "pcsr_attach_dense: cudaMalloc");
  if ((e = cudaMemcpy(d_rrp, rest_rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (rn && (e = cudaMemcpy(d_rci, rest_ci.data(), rn * 4, cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (rn && (e = cudaMemcpy(d_rvl, rest_vl.data(), rn * 4, cudaMemcpyHostToDevice)) != cudaSuccess))
    return fail(e, "pcsr_attach_dense: cudaMemcpy");
  D->rest = new (std::nothrow) pspmm_pcsr_s();
  if (!D->rest) {
    cudaFree(d_rrp);
    cudaFree(d_rci);
    cudaFree(d_rvl);
    destroy_dense(D);
    PSPMM_FAIL(PSPMM_ERR_OOM, "pcsr_attach_dense: host allocation failed");
  }
  // SG of an empty rest is undefined under Eq. 3 (PSPMM_ERR_EMPTY): any SG
  // gives the same (empty) chunks, so force omega there
  st = build_pcsr(n, A->n_cols, rn, d_rrp, d_rci, d_rvl, A->V, A->S, A->omega,
                  rn == 0 ? A->omega : 0, stream, D->rest);
  // Table-3 features of the rest (a different sparse matrix from A), for
  // pspmm_decide_dense to pick the rest's engine knobs
  if (st == PSPMM_OK && rn > 0 && A->n_cols == n &&
      compute_features(n, rn, d_rrp, d_rci, 32, stream, &D->rest_f) == PSPMM_OK)
    D->rest_f_ok = true;
  if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return fail(e, "pcsr_attach_dense");
  cudaFree(d_rrp);
  cudaFree(d_rci);
  cudaFree(d_rvl);
  if (st != PSPMM_OK) {
    destroy_dense(D);
    return st;
  }
  destroy_dense(A->dense);
  A->dense = D;
  if (out_tiles) *out_tiles = D->num_tiles;
  return PSPMM_OK;
}

}  // namespace pspmm
