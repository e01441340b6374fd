// (a6, a7) Engine mode 6: staged-band engine for locality-ordered graphs.
//
// The paper's locality step (§4.4: reordering so that "rows with
// similar column sets are close") leaves each block of consecutive rows
// touching a few contiguous column ranges (a road lattice: the rows
// themselves and the rows one lattice width above and below).  The mode-0 /
// mode-3 engines gather every B row with a dependent rowPtr -> colIdx ->
// B-row chain per row, which keeps them latency-bound on such graphs
// (roadNet: 58 % of the HBM roofline, long-scoreboard stalls).  Here the
// chain is cut:
//
//  - pack (pspmm_pcsr_attach_band, once per graph): rows in blocks of
//    kRows = 128; per block the sorted distinct columns merged into ranges
//    (gaps of at most kGap rows are staged too), each range a contiguous run
//    of B rows; every nonzero's column replaced by its row slot in the
//    block's staged band (blocks whose band exceeds the budget keep the
//    global column and gather from L2 / HBM instead);
//  - kernel (one CTA of 256 threads per block, ~3 resident per SM): thread 0
//    issues one 1-D bulk copy (cp.async.bulk, TMA engine) per range into
//    shared memory; meanwhile every row group (G lanes = K / 4 columns, one
//    float4 each) loads its rows' rowPtr pairs and (slot, value) pairs into
//    registers (lane l holds nonzero l of the row); after the mbarrier
//    completes, each nonzero is a warp-shuffle broadcast of (slot, value)
//    and one LDS.128 of the staged B row (Alg. 2 l.9-15), and the row is
//    written once with a streaming 128-bit store per lane (l.17-23).
//
// The pack is derived data, not part of the bit-exact PCSR contract; the
// handle's rowPtr and val are used as they are.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kRows = kBandRows;  // rows per block (CTA)
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGap = 8;           // merge column ranges separated by <= kGap rows

struct BandArgs {
  const int32_t *__restrict__ rowptr;
  const int32_t *__restrict__ slot;     // per nonzero: staged row slot, or global column
  const float *__restrict__ val;
  const int32_t *__restrict__ rng_ptr;  // blocks + 1
  const int32_t *__restrict__ rng_lo;   // first B row of a range
  const int32_t *__restrict__ rng_len;  // rows of a range
  const int32_t *__restrict__ blk_rows; // staged rows of a block (-1: gathers from global)
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t n_rows, K, accumulate;
  Fanout fan;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ int lda(const int32_t *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float lda(const float *p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void fma4(float4 &acc, float v, const float4 &b) {
  acc.x = fmaf(v, b.x, acc.x);
  acc.y = fmaf(v, b.y, acc.y);
  acc.z = fmaf(v, b.z, acc.z);
  acc.w = fmaf(v, b.w, acc.w);
}

// G lanes per row (K <= 4 G), RPG rows per group: kRows = kWarps (32 / G) RPG.
template <int G>
__global__ void __launch_bounds__(kThreads, 3) spmm_band_kernel(const BandArgs a) {
  constexpr int GPW = 32 / G;                  // row groups per warp
  constexpr int RPG = kRows / (kWarps * GPW);  // rows per group
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, l = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
  const int blk = blockIdx.x;
  const int64_t r0 = (int64_t)blk * kRows;
  const int staged = a.blk_rows[blk];
  const uint32_t rowb = (uint32_t)a.ldb * 4u;  // staged row pitch = B's row pitch
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && staged > 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"((uint32_t)staged * rowb)
                 : "memory");
    uint32_t dst = smem_u32(smem);
    for (int i = a.rng_ptr[blk], e = a.rng_ptr[blk + 1]; i < e; ++i) {
      const uint32_t bytes = (uint32_t)a.rng_len[i] * rowb;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(dst),
          "l"(a.B + (int64_t)a.rng_lo[i] * a.ldb), "r"(bytes), "r"(smem_u32(&bar))
          : "memory");
      dst += bytes;
    }
  }
  // A of this group's rows into registers while the band lands
  int p0[RPG], cnt[RPG], sl[RPG];
  float vv[RPG];
#pragma unroll
  for (int i = 0; i < RPG; ++i) {
    const int64_t r = r0 + (i * kWarps + warp) * GPW + g;
    const bool ok = r < a.n_rows;
    p0[i] = ok ? lda(a.rowptr + r) : 0;
    cnt[i] = ok ? lda(a.rowptr + r + 1) - p0[i] : 0;
  }
#pragma unroll
  for (int i = 0; i < RPG; ++i) {
    const bool ok = l < cnt[i];
    sl[i] = ok ? lda(a.slot + p0[i] + l) : 0;
    vv[i] = ok ? lda(a.val + p0[i] + l) : 0.f;
  }
  const bool cok = l * 4 < a.K;
  const uint32_t sbase = smem_u32(smem) + l * 16;
  const float *gb = a.B + l * 4;
  if (staged > 0) mbar_wait(&bar, 0);
#pragma unroll
  for (int i = 0; i < RPG; ++i) {
    const int64_t r = r0 + (i * kWarps + warp) * GPW + g;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int n = cnt[i];
    const int nb = min(n, G);
    if (staged > 0) {
      for (int j = 0; j < nb; ++j) {
        const int s = __shfl_sync(gmask, sl[i], j, G);
        const float v = __shfl_sync(gmask, vv[i], j, G);
        if (cok) {
          float4 b;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                       : "r"(sbase + (uint32_t)s * rowb));
          fma4(acc, v, b);
        }
      }
      for (int j = G; j < n && cok; ++j) {  // rows longer than G vectors
        const int s = lda(a.slot + p0[i] + j);
        const float v = lda(a.val + p0[i] + j);
        float4 b;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                     : "r"(sbase + (uint32_t)s * rowb));
        fma4(acc, v, b);
      }
    } else {  // band over budget: gather from global (slot = column)
      for (int j = 0; j < nb; ++j) {
        const int s = __shfl_sync(gmask, sl[i], j, G);
        const float v = __shfl_sync(gmask, vv[i], j, G);
        if (cok) fma4(acc, v, __ldg(reinterpret_cast<const float4 *>(gb + (int64_t)s * a.ldb)));
      }
      for (int j = G; j < n && cok; ++j) {
        const int s = lda(a.slot + p0[i] + j);
        const float v = lda(a.val + p0[i] + j);
        fma4(acc, v, __ldg(reinterpret_cast<const float4 *>(gb + (int64_t)s * a.ldb)));
      }
    }
    if (r < a.n_rows && cok) {
      const int64_t off = r * a.ldc + l * 4;
      float4 *p = reinterpret_cast<float4 *>(a.C + off);
      if (a.accumulate) {
        const float4 o = *p;
        acc.x += o.x;
        acc.y += o.y;
        acc.z += o.z;
        acc.w += o.w;
      }
      fan_store4(a.C, a.fan, off, acc);
    }
  }
  if (a.fan.n) __threadfence_system();
}

template <typename T>
pspmm_status upload(T **dst, const std::vector<T> &src) {
  PSPMM_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(1, src.size()) * sizeof(T)));
  if (!src.empty())
    PSPMM_CUDA_TRY(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return PSPMM_OK;
}

int lanes_for(int K) {
  int G = 4;
  while (G * 4 < K) G <<= 1;
  return G;
}

template <int G>
pspmm_status launch_band(const BandArgs &args, int64_t nblk, size_t smem, cudaStream_t stream) {
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(spmm_band_kernel<G>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  spmm_band_kernel<G><<<(unsigned)nblk, kThreads, smem, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace

void destroy_band(Band *D) {
  if (!D) return;
  cudaFree(D->d_slot);
  cudaFree(D->d_rng_ptr);
  cudaFree(D->d_rng_lo);
  cudaFree(D->d_rng_len);
  cudaFree(D->d_blk_rows);
  delete D;
}

// Host pack: per block of kRows rows the merged column ranges and the
// nonzeros' band slots (blocks split over host threads).  Synchronises
// `stream`.
pspmm_status attach_band(pspmm_pcsr_s *A, int32_t k_max, cudaStream_t stream, double *staged_frac) {
  if (!A) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "attach_band: null handle");
  if (A->V != 1 || A->S != 0)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "attach_band: needs a V = 1, S = 0 handle (CSR order)");
  if (k_max < 4 || k_max > kBandMaxK || k_max % 4 != 0)
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "attach_band: k_max must be a multiple of 4 in [4, 128]");
  const int64_t n = A->n_rows, nnz = A->nnz;
  const int64_t nblk = (n + kRows - 1) / kRows;
  const int64_t max_rows = kBandBytes / ((int64_t)k_max * 4);  // staged rows per block
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  std::vector<int32_t> rp(n + 1), ci(nnz);
  PSPMM_CUDA_TRY(cudaMemcpy(rp.data(), A->d_rowptr, (n + 1) * 4, cudaMemcpyDeviceToHost));
  if (nnz) PSPMM_CUDA_TRY(cudaMemcpy(ci.data(), A->d_colidx, nnz * 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> slot(std::max<int64_t>(nnz, 1)), blk_rows(nblk);
  std::vector<std::vector<int32_t>> lo_t(nblk), len_t(nblk);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t)
    th.emplace_back([&, t] {
      std::vector<int32_t> cols;
      for (int64_t b = t; b < nblk; b += nth) {
        const int64_t q0 = rp[b * kRows], q1 = rp[std::min(n, (b + 1) * kRows)];
        cols.assign(ci.begin() + q0, ci.begin() + q1);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        std::vector<int32_t> &lo = lo_t[b], &len = len_t[b];
        int64_t rows = 0;
        for (size_t i = 0; i < cols.size();) {
          size_t j = i;
          while (j + 1 < cols.size() && cols[j + 1] - cols[j] <= kGap + 1) ++j;
          lo.push_back(cols[i]);
          len.push_back(cols[j] - cols[i] + 1);
          rows += cols[j] - cols[i] + 1;
          i = j + 1;
        }
        if (rows > max_rows || rows == 0) {  // over budget (or empty): global gathers
          blk_rows[b] = rows == 0 ? 0 : -1;
          lo.clear();
          len.clear();
          for (int64_t p = q0; p < q1; ++p) slot[p] = ci[p];
          continue;
        }
        blk_rows[b] = (int32_t)rows;
        // column -> slot: ranges are sorted; slot = range base + offset
        std::vector<int64_t> base(lo.size());
        int64_t acc = 0;
        for (size_t k = 0; k < lo.size(); ++k) {
          base[k] = acc;
          acc += len[k];
        }
        for (int64_t p = q0; p < q1; ++p) {
          const size_t k = std::upper_bound(lo.begin(), lo.end(), ci[p]) - lo.begin() - 1;
          slot[p] = (int32_t)(base[k] + (ci[p] - lo[k]));
        }
      }
    });
  for (auto &x : th) x.join();
  std::vector<int32_t> rng_ptr(nblk + 1, 0), rng_lo, rng_len;
  int64_t staged_blocks = 0, nonempty = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    rng_ptr[b + 1] = rng_ptr[b] + (int32_t)lo_t[b].size();
    rng_lo.insert(rng_lo.end(), lo_t[b].begin(), lo_t[b].end());
    rng_len.insert(rng_len.end(), len_t[b].begin(), len_t[b].end());
    if (blk_rows[b] != 0) ++nonempty;
    if (blk_rows[b] > 0) ++staged_blocks;
  }
  Band *D = new Band();
  struct Guard {
    Band *d;
    ~Guard() { destroy_band(d); }
  } guard{D};
  D->num_blocks = nblk;
  D->k_max = k_max;
  D->staged_frac = nonempty ? (double)staged_blocks / nonempty : 1.0;
  pspmm_status st;
  if ((st = upload(&D->d_slot, slot)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_rng_ptr, rng_ptr)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_rng_lo, rng_lo)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_rng_len, rng_len)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_blk_rows, blk_rows)) != PSPMM_OK) return st;
  destroy_band(A->band);
  A->band = D;
  guard.d = nullptr;
  if (staged_frac) *staged_frac = D->staged_frac;
  return PSPMM_OK;
}

bool band_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                    const float *d_C) {
  return A && A->band && A->V == 1 && A->S == 0 && K % 4 == 0 && K <= A->band->k_max &&
         ldb % 4 == 0 && ldb <= A->band->k_max && ldc % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0;
}

pspmm_status run_spmm_band(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                           float *d_C, int64_t ldc, cudaStream_t stream, int32_t accumulate,
                           const Fanout &fan) {
  if (!band_supported(A, K, ldb, ldc, d_B, d_C))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run mode 6: needs pspmm_pcsr_attach_band on a V = 1, S = 0 handle, "
               "K % 4 == 0, K <= ldb <= the pack's k_max, ldc % 4 == 0, 16-B aligned B and C");
  const Band *D = A->band;
  if (D->num_blocks == 0) return PSPMM_OK;
  BandArgs args;
  args.rowptr = A->d_rowptr;
  args.slot = D->d_slot;
  args.val = A->d_val;
  args.rng_ptr = D->d_rng_ptr;
  args.rng_lo = D->d_rng_lo;
  args.rng_len = D->d_rng_len;
  args.blk_rows = D->d_blk_rows;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.K = K;
  args.accumulate = accumulate;
  args.fan = fan;
  // dynamic shared memory: the largest band this k_max allows at this pitch
  const size_t smem = (size_t)(kBandBytes / ((int64_t)D->k_max * 4)) * (size_t)ldb * 4;
  switch (lanes_for(K)) {
    case 4: return launch_band<4>(args, D->num_blocks, smem, stream);
    case 8: return launch_band<8>(args, D->num_blocks, smem, stream);
    case 16: return launch_band<16>(args, D->num_blocks, smem, stream);
    default: return launch_band<32>(args, D->num_blocks, smem, stream);
  }
}

}  // namespace pspmm
