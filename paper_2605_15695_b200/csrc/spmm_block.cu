// (a6, a7) Engine mode 5: row-block engine with shared-memory B reuse.
//
// The paper blocks rows so that "B's data reuse" is exploited "through
// registers or shared memory" (§3.1).  Vectorized blocking (V = 2,
// registers) only pays when consecutive rows share columns; on
// block-structured graphs (ogbn-proteins-shaped: 3.6 %-dense diagonal
// blocks) two rows rarely share a column, but a block of R = 128 rows touches
// each column of its block ~4.6 times.  This engine captures that reuse in
// shared memory:
//
//  - one CTA per (row block of kR = 128 rows, slice of kKs = 128 columns of
//    C); the row block's columns are cut into windows of kWc = 128 B rows,
//    and only the windows the block touches are visited;
//  - a producer warp stages each window's B tile (kWc rows x kKs columns,
//    64 KB) into a 3-deep shared-memory ring with one 2-D TMA copy
//    (cp.async.bulk.tensor, completion on the stage's mbarrier), so a B row is
//    fetched from L2 once per row block instead of once per nonzero;
//  - 16 consumer warps each own 8 rows of the block (degree-balanced "snake"
//    assignment, so the warps finish together); for every window a warp walks
//    its rows' nonzeros inside the window from a window-major packed stream
//    (col - window start, value; 8 B per nonzero, the CSR's nonzeros reordered
//    once per graph by pspmm_pcsr_attach_blocks), reads the B row from shared
//    memory (LDS.128: lane l holds C columns 4l..4l+3 of the slice) and
//    accumulates res[8] float4 in registers (Alg. 2 l.9-15);
//  - write-back: one streaming 128-bit store per (row, lane) (Alg. 2
//    l.17-23; every C element has exactly one writer, so no atomics; rows of
//    the last partial block beyond n are never written, c-6).
//
// The derived pack is NOT part of the bit-exact PCSR contract (like the
// mode-1 split and the unit order); A's PCSR arrays are untouched.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <numeric>
#include <thread>
#include <vector>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kR = kBlockRows;      // rows per row block (CTA)
constexpr int kWc = kBlockWindow;   // B rows per window
constexpr int kKs = 128;            // C columns per CTA (lane: one float4)
constexpr int kNW = 16;             // consumer warps
constexpr int kRW = kR / kNW;       // rows per consumer warp (8)
constexpr int kStages = 3;
constexpr int kTile = kWc * kKs * 4;  // bytes of one staged B window (64 KB)
static_assert(kRW == 8, "win_cnt packs 8 u8 counts per (window, warp) into a uint2");
static_assert(kWc <= 255, "per-(row, window) counts are u8");

struct BlockArgs {
  const int32_t *__restrict__ win_ptr;   // row blocks + 1: window range of each block
  const int32_t *__restrict__ win_c0;    // per window: first B row
  const uint2 *__restrict__ win_cnt;     // [window][kNW]: 8 u8 counts (one per row slot)
  const int32_t *__restrict__ win_base;  // [window][kNW]: first packed nonzero
  const int2 *__restrict__ pairs;        // packed nonzeros (col - window start, value bits)
  const int16_t *__restrict__ rowmap;    // [block][kNW][kRW]: local row of a slot, -1 = none
  float *__restrict__ C;
  int64_t ldc;
  int32_t n_rows, accumulate;
  Fanout fan;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 2-D TMA tile: columns [c0, c0 + kKs) of B rows [r0, r0 + kWc) -> dst
// (row-major kWc x kKs fp32; rows beyond n_cols are zero-filled)
__device__ __forceinline__ void tma_tile(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                         int r0, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "l"(policy)
      : "memory");
}
// packed nonzero: read once per slice, streamed (no L1 allocation)
__device__ __forceinline__ int2 ld_pair(const int2 *p) {
  int2 v;
  asm("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__global__ void __maxnreg__(120)
    spmm_block_kernel(const __grid_constant__ CUtensorMap map, const BlockArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kTile);
  uint64_t *empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x;
  const int k0 = blockIdx.y * kKs;
  const int w0 = a.win_ptr[blk], w1 = a.win_ptr[blk + 1];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kNW) {  // producer: one elected lane streams the windows' B tiles
    if (lane == 0) {
      uint64_t pol;  // a B tile is re-staged by the other row blocks of the same graph block
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      for (int i = w0, t = 0; i < w1; ++i, ++t) {
        const int s = t % kStages;
        if (t >= kStages) mbar_wait(&empty[s], ((t / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kTile);
        tma_tile(smem + s * kTile, &map, &full[s], k0, a.win_c0[i], pol);
      }
    }
    return;
  }

  float4 acc[kRW];
#pragma unroll
  for (int r = 0; r < kRW; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t sbase = smem_u32(smem) + lane * 16;

  for (int i = w0, t = 0; i < w1; ++i, ++t) {
    const int s = t % kStages;
    const uint2 cnt = a.win_cnt[(int64_t)i * kNW + warp];
    int q = a.win_base[(int64_t)i * kNW + warp];
    mbar_wait(&full[s], (t / kStages) & 1);
    const uint32_t tile = sbase + s * kTile;
#pragma unroll
    for (int r = 0; r < kRW; ++r) {
      const int n = ((r < 4 ? cnt.x : cnt.y) >> (8 * (r & 3))) & 0xff;
      const int2 *pp = a.pairs + q;
      for (int j = 0; j < n; j += 4) {
        int2 pr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pr[u] = (j + u < n) ? ld_pair(pp + j + u) : make_int2(0, 0);
        float4 b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          b[u] = (j + u < n) ? lds128(tile + pr[u].x * (kKs * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float v = __int_as_float(pr[u].y);
          acc[r].x = fmaf(v, b[u].x, acc[r].x);
          acc[r].y = fmaf(v, b[u].y, acc[r].y);
          acc[r].z = fmaf(v, b[u].z, acc[r].z);
          acc[r].w = fmaf(v, b[u].w, acc[r].w);
        }
      }
      q += n;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // write-back (Alg. 2 l.17-23): one writer per element
  const int16_t *rm = a.rowmap + ((int64_t)blk * kNW + warp) * kRW;
#pragma unroll
  for (int r = 0; r < kRW; ++r) {
    const int local = rm[r];
    const int64_t row = (int64_t)blk * kR + local;
    if (local < 0 || row >= a.n_rows) continue;
    const int64_t off = row * a.ldc + k0 + lane * 4;
    float4 v = acc[r];
    float4 *p = reinterpret_cast<float4 *>(a.C + off);
    if (a.accumulate) {
      const float4 o = *p;
      v.x += o.x;
      v.y += o.y;
      v.z += o.z;
      v.w += o.w;
    }
    __stcs(p, v);
#pragma unroll 1
    for (int d = 0; d < a.fan.n; ++d) __stcs(reinterpret_cast<float4 *>(a.fan.peer[d] + off), v);
  }
  if (a.fan.n) __threadfence_system();
}

// Touched windows per row block (device): a bitmap of the block's windows in
// shared memory, one atomicOr per nonzero, then a popcount.
__global__ void touched_windows_kernel(const int32_t *__restrict__ rowptr,
                                       const int32_t *__restrict__ colidx, int64_t n_rows,
                                       int32_t words, unsigned long long *__restrict__ total) {
  extern __shared__ uint32_t bits[];
  for (int w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kR;
  const int64_t r1 = std::min<int64_t>(n_rows, r0 + kR);
  const int64_t p0 = rowptr[r0], p1 = rowptr[r1];
  for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const uint32_t w = (uint32_t)colidx[p] / kWc;
    atomicOr(&bits[w >> 5], 1u << (w & 31));
  }
  __syncthreads();
  unsigned long long c = 0;
  for (int w = threadIdx.x; w < words; w += blockDim.x) c += __popc(bits[w]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

template <typename T>
pspmm_status upload(T **dst, const std::vector<T> &src) {
  PSPMM_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(1, src.size()) * sizeof(T)));
  if (!src.empty())
    PSPMM_CUDA_TRY(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return PSPMM_OK;
}

}  // namespace

void destroy_blocks(RowBlocks *B) {
  if (!B) return;
  cudaFree(B->d_win_ptr);
  cudaFree(B->d_win_c0);
  cudaFree(B->d_win_cnt);
  cudaFree(B->d_win_base);
  cudaFree(B->d_pairs);
  cudaFree(B->d_rowmap);
  delete B;
}

pspmm_status block_reuse(const pspmm_pcsr_s *A, cudaStream_t stream, double *reuse,
                         int64_t *touched) {
  if (!A || !reuse) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "block_reuse: null argument");
  if (A->V != 1 || A->S != 0)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "block_reuse: needs a V = 1, S = 0 handle (CSR order)");
  const int64_t nwin = (A->n_cols + kWc - 1) / kWc;
  const int64_t words = (nwin + 31) / 32;
  if (words * 4 > 200 * 1024)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "block_reuse: more columns than the window bitmap holds");
  const int64_t blocks = (A->n_rows + kR - 1) / kR;
  *reuse = 0.0;
  if (touched) *touched = 0;
  if (A->nnz == 0 || blocks == 0) return PSPMM_OK;
  unsigned long long *d_total = nullptr;
  PSPMM_CUDA_TRY(cudaMallocAsync(&d_total, sizeof(unsigned long long), stream));
  PSPMM_CUDA_TRY(cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), stream));
  const size_t smem = (size_t)std::max<int64_t>(1, words) * 4;
  if (smem > 48 * 1024)
    PSPMM_CUDA_TRY(cudaFuncSetAttribute(touched_windows_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  touched_windows_kernel<<<(unsigned)blocks, 256, smem, stream>>>(
      A->d_rowptr, A->d_colidx, A->n_rows, (int32_t)words, d_total);
  PSPMM_CUDA_TRY(cudaGetLastError());
  unsigned long long h = 0;
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&h, d_total, sizeof(h), cudaMemcpyDeviceToHost, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(d_total, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  if (touched) *touched = (int64_t)h;
  *reuse = h ? (double)A->nnz / ((double)h * kWc) : 0.0;
  return PSPMM_OK;
}

// Build the mode-5 pack on the host (one pass per row block, blocks split
// over host threads): degree-balanced slot assignment, the touched windows,
// per-(window, warp, slot) counts and the window-major nonzero stream.
pspmm_status attach_blocks(pspmm_pcsr_s *A, cudaStream_t stream) {
  if (!A) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "attach_blocks: null handle");
  if (A->V != 1 || A->S != 0)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "attach_blocks: needs a V = 1, S = 0 handle (CSR order)");
  const int64_t n = A->n_rows, nnz = A->nnz;
  const int64_t nblk = (n + kR - 1) / kR;
  const int64_t nwin_all = (A->n_cols + kWc - 1) / kWc;
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  std::vector<int32_t> rp(n + 1), ci(nnz);
  std::vector<float> vl(nnz);
  PSPMM_CUDA_TRY(cudaMemcpy(rp.data(), A->d_rowptr, (n + 1) * 4, cudaMemcpyDeviceToHost));
  if (nnz) {
    PSPMM_CUDA_TRY(cudaMemcpy(ci.data(), A->d_colidx, nnz * 4, cudaMemcpyDeviceToHost));
    PSPMM_CUDA_TRY(cudaMemcpy(vl.data(), A->d_val, nnz * 4, cudaMemcpyDeviceToHost));
  }
  // pass 1: touched windows per block
  std::vector<int32_t> nwin(nblk, 0);
  std::vector<int16_t> rowmap((size_t)nblk * kNW * kRW, (int16_t)-1);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto par = [&](auto &&fn) {
    std::vector<std::thread> th;
    for (int t = 0; t < nth; ++t)
      th.emplace_back([&, t] {
        std::vector<int32_t> mark(nwin_all, -1);
        for (int64_t b = t; b < nblk; b += nth) fn(b, mark);
      });
    for (auto &x : th) x.join();
  };
  par([&](int64_t b, std::vector<int32_t> &mark) {
    const int64_t r0 = b * kR, r1 = std::min(n, r0 + kR);
    int32_t cnt = 0;
    for (int64_t p = rp[r0]; p < rp[r1]; ++p) {
      const int32_t w = ci[p] / kWc;
      if (mark[w] != (int32_t)b) {
        mark[w] = (int32_t)b;
        ++cnt;
      }
    }
    nwin[b] = cnt;
    // degree-balanced slots: rows by descending degree, dealt to the warps
    // in a snake order (0..15, 15..0, ...), slot = round
    int idx[kR];
    const int rows = (int)(r1 - r0);
    for (int k = 0; k < rows; ++k) idx[k] = k;
    std::stable_sort(idx, idx + rows, [&](int x, int y) {
      return rp[r0 + x + 1] - rp[r0 + x] > rp[r0 + y + 1] - rp[r0 + y];
    });
    for (int k = 0; k < rows; ++k) {
      const int round = k / kNW, pos = k % kNW;
      const int w = (round & 1) ? kNW - 1 - pos : pos;
      rowmap[((size_t)b * kNW + w) * kRW + round] = (int16_t)idx[k];
    }
  });
  std::vector<int32_t> win_ptr(nblk + 1, 0);
  for (int64_t b = 0; b < nblk; ++b) win_ptr[b + 1] = win_ptr[b] + nwin[b];
  const int64_t W = win_ptr[nblk];
  std::vector<int32_t> win_c0(W), win_base((size_t)W * kNW);
  std::vector<uint2> win_cnt((size_t)W * kNW);
  std::vector<int2> pairs(nnz);
  // pass 2: counts, bases and the packed stream (a block's nonzeros keep the
  // block's CSR range [rowptr[r0], rowptr[r1]), reordered window-major)
  par([&](int64_t b, std::vector<int32_t> &mark) {
    const int64_t r0 = b * kR, r1 = std::min(n, r0 + kR);
    const int64_t wb = win_ptr[b], nw = nwin[b];
    std::vector<int32_t> wins;
    wins.reserve(nw);
    for (int64_t p = rp[r0]; p < rp[r1]; ++p) {
      const int32_t w = ci[p] / kWc;
      if (mark[w] != (int32_t)b) {
        mark[w] = (int32_t)b;
        wins.push_back(w);
      }
    }
    std::sort(wins.begin(), wins.end());
    for (int64_t k = 0; k < nw; ++k) {
      mark[wins[k]] = (int32_t)(-2 - k);  // window -> local index
      win_c0[wb + k] = wins[k] * kWc;
    }
    std::vector<uint8_t> cnt((size_t)nw * kNW * kRW, 0);
    for (int w = 0; w < kNW; ++w)
      for (int s = 0; s < kRW; ++s) {
        const int local = rowmap[((size_t)b * kNW + w) * kRW + s];
        if (local < 0) continue;
        for (int64_t p = rp[r0 + local]; p < rp[r0 + local + 1]; ++p) {
          const int64_t k = -2 - mark[ci[p] / kWc];
          ++cnt[((size_t)k * kNW + w) * kRW + s];
        }
      }
    std::vector<int64_t> cur((size_t)nw * kNW * kRW);
    int64_t pos = rp[r0];
    for (int64_t k = 0; k < nw; ++k)
      for (int w = 0; w < kNW; ++w) {
        win_base[(size_t)(wb + k) * kNW + w] = (int32_t)pos;
        uint32_t lo = 0, hi = 0;
        for (int s = 0; s < kRW; ++s) {
          const uint32_t c = cnt[((size_t)k * kNW + w) * kRW + s];
          cur[((size_t)k * kNW + w) * kRW + s] = pos;
          pos += c;
          if (s < 4)
            lo |= c << (8 * s);
          else
            hi |= c << (8 * (s - 4));
        }
        win_cnt[(size_t)(wb + k) * kNW + w] = make_uint2(lo, hi);
      }
    for (int w = 0; w < kNW; ++w)
      for (int s = 0; s < kRW; ++s) {
        const int local = rowmap[((size_t)b * kNW + w) * kRW + s];
        if (local < 0) continue;
        for (int64_t p = rp[r0 + local]; p < rp[r0 + local + 1]; ++p) {
          const int64_t k = -2 - mark[ci[p] / kWc];
          int64_t &c = cur[((size_t)k * kNW + w) * kRW + s];
          int32_t bits;
          memcpy(&bits, &vl[p], 4);
          pairs[c++] = make_int2(ci[p] - win_c0[wb + k], bits);
        }
      }
    for (int64_t k = 0; k < nw; ++k) mark[wins[k]] = -1;
  });
  RowBlocks *R = new RowBlocks();
  struct Guard {
    RowBlocks *r;
    ~Guard() { destroy_blocks(r); }
  } guard{R};
  R->num_blocks = nblk;
  R->num_windows = W;
  pspmm_status st;
  if ((st = upload(&R->d_win_ptr, win_ptr)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_c0, win_c0)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_cnt, win_cnt)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_base, win_base)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_pairs, pairs)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_rowmap, rowmap)) != PSPMM_OK) return st;
  R->reuse = W ? (double)nnz / ((double)W * kWc) : 0.0;
  destroy_blocks(A->blocks);
  A->blocks = R;
  guard.r = nullptr;
  return PSPMM_OK;
}

bool block_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc,
                     const float *d_B, const float *d_C) {
  return A && A->blocks && A->V == 1 && A->S == 0 && K % kKs == 0 && ldb % 4 == 0 &&
         ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0 && (uint64_t)ldb * 4 < (1ull << 40);
}

pspmm_status run_spmm_block(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, cudaStream_t stream, int32_t accumulate,
                            const Fanout &fan) {
  if (!block_supported(A, K, ldb, ldc, d_B, d_C))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run mode 5: needs pspmm_pcsr_attach_blocks on a V = 1, S = 0 handle, "
               "K % 128 == 0, ld % 4 == 0 and 16-B aligned B and C");
  const RowBlocks *R = A->blocks;
  if (R->num_blocks == 0) return PSPMM_OK;
  auto encode = get_encode();
  if (!encode) PSPMM_FAIL(PSPMM_ERR_CUDA, "spmm_run mode 5: cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)std::max<int64_t>(1, A->n_cols)};
  cuuint64_t strides[1] = {(cuuint64_t)ldb * 4};
  cuuint32_t box[2] = {(cuuint32_t)kKs, (cuuint32_t)kWc};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(d_B), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) PSPMM_FAIL(PSPMM_ERR_CUDA, "spmm_run mode 5: tensor map encode failed");
  const size_t smem = (size_t)kStages * kTile + 2 * kStages * sizeof(uint64_t);
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(spmm_block_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  BlockArgs args;
  args.win_ptr = R->d_win_ptr;
  args.win_c0 = R->d_win_c0;
  args.win_cnt = R->d_win_cnt;
  args.win_base = R->d_win_base;
  args.pairs = R->d_pairs;
  args.rowmap = R->d_rowmap;
  args.C = d_C;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.accumulate = accumulate;
  args.fan = fan;
  if (R->num_blocks > 0x7fffffff) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run mode 5: grid");
  spmm_block_kernel<<<dim3((unsigned)R->num_blocks, (unsigned)(K / kKs)), (kNW + 1) * 32, smem,
                      stream>>>(map, args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
