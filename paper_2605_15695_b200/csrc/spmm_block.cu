// (a6, a7) Engine mode 5: row-block engine with shared-memory B reuse.
//
// The paper blocks rows so that "B's data reuse" is exploited "through
// registers or shared memory" (§3.1).  Vectorized blocking (V = 2,
// registers) only pays when consecutive rows share columns; on
// block-structured graphs (ogbn-proteins-shaped: 3.6 %-dense diagonal
// blocks) two rows rarely share a column, but a block of ~128-256 rows
// touches each column of its block ~5-9 times.  This engine captures that
// reuse in shared memory:
//
//  - one CTA per (slice of kKs = 128 columns of C, row block of NW x RW
//    rows); the slice index varies fastest in the grid, so the CTAs of one
//    row block run together and share its packed stream and B rows in L2;
//    the row block's columns are cut into windows of kWc = 128 B rows, and
//    only the windows the block touches are visited;
//  - a producer warp stages each window's B tile (kWc rows x kKs columns,
//    64 KB, one 2-D TMA copy) and the window's packed nonzeros (col - window
//    start, value; 8 B each, one 1-D bulk copy) into a 3-deep shared-memory
//    ring (completion on the stage's mbarrier), so a B row is fetched from L2
//    once per row block instead of once per nonzero, and the (colIdx, val)
//    stream of the block arrives by TMA, not by per-nonzero loads.  A window
//    with more than kBlockMaxPairs nonzeros is split into virtual windows
//    (same B tile, re-staged);
//  - NW consumer warps each own RW rows of the block (degree-balanced
//    "snake" assignment, so the warps finish together).  The register file
//    is split per SM sub-partition (16 K registers each, a CTA's warps dealt
//    round-robin), so NW + 1 warps at R registers need
//    ceil((NW + 1) / 4) x 32 x R <= 16384: 23 + 1 warps at <= 80 registers
//    (RW = 8, the default: 184-row blocks), 15 + 1 at <= 128 (RW = 16).
//    More warps hide the shared-memory latency of the LDS chains (measured:
//    15 / 19 / 23 warps of 8 rows, 3.67 / 3.47 / 3.37 ms on proteins);
//    For every window a warp walks its rows' nonzeros in the staged stream
//    (a broadcast LDS.64 per nonzero), reads the B row from shared memory
//    (LDS.128: lane l holds C columns 4l..4l+3 of the slice) and accumulates
//    res[RW] float4 in registers (Alg. 2 l.9-15): 4 nonzeros per unmasked
//    step, then an exact 2 / 1 remainder (no padded slots);
//  - write-back: one streaming 128-bit store per (row, lane) (Alg. 2
//    l.17-23; every C element has exactly one writer, so no atomics; rows of
//    the last partial block beyond n are never written, c-6).
//
// The derived pack is NOT part of the bit-exact PCSR contract (like the
// mode-1 split and the unit order); A's PCSR arrays are untouched.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <thread>
#include <vector>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kWc = kBlockWindow;   // B rows per window
constexpr int kKs = 128;            // C columns per CTA (lane: one float4)
constexpr int kStages = 3;
constexpr int kTile = kWc * kKs * 4;              // bytes of one staged B window (64 KB)
constexpr int kPairBytes = kBlockMaxPairs * 8;    // bytes of one staged pair block
constexpr int kStage = kTile + kPairBytes;
static_assert(kWc <= 255, "per-(row, window) counts are u8");
static_assert(kBlockMaxPairs % 2 == 0 && kBlockMaxPairs <= 65535, "u16 offsets, 16-B copies");

struct BlockArgs {
  const int32_t *__restrict__ win_ptr;    // row blocks + 1: virtual-window range of each block
  const int32_t *__restrict__ win_c0;     // per virtual window: first B row
  const int64_t *__restrict__ win_pbase;  // per virtual window + 1: first packed pair
  const uint8_t *__restrict__ win_cnt;    // [window][NW][RW]: per-slot counts
  const uint16_t *__restrict__ win_woff;  // [window][NW]: a warp's first pair in the window
  const int2 *__restrict__ pairs;         // packed nonzeros (col - window start, value bits)
  const int16_t *__restrict__ rowmap;     // [block][NW][RW]: local row of a slot, -1 = none
  float *__restrict__ C;
  int64_t ldc;
  int32_t n_rows, accumulate;
  int32_t slices;                         // K / kKs
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
__device__ __forceinline__ void tma_tile(uint32_t dst, const CUtensorMap *map, uint64_t *bar,
                                         int c0, int r0, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (bytes % 16 == 0, 16-B aligned ends)
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int2 lds64(uint32_t addr) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ int4 lds128i(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void fma4(float4 &acc, float v, const float4 &b) {
  acc.x = fmaf(v, b.x, acc.x);
  acc.y = fmaf(v, b.y, acc.y);
  acc.z = fmaf(v, b.z, acc.z);
  acc.w = fmaf(v, b.w, acc.w);
}
template <int RW>
struct Counts;
template <>
struct Counts<8> {
  uint2 v;
  __device__ __forceinline__ void load(const uint8_t *p) { v = *reinterpret_cast<const uint2 *>(p); }
  __device__ __forceinline__ int get(int r) const {
    return ((r < 4 ? v.x : v.y) >> (8 * (r & 3))) & 0xff;
  }
};
template <>
struct Counts<16> {
  uint4 v;
  __device__ __forceinline__ void load(const uint8_t *p) { v = *reinterpret_cast<const uint4 *>(p); }
  __device__ __forceinline__ int get(int r) const {
    const uint32_t w = r < 4 ? v.x : r < 8 ? v.y : r < 12 ? v.z : v.w;
    return (w >> (8 * (r & 3))) & 0xff;
  }
};

// n nonzeros of one row from the staged stream at pair address pa (bytes;
// runs are padded to an even length, so pairs are read two at a time with one
// broadcast LDS.128), B rows from the staged tile at tile (bytes, this lane's
// float4 included)
__device__ __forceinline__ void row_window(float4 &acc, uint32_t &pa, int n, uint32_t tile) {
#pragma unroll 1
  for (int g = n >> 2; g > 0; --g) {
    const int4 q0 = lds128i(pa), q1 = lds128i(pa + 16);
    const float4 b0 = lds128(tile + q0.x * (kKs * 4)), b1 = lds128(tile + q0.z * (kKs * 4));
    const float4 b2 = lds128(tile + q1.x * (kKs * 4)), b3 = lds128(tile + q1.z * (kKs * 4));
    fma4(acc, __int_as_float(q0.y), b0);
    fma4(acc, __int_as_float(q0.w), b1);
    fma4(acc, __int_as_float(q1.y), b2);
    fma4(acc, __int_as_float(q1.w), b3);
    pa += 32;
  }
  const int rem = n & 3;
  if (rem) {
    const int4 q0 = lds128i(pa);
    fma4(acc, __int_as_float(q0.y), lds128(tile + q0.x * (kKs * 4)));
    if (rem >= 2) fma4(acc, __int_as_float(q0.w), lds128(tile + q0.z * (kKs * 4)));
    if (rem == 3) {
      const int2 q1 = lds64(pa + 16);
      fma4(acc, __int_as_float(q1.y), lds128(tile + q1.x * (kKs * 4)));
    }
    pa += rem == 3 ? 32 : 16;
  }
}

template <int RW, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    spmm_block_kernel(const __grid_constant__ CUtensorMap map, const BlockArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStage);
  uint64_t *empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slices = a.slices;  // slice fastest: a block's slices run together
  const int k0 = (int)(blockIdx.x % slices) * kKs;
  const int blk = (int)(blockIdx.x / slices);
  const int w0 = a.win_ptr[blk], w1 = a.win_ptr[blk + 1];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t sm0 = smem_u32(smem);

  if (warp == NW) {  // producer: one elected lane streams the windows' B tiles and pairs
    if (lane == 0) {
      uint64_t pol;  // a B tile is re-staged by the other row blocks of the same graph block
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      int64_t pb = a.win_pbase[w0];
      for (int i = w0, t = 0; i < w1; ++i, ++t) {
        const int s = t % kStages;
        const int64_t pe = a.win_pbase[i + 1];
        const uint32_t pbytes = (uint32_t)(pe - pb) * 8u;
        if (t >= kStages) mbar_wait(&empty[s], ((t / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kTile + pbytes);
        tma_tile(sm0 + s * kStage, &map, &full[s], k0, a.win_c0[i], pol);
        bulk_copy(sm0 + s * kStage + kTile, a.pairs + pb, pbytes, &full[s]);
        pb = pe;
      }
    }
    return;
  }

  float4 acc[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  Counts<RW> cnt, nxt;
  uint32_t woff = 0, woff_n = 0;
  if (w0 < w1) {
    cnt.load(a.win_cnt + ((int64_t)w0 * NW + warp) * RW);
    woff = a.win_woff[(int64_t)w0 * NW + warp];
  }
  for (int i = w0, t = 0; i < w1; ++i, ++t) {
    const int s = t % kStages;
    if (i + 1 < w1) {
      nxt.load(a.win_cnt + ((int64_t)(i + 1) * NW + warp) * RW);
      woff_n = a.win_woff[(int64_t)(i + 1) * NW + warp];
    }
    const uint32_t tile = sm0 + s * kStage + lane * 16;
    uint32_t pa = sm0 + s * kStage + kTile + woff * 8;
    mbar_wait(&full[s], (t / kStages) & 1);
#pragma unroll
    for (int r = 0; r < RW; ++r) row_window(acc[r], pa, cnt.get(r), tile);
    // the stage is refilled by TMA / bulk copies (async proxy) after the
    // release: every lane orders its own generic reads before it (WAR across
    // proxies) and arrives itself, so the release covers each lane's reads
    // without relying on __syncwarp cumulativity
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(&empty[s]);
    cnt = nxt;
    woff = woff_n;
  }

  // write-back (Alg. 2 l.17-23): one writer per element
  const int16_t *rm = a.rowmap + ((int64_t)blk * NW + warp) * RW;
  const int64_t row0 = (int64_t)blk * (NW * RW);
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int local = rm[r];
    const int64_t row = row0 + local;
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
    fan_store4(a.C, a.fan, off, v);
  }
  if (a.fan.n) __threadfence_system();
}

// Touched windows per 128-row block (device; the reuse feature): a bitmap of the block's windows in
// shared memory, one atomicOr per nonzero, then a popcount.
__global__ void touched_windows_kernel(const int32_t *__restrict__ rowptr,
                                       const int32_t *__restrict__ colidx, int64_t n_rows,
                                       int32_t words, unsigned long long *__restrict__ total) {
  extern __shared__ uint32_t bits[];
  for (int w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kReuseRows;
  const int64_t r1 = std::min<int64_t>(n_rows, r0 + kReuseRows);
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

PFN_cuTensorMapEncodeTiled_v12000 get_encode_impl() {
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
void *tensor_map_encoder() { return reinterpret_cast<void *>(get_encode_impl()); }

void destroy_blocks(RowBlocks *B) {
  if (!B) return;
  cudaFree(B->d_win_ptr);
  cudaFree(B->d_win_c0);
  cudaFree(B->d_win_pbase);
  cudaFree(B->d_win_cnt);
  cudaFree(B->d_win_woff);
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
  const int64_t blocks = (A->n_rows + kReuseRows - 1) / kReuseRows;
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

// Build the mode-5 pack on the host (blocks split over host threads):
// degree-balanced slot assignment, the touched windows, the split into
// virtual windows of <= kBlockMaxPairs nonzeros, per-(virtual window, warp,
// slot) counts, per-(virtual window, warp) offsets and the packed stream.
pspmm_status attach_blocks(pspmm_pcsr_s *A, cudaStream_t stream) {
  if (!A) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "attach_blocks: null handle");
  if (A->V != 1 || A->S != 0)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "attach_blocks: needs a V = 1, S = 0 handle (CSR order)");
  // rows per consumer warp and consumer warps per CTA (A/B knobs for the
  // tools: PSPMM_BLOCK_RW = 8 | 16, PSPMM_BLOCK_NW = 15 | 19 | 23 with rw = 8)
  int rw = kBlockRw, nw = kBlockNw;
  if (const char *e = std::getenv("PSPMM_BLOCK_RW")) rw = std::atoi(e) == 16 ? 16 : 8;
  if (const char *e = std::getenv("PSPMM_BLOCK_NW")) nw = std::atoi(e);
  if (!(nw == 15 || (rw == 8 && (nw == 19 || nw == 23)))) nw = 15;
  const int kNW = nw;  // the pack's consumer warps
  const int kR = kNW * rw, slots = kNW * rw;
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
  std::vector<int16_t> rowmap((size_t)nblk * slots, (int16_t)-1);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto par = [&](auto &&fn) {
    std::vector<std::thread> th;
    for (int t = 0; t < nth; ++t)
      th.emplace_back([&, t] {
        for (int64_t b = t; b < nblk; b += nth) fn(b);
      });
    for (auto &x : th) x.join();
  };
  // Per block: walk its touched windows in ascending order; for each, the
  // per-slot counts (row cursors advance monotonically, columns are sorted).
  auto walk = [&](int64_t b, auto &&on_window) {
    const int64_t r0 = b * kR, r1 = std::min(n, r0 + kR);
    std::vector<int32_t> wins;
    for (int64_t p = rp[r0]; p < rp[r1]; ++p) wins.push_back(ci[p] / kWc);
    std::sort(wins.begin(), wins.end());
    wins.erase(std::unique(wins.begin(), wins.end()), wins.end());
    std::vector<int64_t> cur(slots), end(slots);
    for (int q = 0; q < slots; ++q) {
      const int local = rowmap[(size_t)b * slots + q];
      cur[q] = local < 0 ? 0 : rp[r0 + local];
      end[q] = local < 0 ? 0 : rp[r0 + local + 1];
    }
    std::vector<int32_t> cnt(slots);
    for (int32_t w : wins) {
      const int32_t lim = (w + 1) * kWc;
      for (int q = 0; q < slots; ++q) {
        int64_t e = cur[q];
        while (e < end[q] && ci[e] < lim) ++e;
        cnt[q] = (int32_t)(e - cur[q]);
      }
      on_window(w, cnt, cur);  // cur[q] = first nonzero of slot q in this window
      for (int q = 0; q < slots; ++q) cur[q] += cnt[q];
    }
  };
  // pass 1: degree-balanced slots (rows by descending degree, dealt to the
  // warps in a snake order 0..14, 14..0, ..., slot = round), then the number
  // of virtual windows and padded pairs per block
  std::vector<int64_t> nvirt(nblk, 0), npairs(nblk, 0), nwins(nblk, 0);
  par([&](int64_t b) {
    const int64_t r0 = b * kR, r1 = std::min(n, r0 + kR);
    std::vector<int> idx(r1 - r0);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) {
      return rp[r0 + x + 1] - rp[r0 + x] > rp[r0 + y + 1] - rp[r0 + y];
    });
    for (size_t k = 0; k < idx.size(); ++k) {
      const int round = (int)(k / kNW), pos = (int)(k % kNW);
      const int w = (round & 1) ? kNW - 1 - pos : pos;
      rowmap[(size_t)b * slots + w * rw + round] = (int16_t)idx[k];
    }
    walk(b, [&](int32_t, const std::vector<int32_t> &cnt, const std::vector<int64_t> &) {
      // the same split as pass 2: runs padded to even, cut at kBlockMaxPairs
      int64_t v = 1, used = 0, T = 0;
      for (int32_t c : cnt) {
        while (c > 0) {
          if (used == kBlockMaxPairs) {
            ++v;
            used = 0;
          }
          const int take = (int)std::min<int64_t>(c, kBlockMaxPairs - used);
          used += take + (take & 1);
          T += take + (take & 1);
          c -= take;
        }
      }
      nvirt[b] += v;
      npairs[b] += T;
      nwins[b] += 1;
    });
  });
  std::vector<int32_t> win_ptr(nblk + 1, 0);
  std::vector<int64_t> pair_ptr(nblk + 1, 0);
  int64_t touched = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    win_ptr[b + 1] = win_ptr[b] + (int32_t)nvirt[b];
    pair_ptr[b + 1] = pair_ptr[b] + npairs[b];
    touched += nwins[b];
    if (win_ptr[b + 1] < win_ptr[b] || (int64_t)win_ptr[b + 1] != (int64_t)win_ptr[b] + nvirt[b])
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "attach_blocks: too many windows");
  }
  const int64_t W = win_ptr[nblk];
  // the per-window metadata must stay small next to the nonzeros: graphs
  // without in-block reuse (each window holding a handful of nonzeros) are
  // not this engine's (pspmm_decide_blocks would not pick it either)
  if ((double)W * (slots + 2 * kNW + 12) > 2.0 * 8.0 * (double)std::max<int64_t>(nnz, 1) + (1 << 20))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "attach_blocks: too little in-block reuse (window metadata would exceed 2x the "
               "packed nonzeros)");
  std::vector<int32_t> win_c0(W);
  std::vector<int64_t> win_pbase(W + 1);
  std::vector<uint8_t> win_cnt((size_t)W * slots, 0);
  std::vector<uint16_t> win_woff((size_t)W * kNW, 0);
  std::vector<int2> pairs(std::max<int64_t>(pair_ptr[nblk], 2), make_int2(0, 0));
  std::atomic<bool> bad{false};
  // pass 2: split each window's (warp, slot)-ordered nonzeros into virtual
  // windows and fill the stream
  par([&](int64_t b) {
    int64_t v = win_ptr[b], pos = pair_ptr[b];
    walk(b, [&](int32_t w, const std::vector<int32_t> &cnt, const std::vector<int64_t> &cur) {
      int64_t T = 0;
      for (int32_t c : cnt) T += c;
      int used = 0;
      win_c0[v] = w * kWc;
      win_pbase[v] = pos;
      int last_warp = -1;
      for (int q = 0; q < slots; ++q) {
        const int warp = q / rw, slot = q % rw;
        int64_t e = cur[q];
        int32_t c = cnt[q];
        while (c > 0) {
          if (used == kBlockMaxPairs) {  // close this virtual window, open the next
            for (int ww = last_warp + 1; ww < kNW; ++ww) win_woff[(size_t)v * kNW + ww] = used;
            ++v;
            win_c0[v] = w * kWc;
            win_pbase[v] = pos;
            used = 0;
            last_warp = -1;
          }
          if (warp != last_warp) {
            for (int ww = last_warp + 1; ww <= warp; ++ww) win_woff[(size_t)v * kNW + ww] = used;
            last_warp = warp;
          }
          const int take = std::min<int>(c, kBlockMaxPairs - used);
          win_cnt[(size_t)v * slots + q] = (uint8_t)take;
          for (int k = 0; k < take; ++k, ++e) {
            int32_t bits;
            std::memcpy(&bits, &vl[e], 4);
            pairs[pos++] = make_int2(ci[e] - w * kWc, bits);
          }
          if (take & 1) pairs[pos++] = make_int2(0, 0);  // runs padded to even (LDS.128 pairs)
          used += take + (take & 1);
          c -= take;
          (void)slot;
        }
      }
      for (int ww = last_warp + 1; ww < kNW; ++ww) win_woff[(size_t)v * kNW + ww] = used;
      ++v;
      (void)T;
    });
    if (v != win_ptr[b + 1] || pos != pair_ptr[b + 1]) bad = true;
  });
  if (bad) PSPMM_FAIL(PSPMM_ERR_CUDA, "attach_blocks: internal pack size mismatch");
  win_pbase[W] = pair_ptr[nblk];
  RowBlocks *R = new RowBlocks();
  struct Guard {
    RowBlocks *r;
    ~Guard() { destroy_blocks(r); }
  } guard{R};
  R->num_blocks = nblk;
  R->num_windows = touched;
  R->num_virtual = W;
  R->rw = rw;
  R->nw = nw;
  pspmm_status st;
  if ((st = upload(&R->d_win_ptr, win_ptr)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_c0, win_c0)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_pbase, win_pbase)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_cnt, win_cnt)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_win_woff, win_woff)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_pairs, pairs)) != PSPMM_OK) return st;
  if ((st = upload(&R->d_rowmap, rowmap)) != PSPMM_OK) return st;
  R->reuse = touched ? (double)nnz / ((double)touched * kWc) : 0.0;
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

namespace {
template <int RW, int NW>
pspmm_status launch_block(const CUtensorMap &map, const BlockArgs &args, int64_t nblk, int slices,
                          cudaStream_t stream) {
  const size_t smem = (size_t)kStages * kStage + 2 * kStages * sizeof(uint64_t);
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(spmm_block_kernel<RW, NW>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  spmm_block_kernel<RW, NW><<<(unsigned)(nblk * slices), (NW + 1) * 32, smem, stream>>>(map, args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}
}  // namespace

pspmm_status run_spmm_block(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, cudaStream_t stream, int32_t accumulate,
                            const Fanout &fan) {
  if (!block_supported(A, K, ldb, ldc, d_B, d_C))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run mode 5: needs pspmm_pcsr_attach_blocks on a V = 1, S = 0 handle, "
               "K % 128 == 0, ld % 4 == 0 and 16-B aligned B and C");
  const RowBlocks *R = A->blocks;
  if (R->num_blocks == 0) return PSPMM_OK;
  if (K / kKs > 65535 || R->num_blocks * (K / kKs) > 0x7fffffff)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run mode 5: grid too large");
  auto encode = get_encode_impl();
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
  BlockArgs args;
  args.win_ptr = R->d_win_ptr;
  args.win_c0 = R->d_win_c0;
  args.win_cnt = R->d_win_cnt;
  args.win_pbase = R->d_win_pbase;
  args.win_woff = R->d_win_woff;
  args.pairs = R->d_pairs;
  args.rowmap = R->d_rowmap;
  args.C = d_C;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.accumulate = accumulate;
  args.fan = fan;
  args.slices = K / kKs;
  const int sl = K / kKs;
  if (R->rw == 16) return launch_block<16, 15>(map, args, R->num_blocks, sl, stream);
  if (R->nw == 19) return launch_block<8, 19>(map, args, R->num_blocks, sl, stream);
  if (R->nw == 23) return launch_block<8, 23>(map, args, R->num_blocks, sl, stream);
  return launch_block<8, 15>(map, args, R->num_blocks, sl, stream);
}

}  // namespace pspmm
