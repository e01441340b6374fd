// (f3) The dense product of a GNN layer, T = X . W, on the tcgen05 tensor
// cores (a GCN / GIN layer is H' = A . H . W).
//
// X is n x Ki (row major, ldx), W is Ki x Ko (row major, ldw), T is n x Ko.
// With Ki, Ko ~ 64..256 the product moves 4 n (Ki + Ko) bytes for 2 n Ki Ko
// flops: 16 flop/B at Ki = Ko = 64, above the B200's FFMA / HBM balance
// (~11 flop/B), so on CUDA cores it is FFMA-bound (~26 us for Reddit's
// 233k x 64 x 64); on the tensor cores it is HBM-bound (~18 us).
//
// fp32 accuracy with TF32 inputs ("3xTF32"): x = hi + lo with hi = rna(x),
// lo = rna(x - hi); X.W ~ Xhi.Whi + Xhi.Wlo + Xlo.Whi (the dropped lo.lo
// term is below 2^-22 relative), accumulated in fp32 in TMEM.
//
// Default: gemm_tc_direct_kernel (below) — the TMA chunk is itself the A
// operand's hi part, splitters write only lo, epilogue by TMA tensor stores.
// gemm_tc_kernel (PSPMM_GEMM_DIRECT=0) is the raw-ring form described here.
// One persistent CTA per SM, warp-specialised (10 warps):
//  - warp 9 lane 0 (TMA): streams X in chunks of 128 rows x 32 columns
//    (16 KB, one 2-D TMA copy, 128-B swizzle, rows past n zero-filled) into
//    a ring of up to 8 raw stages, so up to 128 KB of X is in flight per SM
//    (thread-issued loads kept only 16 KB in flight: 1.8 TB/s);
//  - warps 0-3 (splitters): thread r owns row r of the chunk; it reads its
//    128 bytes from the raw stage (swizzled, conflict-free), splits them and
//    writes hi / lo into an operand stage in the no-swizzle K-major
//    core-matrix layout (core matrix = 8 rows x 16 B; consecutive rows 16 B
//    apart, so the stores are conflict-free), then fence.proxy.async and an
//    mbarrier arrive;
//  - warp 4 lane 0 (MMA): per chunk 4 K-steps x 3 tcgen05.mma.kind::tf32
//    (M = 128, N = Ko, K = 8) into one of two TMEM accumulators (2 x Ko
//    columns), tcgen05.commit frees the stage / publishes the accumulator;
//  - warps 5-8 (epilogue): tcgen05.ld 32x32b (warp w reads TMEM lanes
//    32 (w % 4) .. + 31 = rows of the tile), streaming stores of T, then
//    free the accumulator, so the next tile's MMAs overlap this epilogue.
//  W's hi / lo image (all of Ki x Ko) is split once per CTA into shared
//  memory by the loaders before the first tile.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kM = 128;                 // rows per tile (MMA M, TMEM lanes)
constexpr int kKc = 32;                 // X columns per chunk
constexpr int kChunkPart = kM * kKc * 4;  // one part (hi or lo) of a chunk: 16 KB
constexpr int kChunkBytes = 2 * kChunkPart;
constexpr int kRawBytes = kM * kKc * 4;  // one raw fp32 chunk: 16 KB
constexpr int kLoaders = 128, kEpi = 128;
constexpr int kThreads = kLoaders + 32 + kEpi + 32;  // 320: splitters, MMA, epilogue, TMA
constexpr int kOpStages = 4;  // default split-operand ring depth (fewer if smem is short)
constexpr int kMaxSmem = 227 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// UMMA shared-memory descriptor, no swizzle, K-major (as spmm_dense.cu):
// lbo = bytes between core matrices adjacent along K, sbo = along M / N.
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// UMMA descriptor of a K-major operand in the 128-B swizzle layout TMA
// writes (SWIZZLE_128B, layout type 2 at bits 61-63): 8-row x 128-B atoms,
// SBO = 1024 B between 8-row groups, LBO unused for swizzled K-major; a K
// step inside the 128-B row advances the start address (the hardware applies
// the XOR on the address bits, the stage base is 1024-B aligned).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;             // LBO (ignored)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
// kind::tf32 instruction descriptor: D fp32, A / B TF32, both K-major, M = 128
__device__ __forceinline__ uint32_t idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kM >> 4) << 24);
}
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split4(const float4 &x, float4 &hi, float4 &lo) {
  hi = make_float4(tf32_rn(x.x), tf32_rn(x.y), tf32_rn(x.z), tf32_rn(x.w));
  lo = make_float4(tf32_rn(x.x - hi.x), tf32_rn(x.y - hi.y), tf32_rn(x.z - hi.z),
                   tf32_rn(x.w - hi.w));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id,
                                         uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 16 columns of this thread's TMEM lane, no wait (the caller waits once for
// several loads: tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
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

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                       int r0) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0)
      : "memory");
}

struct GemmArgs {
  const float *__restrict__ X;
  const float *__restrict__ W;
  float *__restrict__ T;
  int64_t n, ldx, ldw, ldt;
  int32_t Ki, Ko, raw_stages, tmem_cols;
  int32_t stage_out;  // 1: the epilogue stages the tile in shared memory (coalesced rows)
  int32_t op_stages;  // split-operand ring depth (2..4)
};

__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap xmap, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int Ki = a.Ki, Ko = a.Ko, S = a.op_stages, R = a.raw_stages;
  const uint32_t wpart = (uint32_t)Ki * Ko * 4;  // one part of W's image
  uint8_t *raw0 = smem;                          // R x 16 KB raw X chunks (1 KB aligned)
  uint8_t *stage0 = raw0 + (size_t)R * kRawBytes;  // S x [hi 16 KB | lo 16 KB]
  uint8_t *wimg = stage0 + (size_t)S * kChunkBytes;  // [hi | lo], each [Ki/4][Ko][4]
  uint8_t *otile = wimg + 2 * wpart;  // stage_out: 128 rows x Ko fp32, 16-B chunks swizzled
  uint64_t *bar = reinterpret_cast<uint64_t *>(otile + (a.stage_out ? (size_t)kM * Ko * 4 : 0));
  uint64_t *full = bar, *empty = bar + S, *accf = bar + 2 * S, *acce = bar + 2 * S + 2;
  uint64_t *rfull = bar + 2 * S + 4, *rempty = rfull + R;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rempty + R);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tiles = (a.n + kM - 1) / kM;
  const int chunks = Ki / kKc;

  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], kLoaders);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kEpi);
    }
    for (int r = 0; r < R; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], kLoaders);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // W -> hi / lo image: element (k, n) at [k / 4][n][k % 4]; every thread
  // has 8 W loads in flight before it splits and stores them
  {
    const int q = Ko / 4;  // float4 per W row
    const int total = Ki * q;
    for (int base = tid; base < total; base += kThreads * 8) {
      float4 w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * kThreads;
        w[u] = i < total ? __ldg(reinterpret_cast<const float4 *>(a.W + (int64_t)(i / q) * a.ldw +
                                                                   4 * (i % q)))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * kThreads;
        if (i >= total) break;
        const int k = i / q, n4 = i % q;
        float4 hi, lo;
        split4(w[u], hi, lo);
        const float h[4] = {hi.x, hi.y, hi.z, hi.w}, l[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t off = ((uint32_t)(k >> 2) * Ko + 4 * n4 + e) * 16 + (k & 3) * 4;
          *reinterpret_cast<float *>(wimg + off) = h[e];
          *reinterpret_cast<float *>(wimg + wpart + off) = l[e];
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 9) {  // TMA producer: raw X chunks
    if (lane == 0) {
      int it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int c = 0; c < chunks; ++c, ++it) {
          const int r = it % R;
          if (it >= R) mbar_wait(&rempty[r], ((it / R) - 1) & 1);
          mbar_expect_tx(&rfull[r], kRawBytes);
          tma_2d(smem_u32(raw0 + (size_t)r * kRawBytes), &xmap, &rfull[r], c * kKc, (int)(t * kM));
        }
    }
    __syncwarp();
  } else if (warp < 4) {  // splitters: thread tid owns row tid of each chunk
    int it = 0;           // chunk counter across tiles (both rings advance together)
    const uint32_t sw = (uint32_t)(tid & 7);
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int c = 0; c < chunks; ++c, ++it) {
        const int r = it % R, s = it % S;
        mbar_wait(&rfull[r], (it / R) & 1);
        const uint8_t *rw = raw0 + (size_t)r * kRawBytes + tid * 128;
        float4 x[8];
#pragma unroll
        for (int g = 0; g < 8; ++g)  // 128-B swizzle: chunk g of row i at g ^ (i % 8)
          x[g] = *reinterpret_cast<const float4 *>(rw + ((g ^ sw) << 4));
        // the raw stage is refilled by the TMA (async proxy) after this
        // release: order the generic reads before it (WAR across proxies)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&rempty[r]);
        if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
        uint8_t *st = stage0 + (size_t)s * kChunkBytes;
#pragma unroll
        for (int g = 0; g < 8; ++g) {  // core-matrix layout: [k-group][row][16 B]
          float4 hi, lo;
          split4(x[g], hi, lo);
          *reinterpret_cast<float4 *>(st + g * (kM * 16) + tid * 16) = hi;
          *reinterpret_cast<float4 *>(st + kChunkPart + g * (kM * 16) + tid * 16) = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&full[s]);
      }
    }
  } else if (warp == 4) {  // MMA issuer
    if (lane == 0) {
      const uint32_t id = idesc(Ko);
      const uint32_t bytes_b = (uint32_t)Ko * 16;  // one K group of W (Ko x 16 B)
      const uint32_t whi = smem_u32(wimg), wlo = whi + wpart;
      int it = 0, tl = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
        const int b = tl & 1;
        if (tl >= 2) mbar_wait(&acce[b], ((tl >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(b * Ko);
        for (int c = 0; c < chunks; ++c, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t xhi = smem_u32(stage0 + (size_t)s * kChunkBytes), xlo = xhi + kChunkPart;
#pragma unroll
          for (int ks = 0; ks < kKc / 8; ++ks) {
            const uint32_t oa = ks * 2 * (kM * 16);
            const uint32_t ob = (uint32_t)(c * (kKc / 4) + 2 * ks) * bytes_b;
            const uint64_t dah = desc(xhi + oa, kM * 16, 128), dal = desc(xlo + oa, kM * 16, 128);
            const uint64_t dbh = desc(whi + ob, bytes_b, 128), dbl = desc(wlo + ob, bytes_b, 128);
            mma_tf32(acc, dah, dbh, id, (c > 0 || ks > 0) ? 1u : 0u);
            mma_tf32(acc, dah, dbl, id, 1u);
            mma_tf32(acc, dal, dbh, id, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accf[b]);
      }
    }
    __syncwarp();
  } else {  // epilogue (warps 5-8): warp w reads TMEM lanes 32 (w % 4) .. + 31
    const int quarter = warp & 3;
    int tl = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
      const int b = tl & 1;
      mbar_wait(&accf[b], (tl >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int rloc = quarter * 32 + lane;
      const int64_t row = t * kM + rloc;
      const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * Ko);
      if (a.stage_out) {
        // TMEM -> shared tile (thread = row; 16-B chunk j of row r stored at
        // chunk j ^ (r % 8) of its 128-B group: 4 wavefronts per warp store)
        const int q = Ko / 4;  // 16-B chunks per row
        for (int c0 = 0; c0 < Ko; c0 += 64) {  // up to 4 loads in flight, one wait
          uint32_t v[4][16];
          const int nc = Ko - c0 < 64 ? (Ko - c0) / 16 : 4;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < nc) tmem_ld16_nowait(tb + c0 + 16 * u, v[u]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < nc) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int ch = (c0 + 16 * u) / 4 + j, sw = (ch & ~7) | ((ch ^ rloc) & 7);
                *reinterpret_cast<uint4 *>(otile + ((size_t)rloc * q + sw) * 16) =
                    make_uint4(v[u][4 * j], v[u][4 * j + 1], v[u][4 * j + 2], v[u][4 * j + 3]);
              }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&acce[b]);  // TMEM buffer free: the next tile's MMAs may start
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        // shared tile -> T, row-contiguous: a warp stores 512 consecutive bytes
        const int e = tid - (kLoaders + 32);  // 0..127
        for (int idx = e; idx < kM * q; idx += kEpi) {
          const int r = idx / q, ch = idx % q, sw = (ch & ~7) | ((ch ^ r) & 7);
          const int64_t grow = t * kM + r;
          if (grow < a.n) {
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(smem_u32(otile + ((size_t)r * q + sw) * 16)));
            __stcs(reinterpret_cast<float4 *>(a.T + grow * a.ldt) + ch, v);
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        continue;
      }
      for (int c = 0; c < Ko; c += 16) {
        float v[16];
        tmem_ld16(tb + c, v);
        if (row < a.n) {
          float4 *dst = reinterpret_cast<float4 *>(a.T + row * a.ldt + c);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcs(dst + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acce[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(a.tmem_cols));
}

// The direct form (default): the TMA's 128-B-swizzled X chunk IS the A
// operand's hi part (kind::tf32 reads the fp32 bits and keeps the top 19:
// hi = trunc(x)); the splitters only write lo = x - trunc(x), exact in fp32,
// into the stage's second half in the same swizzled layout.  A stage is
// [X chunk 16 KB (TMA) | lo 16 KB], freed by the MMA's commit, so every
// stage's TMA is in flight with no separate raw ring.  (The dropped terms:
// lo's own truncation and lo.lo, each < 2^-20 relative per product, inside
// the c-1 bound.)
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_direct_kernel(const __grid_constant__ CUtensorMap xmap,
                          const __grid_constant__ CUtensorMap tmap, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int Ki = a.Ki, Ko = a.Ko, S = a.op_stages;
  const uint32_t wpart = (uint32_t)Ki * Ko * 4;
  uint8_t *stage0 = smem;                             // S x [X 16 KB | lo 16 KB]
  uint8_t *wimg = stage0 + (size_t)S * kChunkBytes;   // [hi | lo], each [Ki/4][Ko][4]
  uint8_t *otile = wimg + 2 * wpart;  // stage_out: 2 x [Ko/32 blocks of 128 rows x 128 B]
  uint64_t *bar =
      reinterpret_cast<uint64_t *>(otile + (a.stage_out ? 2 * (size_t)kM * Ko * 4 : 0));
  uint64_t *xfull = bar, *lofull = bar + S, *empty = bar + 2 * S, *accf = bar + 3 * S,
           *acce = bar + 3 * S + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tiles = (a.n + kM - 1) / kM;
  const int chunks = Ki / kKc;

  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&lofull[s], kLoaders);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {  // W -> hi / lo image (as gemm_tc_kernel)
    const int q = Ko / 4;
    const int total = Ki * q;
    for (int base = tid; base < total; base += kThreads * 8) {
      float4 w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * kThreads;
        w[u] = i < total ? __ldg(reinterpret_cast<const float4 *>(a.W + (int64_t)(i / q) * a.ldw +
                                                                   4 * (i % q)))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * kThreads;
        if (i >= total) break;
        const int k = i / q, n4 = i % q;
        float4 hi, lo;
        split4(w[u], hi, lo);
        const float h[4] = {hi.x, hi.y, hi.z, hi.w}, l[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t off = ((uint32_t)(k >> 2) * Ko + 4 * n4 + e) * 16 + (k & 3) * 4;
          *reinterpret_cast<float *>(wimg + off) = h[e];
          *reinterpret_cast<float *>(wimg + wpart + off) = l[e];
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 9) {  // TMA producer
    if (lane == 0) {
      int it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int c = 0; c < chunks; ++c, ++it) {
          const int s = it % S;
          if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
          mbar_expect_tx(&xfull[s], kChunkPart);
          tma_2d(smem_u32(stage0 + (size_t)s * kChunkBytes), &xmap, &xfull[s], c * kKc,
                 (int)(t * kM));
        }
    }
    __syncwarp();
  } else if (warp < 4) {  // splitters: lo = x - trunc(x), same swizzled position
    int it = 0;
    const uint32_t sw = (uint32_t)(tid & 7);
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int c = 0; c < chunks; ++c, ++it) {
        const int s = it % S;
        mbar_wait(&xfull[s], (it / S) & 1);
        const uint32_t xr = smem_u32(stage0 + (size_t)s * kChunkBytes) + tid * 128;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const uint32_t o = ((g ^ sw) << 4);
          uint4 x;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                       : "r"(xr + o));
          const float4 lo = make_float4(
              __uint_as_float(x.x) - __uint_as_float(x.x & 0xFFFFE000u),
              __uint_as_float(x.y) - __uint_as_float(x.y & 0xFFFFE000u),
              __uint_as_float(x.z) - __uint_as_float(x.z & 0xFFFFE000u),
              __uint_as_float(x.w) - __uint_as_float(x.w & 0xFFFFE000u));
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(xr + kChunkPart + o),
                       "f"(lo.x), "f"(lo.y), "f"(lo.z), "f"(lo.w)
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&lofull[s]);
      }
    }
  } else if (warp == 4) {  // MMA issuer
    if (lane == 0) {
      const uint32_t id = idesc(Ko);
      const uint32_t bytes_b = (uint32_t)Ko * 16;
      const uint32_t whi = smem_u32(wimg), wlo = whi + wpart;
      int it = 0, tl = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
        const int b = tl & 1;
        if (tl >= 2) mbar_wait(&acce[b], ((tl >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(b * Ko);
        for (int c = 0; c < chunks; ++c, ++it) {
          const int s = it % S;
          mbar_wait(&lofull[s], (it / S) & 1);  // the splitters saw xfull: X landed too
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t xhi = smem_u32(stage0 + (size_t)s * kChunkBytes), xlo = xhi + kChunkPart;
#pragma unroll
          for (int ks = 0; ks < kKc / 8; ++ks) {
            const uint64_t dah = desc_sw128(xhi + ks * 32), dal = desc_sw128(xlo + ks * 32);
            const uint32_t ob = (uint32_t)(c * (kKc / 4) + 2 * ks) * bytes_b;
            const uint64_t dbh = desc(whi + ob, bytes_b, 128), dbl = desc(wlo + ob, bytes_b, 128);
            mma_tf32(acc, dah, dbh, id, (c > 0 || ks > 0) ? 1u : 0u);
            mma_tf32(acc, dah, dbl, id, 1u);
            mma_tf32(acc, dal, dbh, id, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accf[b]);
      }
    }
    __syncwarp();
  } else {  // epilogue (warps 5-8), as gemm_tc_kernel
    const int quarter = warp & 3;
    int tl = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
      const int b = tl & 1;
      mbar_wait(&accf[b], (tl >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int rloc = quarter * 32 + lane;
      const int64_t row = t * kM + rloc;
      const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * Ko);
      if (a.stage_out) {
        // TMEM -> shared tile in the TMA store's 128-B swizzle (32-column
        // blocks of 128 rows x 128 B; chunk j of row r at j ^ (r % 8)), then
        // one elected thread stores the tile with TMA tensor stores; two
        // tile buffers, so a store drains while the next tile is staged
        uint8_t *ot = otile + (size_t)(tl & 1) * kM * Ko * 4;
        const bool leader = tid == kLoaders + 32;
        if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        for (int c0 = 0; c0 < Ko; c0 += 64) {
          uint32_t v[4][16];
          const int nc = Ko - c0 < 64 ? (Ko - c0) / 16 : 4;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < nc) tmem_ld16_nowait(tb + c0 + 16 * u, v[u]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < nc) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int col = c0 + 16 * u + 4 * j;  // first column of this 16-B chunk
                const int blk = col >> 5, ch = (col & 31) >> 2;
                const uint32_t addr = smem_u32(ot + (size_t)blk * kM * 128 + rloc * 128 +
                                               ((ch ^ (rloc & 7)) << 4));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                             "r"(v[u][4 * j]), "r"(v[u][4 * j + 1]), "r"(v[u][4 * j + 2]),
                             "r"(v[u][4 * j + 3])
                             : "memory");
              }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&acce[b]);  // TMEM buffer free: the next tile's MMAs may start
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        if (leader) {
          for (int blk = 0; blk < Ko / 32; ++blk)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmap)),
                "r"(blk * 32), "r"((int)(t * kM)), "r"(smem_u32(ot + (size_t)blk * kM * 128))
                : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        continue;
      }
      for (int c = 0; c < Ko; c += 16) {
        float v[16];
        tmem_ld16(tb + c, v);
        if (row < a.n) {
          float4 *dst = reinterpret_cast<float4 *>(a.T + row * a.ldt + c);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcs(dst + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acce[b]);
    }
  }
  if (a.stage_out && tid == kLoaders + 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(a.tmem_cols));
}

int tmem_cols_for(int Ko) {
  int c = 32;
  while (c < 2 * Ko) c <<= 1;
  return c;
}

}  // namespace

// Shapes the tensor-core product takes: Ki % 32 == 0, Ko % 16 == 0,
// 16 <= Ko <= 256, W's hi / lo image plus two X stages in shared memory,
// 16-B aligned X / W / T with ld % 4 == 0.
// Output-column block width so W's hi / lo image (Ki x Kob x 8 B) fits beside
// two stages and N = Kob <= 256: Ko itself when it fits, else the widest
// divisor of Ko that is a multiple of 16 and fits
// (each block is then an independent launch over the same X: X re-streams).
int gemm_tc_block(int32_t Ki, int32_t Ko) {
  for (int b = std::min(Ko, 256); b >= 16; b -= 16) {  // MMA N <= 256, TMEM 2 x N <= 512
    if (Ko % b != 0) continue;
    if (2ll * Ki * b * 4 + 2ll * kChunkBytes + 2ll * kRawBytes + 1024 + 512 <= kMaxSmem) return b;
  }
  return 0;
}

bool gemm_tc_supported(int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx, const float *d_W,
                       int64_t ldw, const float *d_T, int64_t ldt) {
  if (Ki < kKc || Ki % kKc != 0 || Ko < 16 || Ko % 16 != 0) return false;
  if (gemm_tc_block(Ki, Ko) == 0) return false;
  if (ldx % 4 || ldw % 4 || ldt % 4) return false;
  if ((reinterpret_cast<uintptr_t>(d_X) | reinterpret_cast<uintptr_t>(d_W) |
       reinterpret_cast<uintptr_t>(d_T)) & 15)
    return false;
  if (!tensor_map_encoder()) return false;
  return true;
}

pspmm_status gemm_tc_one(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                         const float *d_W, int64_t ldw, float *d_T, int64_t ldt,
                         cudaStream_t stream);

pspmm_status gemm_tc(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                     const float *d_W, int64_t ldw, float *d_T, int64_t ldt, cudaStream_t stream) {
  if (n == 0) return PSPMM_OK;
  const int b = gemm_tc_block(Ki, Ko);
  if (b <= 0) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "dense_gemm: no tensor-core column block fits");
  for (int j0 = 0; j0 < Ko; j0 += b) {  // T[:, j0:j0+b] = X . W[:, j0:j0+b]
    pspmm_status st = gemm_tc_one(n, Ki, std::min(b, Ko - j0), d_X, ldx, d_W + j0, ldw, d_T + j0,
                                  ldt, stream);
    if (st != PSPMM_OK) return st;
  }
  return PSPMM_OK;
}

pspmm_status gemm_tc_one(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                         const float *d_W, int64_t ldw, float *d_T, int64_t ldt,
                         cudaStream_t stream) {
  if (n > 0x7fffffffll) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "dense_gemm: n >= 2^31");
  const int64_t w = 2ll * Ki * Ko * 4;
  // the staged epilogue (coalesced row stores) when its tile fits beside two
  // raw stages (Ko % 32 == 0, so 16-B chunks swizzle within 128-B groups)
  int ops = kOpStages;
  if (const char *e = std::getenv("PSPMM_GEMM_OPS"))  // A/B knob for the tools (2..4)
    ops = std::max(2, std::min(4, std::atoi(e)));
  while (ops > 2 && 1024 + 512 + w + (int64_t)ops * kChunkBytes + 2ll * kRawBytes > kMaxSmem) --ops;
  const int64_t base = 1024 + 512 + w + (int64_t)ops * kChunkBytes;
  const int64_t otile = (int64_t)kM * Ko * 4;
  const char *se = std::getenv("PSPMM_GEMM_STAGE_OUT");  // A/B knob for the tools (0 = off)
  const bool stage_out = !(se && se[0] == '0') && Ko % 32 == 0 &&
                         base + otile + 2ll * kRawBytes <= kMaxSmem;
  int raw = (int)std::min<int64_t>(8, (kMaxSmem - base - (stage_out ? otile : 0)) / kRawBytes);
  if (const char *e = std::getenv("PSPMM_GEMM_RAW"))  // A/B knob for the tools (2..raw)
    raw = std::max(2, std::min(raw, std::atoi(e)));
  const size_t smem = (size_t)(base + (stage_out ? otile : 0) + (int64_t)raw * kRawBytes);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) PSPMM_FAIL(PSPMM_ERR_CUDA, "dense_gemm: cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)Ki, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
  cuuint32_t box[2] = {(cuuint32_t)kKc, (cuuint32_t)kM};
  cuuint32_t estr[2] = {1, 1};
  if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(d_X), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    PSPMM_FAIL(PSPMM_ERR_CUDA, "dense_gemm: tensor map encode failed");
  GemmArgs args;
  args.X = d_X;
  args.W = d_W;
  args.T = d_T;
  args.n = n;
  args.ldx = ldx;
  args.ldw = ldw;
  args.ldt = ldt;
  args.Ki = Ki;
  args.Ko = Ko;
  args.raw_stages = raw;
  args.stage_out = stage_out ? 1 : 0;
  args.op_stages = ops;
  args.tmem_cols = tmem_cols_for(Ko);
  const int64_t tiles = (n + kM - 1) / kM;
  const int grid = (int)std::min<int64_t>(tiles, num_sms());
  // the direct form (TMA chunk = hi operand, default) with as many 32-KB
  // stages as fit (2..6); PSPMM_GEMM_DIRECT=0 (A/B knob) takes the raw-ring form
  const char *de = std::getenv("PSPMM_GEMM_DIRECT");
  if (!(de && de[0] == '0')) {
    // the direct form's staged epilogue: two tile buffers written out by TMA
    // tensor stores (Ko % 32 == 0)
    bool so = !(se && se[0] == '0') && Ko % 32 == 0 &&
              1024 + 512 + w + 2 * otile + 2ll * kChunkBytes <= kMaxSmem;
    const int64_t base_d = 1024 + 512 + w + (so ? 2 * otile : 0);
    int sd = (int)std::min<int64_t>(6, (kMaxSmem - base_d) / kChunkBytes);
    if (const char *e = std::getenv("PSPMM_GEMM_OPS")) sd = std::max(2, std::min(sd, std::atoi(e)));
    CUtensorMap tmapT;
    if (so) {
      cuuint64_t tdims[2] = {(cuuint64_t)Ko, (cuuint64_t)n};
      cuuint64_t tstr[1] = {(cuuint64_t)ldt * 4};
      cuuint32_t tbox[2] = {32, (cuuint32_t)kM};
      if (encode(&tmapT, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d_T, tdims, tstr, tbox, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        so = false;
    }
    if (!so) std::memset(&tmapT, 0, sizeof(tmapT));
    if (sd >= 2) {
      args.op_stages = sd;
      args.stage_out = so ? 1 : 0;
      const size_t smem_d = (size_t)(base_d + (int64_t)sd * kChunkBytes);
      PSPMM_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_direct_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d));
      gemm_tc_direct_kernel<<<grid, kThreads, smem_d, stream>>>(map, tmapT, args);
      PSPMM_CUDA_TRY(cudaGetLastError());
      return PSPMM_OK;
    }
  }
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  gemm_tc_kernel<<<grid, kThreads, smem, stream>>>(map, args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
