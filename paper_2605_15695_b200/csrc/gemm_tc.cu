// (f3) The dense product of a GNN layer, T = X . W, on the tcgen05 tensor
// cores (a GCN / GIN layer is H' = A . H . W).
//
// X is n x Ki (row major, ldx), W is Ki x Ko (row major, ldw), T is n x Ko.
// With Ki, Ko ~ 64..256 the product moves 4 n (Ki + Ko) bytes for 2 n Ki Ko
// flops: 16 flop/B at Ki = Ko = 64, above the B200's FFMA / HBM balance
// (~11 flop/B), so on CUDA cores it is FFMA-bound (~26 us for Reddit's
// 233k x 64 x 64); on the tensor cores it is HBM-bound (~18 us).
//
// fp32 accuracy with TF32 inputs ("3xTF32"): x = hi + lo; X.W ~ Xhi.Whi +
// Xhi.Wlo + Xlo.Whi, accumulated in fp32 in TMEM (X: hi = trunc(x), below;
// W: hi = rna(w), lo = rna(w - hi)).
//
// One persistent CTA per SM, warp-specialised (10 warps), two rings:
//  - warp 9 lane 0 (TMA): streams X in chunks of 128 rows x 32 columns (16 KB,
//    one 2-D TMA copy, 128-B swizzle, rows past n zero-filled) into a ring of
//    up to 8 X stages; it starts before W's image is built.  The chunk as the
//    TMA wrote it IS the A operand's hi part: kind::tf32 reads the fp32 bits
//    and keeps the top 19, so hi = trunc(x) (a K-major SWIZZLE_128B UMMA
//    descriptor);
//  - warps 0-3 (splitters): thread r owns row r of the chunk and writes
//    lo = x - trunc(x) (exact in fp32) into a buffer of the lo ring, in the
//    same swizzled layout, then fence.proxy.async and an mbarrier arrive;
//  - warp 4 lane 0 (MMA): per chunk 4 K-steps of tcgen05.mma.kind::tf32
//    (M = 128, K = 8) into one of two TMEM accumulators: Xhi.[Whi | Wlo] as
//    one N = 2 Ko MMA plus Xlo.Whi (N = Ko) into its first half when
//    2 Ko <= 256 (the epilogue adds the halves), else three N = Ko MMAs
//    (Xhi.Whi + Xhi.Wlo + Xlo.Whi); tcgen05.commit frees the X stage and
//    the lo buffer, and publishes the accumulator;
//  - warps 5-8 (epilogue): tcgen05.ld 32x32b (warp w reads TMEM lanes
//    32 (w % 4) .. + 31 = rows of the tile), the tile written into a
//    128-B-swizzled shared buffer and stored by one thread with TMA tensor
//    stores (one buffer by default: the next tile is staged once the store
//    has read it; two on request), and the next tile's MMAs overlap this
//    epilogue.
// W's rna hi / lo image (all of Ki x Ko, or a column block of it) is built
// once per CTA in shared memory.  For Ko == 128 (and 128-column blocks of
// wider W) with Ki <= 128, gemm_tc_wt_kernel computes T^T = W^T . X^T with
// W^T as the A operand in tensor memory instead, which frees shared memory
// for the rings.  The dropped terms (lo's own truncation,
// lo.lo) are < 2^-20 relative per product, inside the c-1 bound.
// History and measurements: DESIGN.md section 5 (a plain device copy of the
// same bytes is the practical ceiling at these sizes).
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
constexpr int kLoaders = 128, kEpi = 128;
constexpr int kThreads = kLoaders + 32 + kEpi + 32;  // 320: splitters, MMA, epilogue, TMA
constexpr int kMaxSmem = 227 * 1024;
constexpr int kSmemSlack = 1024 + 512;  // 1-KB alignment of the rings + barriers

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

// The TMA producer of both kernels: X chunk (tile t, chunk c) into X stage
// it % SX once the MMA has released the stage's previous use.
__device__ __forceinline__ void tma_x_loop(const CUtensorMap *xmap, int64_t tiles, int chunks,
                                           int SX, uint8_t *xst0, uint64_t *xfull,
                                           uint64_t *xempty) {
  int it = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
    for (int c = 0; c < chunks; ++c, ++it) {
      const int s = it % SX;
      if (it >= SX) mbar_wait(&xempty[s], ((it / SX) - 1) & 1);
      mbar_expect_tx(&xfull[s], kChunkPart);
      tma_2d(smem_u32(xst0 + (size_t)s * kChunkPart), xmap, &xfull[s], c * kKc, (int)(t * kM));
    }
}

// The splitters of both kernels (warps 0-3, thread = row of the chunk): for
// every X chunk, lo = x - trunc(x) (exact in fp32) into lo buffer it % SL,
// in the chunk's own 128-B swizzle, then a proxy fence and an arrive.
__device__ __forceinline__ void split_loop(int tid, int64_t tiles, int chunks, int SX, int SL,
                                           const uint8_t *xst0, uint8_t *lost0, uint64_t *xfull,
                                           uint64_t *lofull, uint64_t *loempty) {
  int it = 0;
  const uint32_t sw = (uint32_t)(tid & 7);
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int c = 0; c < chunks; ++c, ++it) {
      const int sx = it % SX, sl = it % SL;
      mbar_wait(&xfull[sx], (it / SX) & 1);
      if (it >= SL) mbar_wait(&loempty[sl], ((it / SL) - 1) & 1);
      const uint32_t xr = smem_u32(xst0 + (size_t)sx * kChunkPart) + tid * 128;
      const uint32_t lr = smem_u32(lost0 + (size_t)sl * kChunkPart) + tid * 128;
      uint4 x[8];
#pragma unroll
      for (int g = 0; g < 8; ++g)
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x[g].x), "=r"(x[g].y), "=r"(x[g].z), "=r"(x[g].w)
                     : "r"(xr + ((g ^ sw) << 4)));
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 lo = make_float4(
            __uint_as_float(x[g].x) - __uint_as_float(x[g].x & 0xFFFFE000u),
            __uint_as_float(x[g].y) - __uint_as_float(x[g].y & 0xFFFFE000u),
            __uint_as_float(x[g].z) - __uint_as_float(x[g].z & 0xFFFFE000u),
            __uint_as_float(x[g].w) - __uint_as_float(x[g].w & 0xFFFFE000u));
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lr + ((g ^ sw) << 4)),
                     "f"(lo.x), "f"(lo.y), "f"(lo.z), "f"(lo.w)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&lofull[sl]);
    }
  }
}

struct GemmArgs {
  const float *__restrict__ X;
  const float *__restrict__ W;
  float *__restrict__ T;
  int64_t n, ldx, ldw, ldt;
  int32_t Ki, Ko, tmem_cols;
  int32_t x_stages;   // X ring depth (16 KB each)
  int32_t lo_stages;  // lo ring depth (16 KB each)
  int32_t out_bufs;   // staged output tiles for the TMA-store epilogue (0..2)
  int32_t fuse;       // 1: Xhi.[Whi | Wlo] as one N = 2 Ko MMA (2 Ko <= 256)
};

// The kernel (file header): the X chunks (the hi operand) and the lo chunks
// live in two rings of their own, so a stage of X costs 16 KB and up to 8 X
// chunks are in flight per SM with only 2-3 lo buffers; the TMA warp starts
// streaming X while the other warps build W's image.
// Barriers: xfull (TMA tx) / xempty (MMA commit) per X stage, lofull (the
// 128 splitters) / loempty (MMA commit) per lo buffer; ring depths in
// GemmArgs (x_stages, lo_stages, out_bufs).
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_ring_kernel(const __grid_constant__ CUtensorMap xmap,
                        const __grid_constant__ CUtensorMap tmap, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int Ki = a.Ki, Ko = a.Ko, SX = a.x_stages, SL = a.lo_stages, OB = a.out_bufs;
  const uint32_t wpart = (uint32_t)Ki * Ko * 4;
  uint8_t *xst0 = smem;                              // SX x 16 KB X chunks
  uint8_t *lost0 = xst0 + (size_t)SX * kChunkPart;   // SL x 16 KB lo chunks
  uint8_t *otile = lost0 + (size_t)SL * kChunkPart;  // OB x [Ko/32 blocks of 128 rows x 128 B]
  uint8_t *wimg = otile + (size_t)OB * kM * Ko * 4;  // [hi | lo], each [Ki/4][Ko][4]
  uint64_t *bar = reinterpret_cast<uint64_t *>(wimg + 2 * (size_t)wpart);
  uint64_t *xfull = bar, *xempty = bar + SX, *lofull = bar + 2 * SX, *loempty = lofull + SL;
  uint64_t *accf = loempty + SL, *acce = accf + 2;
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
    for (int s = 0; s < SX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < SL; ++s) {
      mbar_init(&lofull[s], kLoaders);
      mbar_init(&loempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();  // barriers initialised, TMEM address published

  if (warp == 9) {  // TMA producer: starts at once
    if (lane == 0) tma_x_loop(&xmap, tiles, chunks, SX, xst0, xfull, xempty);
    __syncwarp();
  } else {
    {  // W -> hi / lo image (warps 0-8), then a barrier among those warps only
      const int nt = kThreads - 32;
      const int q = Ko / 4;
      const int total = Ki * q;
      for (int base = tid; base < total; base += nt * 8) {
        float4 w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * nt;
          w[u] = i < total ? __ldg(reinterpret_cast<const float4 *>(
                                 a.W + (int64_t)(i / q) * a.ldw + 4 * (i % q)))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = base + u * nt;
          if (i >= total) break;
          const int k = i / q, n4 = i % q;
          float4 hi, lo;
          split4(w[u], hi, lo);
          const float h[4] = {hi.x, hi.y, hi.z, hi.w}, l[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (a.fuse) {  // one [Ki/4][2 Ko][4] image: hi at n, lo at Ko + n
              const uint32_t off = ((uint32_t)(k >> 2) * 2 * Ko + 4 * n4 + e) * 16 + (k & 3) * 4;
              *reinterpret_cast<float *>(wimg + off) = h[e];
              *reinterpret_cast<float *>(wimg + off + (uint32_t)Ko * 16) = l[e];
            } else {
              const uint32_t off = ((uint32_t)(k >> 2) * Ko + 4 * n4 + e) * 16 + (k & 3) * 4;
              *reinterpret_cast<float *>(wimg + off) = h[e];
              *reinterpret_cast<float *>(wimg + wpart + off) = l[e];
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 2, %0;" ::"r"(kThreads - 32) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // splitters
      split_loop(tid, tiles, chunks, SX, SL, xst0, lost0, xfull, lofull, loempty);
    } else if (warp == 4) {  // MMA issuer
      if (lane == 0) {
        const uint32_t id = idesc(Ko), id2 = idesc(2 * Ko);
        const uint32_t bytes_b = (uint32_t)Ko * 16 * (a.fuse ? 2 : 1);
        const uint32_t whi = smem_u32(wimg), wlo = whi + wpart;
        int it = 0, tl = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
          const int b = tl & 1;
          if (tl >= 2) mbar_wait(&acce[b], ((tl >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t acc = tmem + (uint32_t)(b * Ko * (a.fuse ? 2 : 1));
          for (int c = 0; c < chunks; ++c, ++it) {
            const int sx = it % SX, sl = it % SL;
            mbar_wait(&lofull[sl], (it / SL) & 1);  // the splitters saw xfull: X landed too
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t xhi = smem_u32(xst0 + (size_t)sx * kChunkPart);
            const uint32_t xlo = smem_u32(lost0 + (size_t)sl * kChunkPart);
#pragma unroll
            for (int ks = 0; ks < kKc / 8; ++ks) {
              const uint64_t dah = desc_sw128(xhi + ks * 32), dal = desc_sw128(xlo + ks * 32);
              const uint32_t ob = (uint32_t)(c * (kKc / 4) + 2 * ks) * bytes_b;
              if (a.fuse) {
                // N = 2 Ko: D[:, 0:Ko] = Xhi.Whi, D[:, Ko:2Ko] = Xhi.Wlo in one
                // MMA (X_hi read once); then D[:, 0:Ko] += Xlo.Whi (N = Ko)
                const uint64_t dbw = desc(whi + ob, bytes_b, 128);
                mma_tf32(acc, dah, dbw, id2, (c > 0 || ks > 0) ? 1u : 0u);
                mma_tf32(acc, dal, dbw, id, 1u);
              } else {
                const uint64_t dbh = desc(whi + ob, bytes_b, 128), dbl = desc(wlo + ob, bytes_b, 128);
                mma_tf32(acc, dah, dbh, id, (c > 0 || ks > 0) ? 1u : 0u);
                mma_tf32(acc, dah, dbl, id, 1u);
                mma_tf32(acc, dal, dbh, id, 1u);
              }
            }
            mma_commit(&xempty[sx]);
            mma_commit(&loempty[sl]);
          }
          mma_commit(&accf[b]);
        }
      }
      __syncwarp();
    } else {  // epilogue (warps 5-8), OB staged tile buffers
      const int quarter = warp & 3;
      const bool leader = tid == kLoaders + 32;
      int tl = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
        const int b = tl & 1;
        mbar_wait(&accf[b], (tl >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int rloc = quarter * 32 + lane;
        const int64_t row = t * kM + rloc;
        const uint32_t tb =
            tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * Ko * (a.fuse ? 2 : 1));
        if (OB > 0) {
          uint8_t *ot = otile + (size_t)(OB == 2 ? (tl & 1) : 0) * kM * Ko * 4;
          if (leader) {
            if (OB == 2)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
          const int step = a.fuse ? 32 : 64;  // fused: the Xhi.Wlo half loads beside
          for (int c0 = 0; c0 < Ko; c0 += step) {
            uint32_t v[4][16];
            const int nc = Ko - c0 < step ? (Ko - c0) / 16 : step / 16;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < nc) tmem_ld16_nowait(tb + c0 + 16 * u, v[u]);
            if (a.fuse) {
#pragma unroll
              for (int u = 0; u < 2; ++u)
                if (u < nc) tmem_ld16_nowait(tb + Ko + c0 + 16 * u, v[2 + u]);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (a.fuse) {
#pragma unroll
              for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  v[u][j] = __float_as_uint(__uint_as_float(v[u][j]) + __uint_as_float(v[2 + u][j]));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < nc) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int col = c0 + 16 * u + 4 * j;
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
          mbar_arrive(&acce[b]);
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
          if (a.fuse) {
            float w[16];
            tmem_ld16(tb + Ko + c, w);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += w[j];
          }
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
      if (OB > 0 && leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot),
                 "r"(a.tmem_cols));
  }
}

// kind::tf32 instruction descriptor for an M x N tile (D fp32, A / B TF32,
// both K-major)
__device__ __forceinline__ uint32_t idesc_mn(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[tmem] . B[smem]: the A operand read from tensor memory
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t db, uint32_t id,
                                            uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// The W-in-TMEM form, for Ko == 128 and Ki <= 128: the product is computed
// transposed, T^T = W^T . X^T, so W^T (M = Ko = 128 rows, K = Ki) is the A
// operand and lives in tensor memory (its hi and lo images: 2 Ki of the 512
// columns; the epilogue warps write them once per CTA with tcgen05.st), X^T
// is the B operand (N = 128 tile rows, K-major: the TMA chunk exactly as in
// gemm_tc_ring_kernel, and its lo), and D^T (lane = output column, column =
// tile row) is double-buffered in the other 256 columns.  Shared memory then
// holds only the X / lo rings and the staged output tiles: W's 128-KB image
// no longer crowds them out.  Epilogue: warp q owns output columns
// 32q .. 32q + 31 (TMEM lanes), i.e. exactly one 32-column block of the
// TMA store; a thread writes its column of 128 rows into the 128-B-swizzled
// tile (one conflict-free 128-B row per warp store).
constexpr int kWtD = 0, kWtW = 256;  // TMEM columns: D buffers at 0 / 128, W^T at 256
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_wt_kernel(const __grid_constant__ CUtensorMap xmap,
                      const __grid_constant__ CUtensorMap tmap, const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int Ki = a.Ki, SX = a.x_stages, SL = a.lo_stages, OB = a.out_bufs;
  constexpr int Ko = 128;
  uint8_t *xst0 = smem;                              // SX x 16 KB X chunks
  uint8_t *lost0 = xst0 + (size_t)SX * kChunkPart;   // SL x 16 KB lo chunks
  uint8_t *otile = lost0 + (size_t)SL * kChunkPart;  // OB x [4 blocks of 128 rows x 128 B]
  uint64_t *bar = reinterpret_cast<uint64_t *>(otile + (size_t)OB * kM * Ko * 4);
  uint64_t *xfull = bar, *xempty = bar + SX, *lofull = bar + 2 * SX, *loempty = lofull + SL;
  uint64_t *accf = loempty + SL, *acce = accf + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tiles = (a.n + kM - 1) / kM;
  const int chunks = Ki / kKc;

  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < SX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < SL; ++s) {
      mbar_init(&lofull[s], kLoaders);
      mbar_init(&loempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();  // barriers initialised, TMEM address published
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 9) {  // TMA producer: starts at once
    if (lane == 0) tma_x_loop(&xmap, tiles, chunks, SX, xst0, xfull, xempty);
    __syncwarp();
  } else if (warp < 4) {  // splitters
    split_loop(tid, tiles, chunks, SX, SL, xst0, lost0, xfull, lofull, loempty);
  } else if (warp == 4) {  // MMA issuer: waits for W^T in TMEM (named barrier 2)
    asm volatile("bar.sync 2, %0;" ::"r"(32 + kEpi) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (lane == 0) {
      const uint32_t id = idesc_mn(Ko, kM);
      const uint32_t whi = tmem + kWtW, wlo = whi + (uint32_t)Ki;
      int it = 0, tl = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
        const int b = tl & 1;
        if (tl >= 2) mbar_wait(&acce[b], ((tl >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + kWtD + (uint32_t)(b * kM);
        for (int c = 0; c < chunks; ++c, ++it) {
          const int sx = it % SX, sl = it % SL;
          mbar_wait(&lofull[sl], (it / SL) & 1);  // the splitters saw xfull: X landed too
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t xhi = smem_u32(xst0 + (size_t)sx * kChunkPart);
          const uint32_t xlo = smem_u32(lost0 + (size_t)sl * kChunkPart);
#pragma unroll
          for (int ks = 0; ks < kKc / 8; ++ks) {
            const uint64_t dbh = desc_sw128(xhi + ks * 32), dbl = desc_sw128(xlo + ks * 32);
            const uint32_t k0 = (uint32_t)(c * kKc + ks * 8);  // TMEM column of this K step
            mma_tf32_ts(acc, whi + k0, dbh, id, (c > 0 || ks > 0) ? 1u : 0u);
            mma_tf32_ts(acc, wlo + k0, dbh, id, 1u);
            mma_tf32_ts(acc, whi + k0, dbl, id, 1u);
          }
          mma_commit(&xempty[sx]);
          mma_commit(&loempty[sl]);
        }
        mma_commit(&accf[b]);
      }
    }
    __syncwarp();
  } else {  // warps 5-8: W^T -> TMEM once, then the epilogue
    const int q = warp & 3;  // TMEM lane quarter = output columns 32q .. 32q + 31
    const int col = 32 * q + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    for (int k0 = 0; k0 < Ki; k0 += 16) {  // W[k][col] for 16 k: coalesced over the warp
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float w = __ldg(a.W + (int64_t)(k0 + j) * a.ldw + col);
        const float h = tf32_rn(w);
        hi[j] = __float_as_uint(h);
        lo[j] = __float_as_uint(tf32_rn(w - h));
      }
      tmem_st16(lane_base + kWtW + k0, hi);
      tmem_st16(lane_base + kWtW + Ki + k0, lo);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 2, %0;" ::"r"(32 + kEpi) : "memory");
    const bool leader = tid == kLoaders + 32;
    int tl = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
      const int b = tl & 1;
      mbar_wait(&accf[b], (tl >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tb = lane_base + kWtD + (uint32_t)(b * kM);  // columns = tile rows
      if (OB > 0) {
        uint8_t *ot = otile + (size_t)(OB == 2 ? (tl & 1) : 0) * kM * Ko * 4 +
                      (size_t)q * kM * 128;  // this warp's 32-column block
        if (leader) {
          if (OB == 2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        const uint32_t obase = smem_u32(ot) + (uint32_t)(lane & 3) * 4;
        for (int r0 = 0; r0 < kM; r0 += 64) {
          uint32_t v[4][16];
#pragma unroll
          for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tb + r0 + 16 * u, v[u]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int r = r0 + 16 * u + j;  // tile row; chunk (lane / 4) of row r, swizzled
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(obase + r * 128 +
                                                          ((((uint32_t)lane >> 2) ^ (r & 7)) << 4)),
                           "r"(v[u][j])
                           : "memory");
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&acce[b]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(kEpi) : "memory");
        if (leader) {
          uint8_t *ob = otile + (size_t)(OB == 2 ? (tl & 1) : 0) * kM * Ko * 4;
          for (int blk = 0; blk < Ko / 32; ++blk)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmap)),
                "r"(blk * 32), "r"((int)(t * kM)), "r"(smem_u32(ob + (size_t)blk * kM * 128))
                : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        continue;
      }
      // no staged tile: each thread stores its column, 32 consecutive
      // columns per warp store (128 B per row)
      for (int r0 = 0; r0 < kM; r0 += 16) {
        float v[16];
        tmem_ld16(tb + r0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t row = t * kM + r0 + j;
          if (row < a.n) __stcs(a.T + row * a.ldt + col, v[j]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acce[b]);
    }
    if (OB > 0 && leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
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
    if (2ll * Ki * b * 4 + 4ll * kChunkPart + kSmemSlack <= kMaxSmem) return b;  // 2 X + 2 lo
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
  int b = gemm_tc_block(Ki, Ko);
  // Ko a multiple of 128 and Ki <= 128: 128-column blocks on the W-in-TMEM
  // form (64 x 256: 82.5 us for two blocks vs 112.6 us for one shared-memory
  // launch); PSPMM_GEMM_WT=0 / PSPMM_GEMM_WT128=0 (A/B
  // knobs) keep the widest shared-memory block
  const char *wte = std::getenv("PSPMM_GEMM_WT"), *w128 = std::getenv("PSPMM_GEMM_WT128");
  if (Ko % 128 == 0 && Ki <= 128 && !(wte && wte[0] == '0') && !(w128 && w128[0] == '0'))
    b = 128;
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
  const int64_t w = 2ll * Ki * Ko * 4;       // W's hi / lo image
  const int64_t otile = (int64_t)kM * Ko * 4;  // one staged output tile
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
  // ring depths: 2 lo buffers (PSPMM_GEMM_LO, 2..4), as many X stages as fit
  // (<= 8, PSPMM_GEMM_XS caps it), and the most staged output buffers
  // (PSPMM_GEMM_OB sets it; Ko % 32 == 0) that leave >= 4 X stages for two
  // buffers, >= 3 for one; without a staged epilogue >= 2.  The knobs are
  // A/B switches for tools/gemm_forms.py.
  int sl = 2;
  if (const char *e = std::getenv("PSPMM_GEMM_LO")) sl = std::max(2, std::min(4, std::atoi(e)));
  int xcap = 8;
  if (const char *e = std::getenv("PSPMM_GEMM_XS")) xcap = std::max(2, std::min(8, std::atoi(e)));
  // one staged output tile by default: the X stages it leaves pay more than
  // a second tile (W-in-TMEM 128 x 128: 53.5 us vs 61.4 us with two tiles
  // and 4 stages; shared-memory form 128 x 64: 53.2 vs 55.3 us)
  int obmax = Ko % 32 == 0 ? 1 : 0;
  if (const char *e = std::getenv("PSPMM_GEMM_OB"))
    obmax = Ko % 32 == 0 ? std::max(0, std::min(2, std::atoi(e))) : 0;
  CUtensorMap tmapT;
  std::memset(&tmapT, 0, sizeof(tmapT));
  if (obmax > 0) {
    cuuint64_t tdims[2] = {(cuuint64_t)Ko, (cuuint64_t)n};
    cuuint64_t tstr[1] = {(cuuint64_t)ldt * 4};
    cuuint32_t tbox[2] = {32, (cuuint32_t)kM};
    if (encode(&tmapT, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d_T, tdims, tstr, tbox, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      obmax = 0;
  }
  const int64_t tiles = (n + kM - 1) / kM;
  const int grid = (int)std::min<int64_t>(tiles, num_sms());
  // Ko == 128, Ki <= 128: W^T in tensor memory (gemm_tc_wt_kernel), no W
  // image in shared memory; PSPMM_GEMM_WT=0 (A/B knob) keeps the ring form
  const char *wte = std::getenv("PSPMM_GEMM_WT");
  if (Ko == 128 && Ki <= 128 && !(wte && wte[0] == '0')) {
    int ob = -1, sx = 0;
    for (int o = obmax; o >= 0; --o) {
      const int64_t left = kMaxSmem - kSmemSlack - (int64_t)o * otile - (int64_t)sl * kChunkPart;
      const int s = (int)std::min<int64_t>(xcap, left / kChunkPart);
      if (s >= (o == 2 ? 4 : o == 1 ? 3 : 2)) {
        ob = o;
        sx = s;
        break;
      }
    }
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
    args.x_stages = sx;
    args.lo_stages = sl;
    args.out_bufs = ob;
    args.tmem_cols = 512;
    args.fuse = 0;
    const size_t smem = (size_t)(kSmemSlack + (int64_t)ob * otile + (int64_t)(sx + sl) * kChunkPart);
    PSPMM_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_wt_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gemm_tc_wt_kernel<<<grid, kThreads, smem, stream>>>(map, tmapT, args);
    PSPMM_CUDA_TRY(cudaGetLastError());
    return PSPMM_OK;
  }
  int ob = -1, sx = 0;
  for (int o = obmax; o >= 0; --o) {
    const int64_t left = kMaxSmem - kSmemSlack - w - (int64_t)o * otile - (int64_t)sl * kChunkPart;
    const int s = (int)std::min<int64_t>(xcap, left / kChunkPart);
    if (s >= (o == 2 ? 4 : o == 1 ? 3 : 2)) {
      ob = o;
      sx = s;
      break;
    }
  }
  if (ob < 0) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "dense_gemm: shared memory too small for two X stages");
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
  args.x_stages = sx;
  args.lo_stages = sl;
  args.out_bufs = ob;
  // the fused-N MMA (X_hi read once per K step): PSPMM_GEMM_FUSE=0 (A/B knob) off
  const char *fe = std::getenv("PSPMM_GEMM_FUSE");
  args.fuse = (2 * Ko <= 256 && !(fe && fe[0] == '0')) ? 1 : 0;
  args.tmem_cols = tmem_cols_for(Ko * (args.fuse ? 2 : 1));
  const size_t smem = (size_t)(kSmemSlack + w + (int64_t)ob * otile + (int64_t)(sx + sl) * kChunkPart);
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_ring_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gemm_tc_ring_kernel<<<grid, kThreads, smem, stream>>>(map, tmapT, args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
