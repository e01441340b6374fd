// (a6, a7) Engine mode 3: short-row pipeline for low-degree graphs
// (roadNet-like, d ~ 3), V = 1 and S = 0 only.  Same computation as Alg. 2
// (P:215-267); what changes is the schedule.  The mode-0 engine gives each
// row group one unit and retires, so every row pays the dependent
// rowPtr -> colIdx -> B-row -> store latency chain with nothing else in
// flight.  Here a row group (G lanes, F float4 accumulators per lane) walks
// rows r, r + stride, ... with a two-deep software pipeline: the rowPtr pair
// two rows ahead and the (colIdx, val) of the next row (one vector per lane,
// rows up to G vectors; longer rows continue in a slow loop) are in flight
// while the current row's B rows are gathered.  The register footprint stays
// small (no staged tiles), so more warps are resident.
#include <algorithm>

#include "common.cuh"

namespace pspmm {
namespace {

struct ShortArgs {
  const int32_t *__restrict__ rowptr;
  const int32_t *__restrict__ colidx;
  const float *__restrict__ val;
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t row_begin, row_end, K;
  int32_t accumulate;  // 1: C += A.B
  Fanout fan;          // peer copies of C (f2)
};

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

#ifndef PSPMM_SHORT_MINB
// resident 256-thread blocks per SM: 3 = 85 registers, no spills (A/B on
// roadNet: 0.148 ms vs 0.156 at 4 blocks / 64 registers with spills)
#define PSPMM_SHORT_MINB 3
#endif
#ifndef PSPMM_SHORT_WAVES
#define PSPMM_SHORT_WAVES 1  // grid = one wave of resident blocks (A/B: 1 beats 2 and 4)
#endif

// FMA of one gathered float4 into an accumulator
__device__ __forceinline__ void fma4(float4 &acc, float v, const float4 &b) {
  acc.x = fmaf(v, b.x, acc.x);
  acc.y = fmaf(v, b.y, acc.y);
  acc.z = fmaf(v, b.z, acc.z);
  acc.w = fmaf(v, b.w, acc.w);
}

// Lean form: 32-bit row / offset arithmetic, a per-lane B base pointer, and
// a fast path for the common row (at most U = min(G, 8 / F) vectors: one
// batch of predicated 128-bit gathers, predicated FMAs, no zero-filled
// registers); longer rows continue in a generic window loop.
template <int F, int G>
__global__ void __launch_bounds__(256, PSPMM_SHORT_MINB) spmm_short_kernel(const ShortArgs a) {
  constexpr int U = (8 / F) < G ? (8 / F) : G;  // vectors gathered together
  const int lane = threadIdx.x & 31;
  const int g = lane / G, l = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
  const int groups = (int)((gridDim.x * blockDim.x) >> 5) * (32 / G);
  int r = a.row_begin + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G) + g;
  const int col0 = blockIdx.y * G * F * 4;
  bool cok[F];
#pragma unroll
  for (int f = 0; f < F; ++f) cok[f] = col0 + (f * G + l) * 4 < a.K;
  const float4 *bl = reinterpret_cast<const float4 *>(a.B + col0 + l * 4);
  const uint32_t ldq = (uint32_t)(a.ldb / 4);  // B row stride in float4
  const int32_t *__restrict__ rowptr = a.rowptr;
  const int32_t *__restrict__ colidx = a.colidx;
  const float *__restrict__ val = a.val;
  const int row_end = a.row_end;

  // pipeline registers: rowPtr of r and r + groups, the vectors of r
  int h0 = 0, t0 = 0, h1 = 0, t1 = 0;
  if (r < row_end) {
    h0 = rowptr[r];
    t0 = rowptr[r + 1];
  }
  if (r + groups < row_end) {
    h1 = rowptr[r + groups];
    t1 = rowptr[r + groups + 1];
  }
  int c0 = 0;
  float v0 = 0.f;
  if (h0 + l < t0) {
    c0 = lda(colidx + h0 + l);
    v0 = lda(val + h0 + l);
  }
  for (; r < row_end; r += groups) {
    // prefetch: rowPtr two rows ahead, vectors of the next row
    const int r2 = r + 2 * groups;
    int h2 = 0, t2 = 0;
    if (r2 < row_end) {
      h2 = rowptr[r2];
      t2 = rowptr[r2 + 1];
    }
    int c1 = 0;
    float v1 = 0.f;
    if (h1 + l < t1) {
      c1 = lda(colidx + h1 + l);
      v1 = lda(val + h1 + l);
    }
    const int cnt = t0 - h0;
    float4 acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = make_float4(0.f, 0.f, 0.f, 0.f);
    {  // fast path: the first U vectors
      float4 b[U][F];
      float vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(gmask, c0, u, G);
        vv[u] = __shfl_sync(gmask, v0, u, G);
        const float4 *row = bl + (uint32_t)c * ldq;
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (u < cnt && cok[f]) b[u][f] = __ldg(row + f * G);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < cnt)
#pragma unroll
          for (int f = 0; f < F; ++f)
            if (cok[f]) fma4(acc[f], vv[u], b[u][f]);
    }
    // the rest of a long row: staged vectors U .. G-1, then reloads from
    // colIdx / val (a second staged window measured slower: more registers)
    for (int j = U; j < cnt; ++j) {
      int c;
      float v;
      if (j < G) {
        c = __shfl_sync(gmask, c0, j, G);
        v = __shfl_sync(gmask, v0, j, G);
      } else {
        c = lda(colidx + h0 + j);  // uniform address within the group: broadcast
        v = lda(val + h0 + j);
      }
      const float4 *row = bl + (uint32_t)c * ldq;
#pragma unroll
      for (int f = 0; f < F; ++f)
        if (cok[f]) fma4(acc[f], v, __ldg(row + f * G));
    }
    float4 *crow = reinterpret_cast<float4 *>(a.C + (int64_t)r * a.ldc + col0 + l * 4);
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (cok[f]) {
        float4 v = acc[f];
        if (a.accumulate) {
          const float4 o = crow[f * G];
          v.x += o.x;
          v.y += o.y;
          v.z += o.z;
          v.w += o.w;
        }
        fan_store4(a.C, a.fan, (int64_t)r * a.ldc + col0 + l * 4 + f * G * 4, v);
      }
    h0 = h1;
    t0 = t1;
    h1 = h2;
    t1 = t2;
    c0 = c1;
    v0 = v1;
  }
  if (a.fan.n) __threadfence_system();
}


// Ring form (PSPMM_SHORT_RING = 1): the same row-strided schedule, but the B
// rows of the next row are copied into a lane-private shared-memory slot with
// cp.async (LDGSTS) while the current row is consumed from the other slot.
// In-flight gathers then cost no registers, so two rows per group stay in
// flight at any time (the register form holds one and stalls on it).
// Slot layout: [warp][slot][item = u F + f][lane] float4 (conflict-free).
#ifndef PSPMM_SHORT_RING
#define PSPMM_SHORT_RING 0  // A/B: the ring form measured slower (profiles/r01/mode3_ab/README.md, ab4)
#endif

#ifndef PSPMM_SHORT_RING_CG
#define PSPMM_SHORT_RING_CG 0  // 1: cp.async.cg (L2 only) instead of .ca (L1-allocating)
#endif
__device__ __forceinline__ void cp_async16(float4 *dst, const float4 *src) {
#if PSPMM_SHORT_RING_CG
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
  return;
#endif
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

template <int F, int G>
__global__ void __launch_bounds__(256) spmm_ring_kernel(const ShortArgs a) {
  constexpr int U = (8 / F) < G ? (8 / F) : G;  // vectors staged per row
  constexpr int ITEMS = U * F;                  // float4 per lane per slot
  extern __shared__ float4 ring_smem[];
  const int lane = threadIdx.x & 31;
  const int g = lane / G, l = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
  const int groups = (int)((gridDim.x * blockDim.x) >> 5) * (32 / G);
  float4 *slot0 = ring_smem + (size_t)(threadIdx.x >> 5) * (2 * ITEMS * 32) + lane;
  const int col0 = blockIdx.y * G * F * 4;
  bool cok[F];
#pragma unroll
  for (int f = 0; f < F; ++f) cok[f] = col0 + (f * G + l) * 4 < a.K;
  const float4 *bl = reinterpret_cast<const float4 *>(a.B + col0 + l * 4);
  const uint32_t ldq = (uint32_t)(a.ldb / 4);
  const int32_t *__restrict__ rowptr = a.rowptr;
  const int32_t *__restrict__ colidx = a.colidx;
  const float *__restrict__ val = a.val;
  const int row_end = a.row_end;
  int r = a.row_begin + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G) + g;

  // issue the staged gathers of one row (its first U vectors) into slot s
  auto stage = [&](int s, int h, int t, int c) {
    const int cnt = t - h;
    float4 *dst = slot0 + s * (ITEMS * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cu = __shfl_sync(gmask, c, u, G);
      if (u < cnt) {
        const float4 *row = bl + (uint32_t)cu * ldq;
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) cp_async16(dst + (u * F + f) * 32, row + f * G);
      }
    }
    cp_async_commit();
  };

  // pipeline registers: rowPtr of rows k, k+1, k+2; vectors of rows k, k+1
  int h0 = 0, t0 = 0, h1 = 0, t1 = 0, h2 = 0, t2 = 0;
  if (r < row_end) { h0 = rowptr[r]; t0 = rowptr[r + 1]; }
  if (r + groups < row_end) { h1 = rowptr[r + groups]; t1 = rowptr[r + groups + 1]; }
  if (r + 2 * groups < row_end) { h2 = rowptr[r + 2 * groups]; t2 = rowptr[r + 2 * groups + 1]; }
  int c0 = 0, c1 = 0;
  float v0 = 0.f, v1 = 0.f;
  if (h0 + l < t0) { c0 = lda(colidx + h0 + l); v0 = lda(val + h0 + l); }
  if (h1 + l < t1) { c1 = lda(colidx + h1 + l); v1 = lda(val + h1 + l); }
  stage(0, h0, t0, c0);
  int s = 0;
  for (; r < row_end; r += groups) {
    // row k + 1 into the other slot, then prefetch row k + 2's vectors and
    // row k + 3's rowPtr
    stage(s ^ 1, h1, t1, c1);
    int c2 = 0;
    float v2 = 0.f;
    if (h2 + l < t2) { c2 = lda(colidx + h2 + l); v2 = lda(val + h2 + l); }
    const int r3 = r + 3 * groups;
    int h3 = 0, t3 = 0;
    if (r3 < row_end) { h3 = rowptr[r3]; t3 = rowptr[r3 + 1]; }
    // consume row k (its group of copies is the older of the two in flight)
    cp_async_wait1();
    const int cnt = t0 - h0;
    const float4 *src = slot0 + s * (ITEMS * 32);
    float4 acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float vu = __shfl_sync(gmask, v0, u, G);
      if (u < cnt)
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) fma4(acc[f], vu, src[(u * F + f) * 32]);
    }
    for (int j = U; j < cnt; ++j) {  // the rest of a long row: direct loads
      int c;
      float v;
      if (j < G) {
        c = __shfl_sync(gmask, c0, j, G);
        v = __shfl_sync(gmask, v0, j, G);
      } else {
        c = lda(colidx + h0 + j);
        v = lda(val + h0 + j);
      }
      const float4 *row = bl + (uint32_t)c * ldq;
#pragma unroll
      for (int f = 0; f < F; ++f)
        if (cok[f]) fma4(acc[f], v, __ldg(row + f * G));
    }
    float4 *crow = reinterpret_cast<float4 *>(a.C + (int64_t)r * a.ldc + col0 + l * 4);
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (cok[f]) {
        float4 v = acc[f];
        if (a.accumulate) {
          const float4 o = crow[f * G];
          v.x += o.x;
          v.y += o.y;
          v.z += o.z;
          v.w += o.w;
        }
        fan_store4(a.C, a.fan, (int64_t)r * a.ldc + col0 + l * 4 + f * G * 4, v);
      }
    h0 = h1; t0 = t1; c0 = c1; v0 = v1;
    h1 = h2; t1 = t2; c1 = c2; v1 = v2;
    h2 = h3; t2 = t3;
    s ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (a.fan.n) __threadfence_system();
}

using ShortFn = void (*)(const ShortArgs);

template <int F>
ShortFn pick_g(int G) {
#if PSPMM_SHORT_RING
  switch (G) {
    case 2: return spmm_ring_kernel<F, 2>;
    case 4: return spmm_ring_kernel<F, 4>;
    case 8: return spmm_ring_kernel<F, 8>;
    case 16: return spmm_ring_kernel<F, 16>;
    case 32: return spmm_ring_kernel<F, 32>;
    default: return nullptr;
  }
#else
  switch (G) {
    case 2: return spmm_short_kernel<F, 2>;
    case 4: return spmm_short_kernel<F, 4>;
    case 8: return spmm_short_kernel<F, 8>;
    case 16: return spmm_short_kernel<F, 16>;
    case 32: return spmm_short_kernel<F, 32>;
    default: return nullptr;
  }
#endif
}

ShortFn pick(int F, int G) {
  switch (F) {
    case 1: return pick_g<1>(G);
    case 2: return pick_g<2>(G);
    case 4: return pick_g<4>(G);
    default: return nullptr;
  }
}

int ceil_pow2(int x) {
  int p = 1;
  while (p < x && p < 32) p <<= 1;
  return p;
}

}  // namespace

bool short_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                     const float *d_C, const pspmm_config &cfg) {
  // B offsets are 32-bit float4 counts: B must span < 2^32 float4 (64 GB)
  return A->V == 1 && A->S == 0 && K % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 &&
         (uint64_t)A->n_cols * (uint64_t)(ldb / 4) < (1ull << 32) &&
         (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0 &&
         (cfg.F == 1 || cfg.F == 2 || cfg.F == 4);
}

pspmm_status run_spmm_short(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                            int64_t u0, int64_t u1, int32_t accumulate, const Fanout &fan) {
  if (u1 <= u0) return PSPMM_OK;
  const int F = cfg.F;
  int G = cfg.G ? cfg.G : ceil_pow2((K / 4 + F - 1) / F);
  if (G < 2) G = 2;
  ShortFn fn = pick(F, G);
  if (!fn) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 3: F must be 1, 2 or 4 and G >= 2");
  ShortArgs args;
  args.rowptr = A->d_rowptr;
  args.colidx = A->d_colidx;
  args.val = A->d_val;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.row_begin = (int32_t)u0;
  args.row_end = (int32_t)u1;
  args.K = K;
  args.accumulate = accumulate;
  args.fan = fan;
  const int threads = std::min(cfg.W, 8) * 32;
  const int64_t per_block = threads / 32 * (32 / G);
  int64_t bx = (u1 - u0 + per_block - 1) / per_block;
#if PSPMM_SHORT_RING
  // two slots of (U F) float4 per lane; one wave of resident blocks
  const int U = std::min(8 / F, G);
  const int smem = threads * 2 * U * F * 16;
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PSPMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm < 1) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 3: no resident block");
  bx = std::min<int64_t>(bx, (int64_t)num_sms() * per_sm * PSPMM_SHORT_WAVES);
#else
  const int smem = 0;
  // a few waves of resident blocks (launch bounds: 256 x PSPMM_SHORT_MINB threads / SM)
  const int64_t resident = std::max<int64_t>(1, 256 * PSPMM_SHORT_MINB / threads);
  bx = std::min<int64_t>(bx, (int64_t)num_sms() * resident * PSPMM_SHORT_WAVES);
#endif
  const int64_t by = (K + 4 * G * F - 1) / (4 * G * F);
  fn<<<dim3((unsigned)bx, (unsigned)by), threads, smem, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
