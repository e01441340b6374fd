// (a6, a7) Engine mode 4: asynchronous-copy pipeline for low-degree graphs
// (roadNet-like, d ~ 3), V = 1 and S = 0 only.  Same computation as Alg. 2
// — C[r] = sum over the row's vectors of val * B[colIdx] — with a
// schedule built for latency: in mode 3 the in-flight B rows live in
// registers, so the bytes a warp can have in flight are capped by its
// register budget and every row still waits for its own gathers.  Here:
//  - a row group (G lanes, F float4 columns per lane) owns one contiguous
//    range of rows, so its vectors form ONE contiguous stream
//    [rowPtr[R0], rowPtr[R1]) processed in batches of U vectors;
//  - (colIdx, val) of batch b + 2D and the B rows of batch b + D are copied
//    into shared-memory rings with cp.async (LDGSTS, L1-allocating), while
//    batch b is consumed: the gathers of D batches are in flight without
//    occupying registers, and no row boundary stalls the stream;
//  - rowPtr is staged per 32-row sub-tile (double-buffered, prefetched one
//    sub-tile ahead) to find the row boundaries inside the stream; a row's
//    accumulators are stored when the stream crosses its end (empty rows
//    store zeros, rows >= n never exist here since ranges are clamped).
// Ring slots are lane-private for B ([slot][u][f][lane] float4, conflict-free
// LDS.128) and group-shared for (colIdx, val, rowPtr) — those are read by
// every lane of the group after the step's cp.async.wait_group + __syncwarp.
#include <algorithm>

#include "common.cuh"

namespace pspmm {
namespace {

#ifndef PSPMM_ASYNC_U
#define PSPMM_ASYNC_U 4
#endif
#ifndef PSPMM_ASYNC_D
#define PSPMM_ASYNC_D 3
#endif
constexpr int kU = PSPMM_ASYNC_U;  // vectors per batch
constexpr int kD = PSPMM_ASYNC_D;  // batches of B rows in flight
constexpr int kRC = 2 * kD + 1;  // (colIdx, val) ring slots: batches b .. b + 2D
constexpr int kRB = kD + 1;      // B ring slots: batches b .. b + D
constexpr int kSub = 32;         // rows per staged rowPtr sub-tile

struct AsyncArgs {
  const int32_t *__restrict__ rowptr;
  const int32_t *__restrict__ colidx;
  const float *__restrict__ val;
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t row_begin, row_end, K, rows_per_group;
  int32_t accumulate;  // 1: C += A.B
  int32_t warp_bytes;  // shared memory per warp
  Fanout fan;          // peer copies of C (f2)
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int F, int G>
constexpr int warp_bytes() {  // rounded to 16 B: every warp's B ring stays 16-B aligned
  return (kRB * kU * F * 32 * 16 + (32 / G) * kRC * kU * 8 + (32 / G) * 2 * (kSub + 1) * 4 + 15) /
         16 * 16;
}

template <int F, int G>
__global__ void __launch_bounds__(256) spmm_async_kernel(const AsyncArgs a) {
  constexpr int GPW = 32 / G;
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, l = lane % G;
  unsigned char *wb = smem + (size_t)wib * a.warp_bytes;
  float4 *bS = reinterpret_cast<float4 *>(wb);  // [kRB][kU][F][32]
  int *colS = reinterpret_cast<int *>(wb + kRB * kU * F * 512) + g * kRC * kU;
  float *valS = reinterpret_cast<float *>(wb + kRB * kU * F * 512 + GPW * kRC * kU * 4) +
                g * kRC * kU;
  int *rpS = reinterpret_cast<int *>(wb + kRB * kU * F * 512 + GPW * kRC * kU * 8) +
             g * 2 * (kSub + 1);
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));

  const int64_t gid = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * GPW + g;
  const int64_t R0 = a.row_begin + gid * a.rows_per_group;
  if (R0 >= a.row_end) return;  // uniform within the group
  const int64_t R1 = min(R0 + (int64_t)a.rows_per_group, (int64_t)a.row_end);
  const int col0 = blockIdx.y * (G * F * 4);
  bool cok[F];
#pragma unroll
  for (int f = 0; f < F; ++f) cok[f] = col0 + (f * G + l) * 4 < a.K;
  const float *bbase = a.B + col0 + l * 4;

  const int v0 = __ldg(a.rowptr + R0), v1 = __ldg(a.rowptr + R1);
  const int nb = (v1 - v0 + kU - 1) / kU;

  auto fetch_rp = [&](int k) {  // rowPtr of sub-tile k (kSub + 1 entries)
    const int64_t s0 = R0 + (int64_t)k * kSub;
    if (s0 >= R1) return;
    const int cnt = (int)min((int64_t)kSub, R1 - s0);
    int *dst = rpS + (k & 1) * (kSub + 1);
    for (int i = l; i <= cnt; i += G) cp_async4(dst + i, a.rowptr + s0 + i);
  };
  auto issue_col = [&](int b) {
    if (b >= nb) return;
    const int slot = b % kRC;
    for (int u = l; u < kU; u += G) {
      const int v = v0 + b * kU + u;
      if (v < v1) {
        cp_async4(colS + slot * kU + u, a.colidx + v);
        cp_async4(valS + slot * kU + u, a.val + v);
      }
    }
  };
  auto issue_B = [&](int b) {
    if (b >= nb) return;
    const int cs = b % kRC, bs = b % kRB;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (v0 + b * kU + u < v1) {
        const int c = colS[cs * kU + u];
        const float *src = bbase + (int64_t)c * a.ldb;
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) cp_async16(bS + ((bs * kU + u) * F + f) * 32 + lane, src + f * G * 4);
      }
    }
  };

  float4 acc[F];
#pragma unroll
  for (int f = 0; f < F; ++f) acc[f] = make_float4(0.f, 0.f, 0.f, 0.f);
  auto store_row = [&](int64_t r) {
    float *crow = a.C + r * a.ldc + col0 + l * 4;
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (cok[f]) {
        float4 v = acc[f];
        float4 *p = reinterpret_cast<float4 *>(crow + f * G * 4);
        if (a.accumulate) {
          const float4 o = *p;
          v.x += o.x;
          v.y += o.y;
          v.z += o.z;
          v.w += o.w;
        }
        __stcs(p, v);
#pragma unroll 1
        for (int d = 0; d < a.fan.n; ++d)
          __stcs(reinterpret_cast<float4 *>(a.fan.peer[d] + r * a.ldc + col0 + l * 4 + f * G * 4),
                 v);
        acc[f] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
  };

  // prologue: (colIdx, val) of batches 0 .. D-1, rowPtr of sub-tiles 0 and 1
#pragma unroll
  for (int s = 0; s < kD; ++s) {
    if (s == 0) {
      fetch_rp(0);
      fetch_rp(1);
    }
    issue_col(s);
    cp_commit();
  }
  int64_t row = R0;   // the row the stream is in
  int sub = 0;        // its sub-tile
  int rp_step = -kD;  // commit step of the newest rowPtr prefetch (sub-tile sub + 1)
  int nextb = 0;      // first vector of row + 1
  for (int b = -kD; b < nb; ++b) {
    cp_wait<kD - 1>();
    __syncwarp(gmask);
    if (b == -kD) nextb = rpS[1];
    issue_col(b + 2 * kD);
    issue_B(b + kD);
    cp_commit();
    if (b < 0) continue;
    const int cs = b % kRC, bs = b % kRB;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int v = v0 + b * kU + u;
      if (v >= v1) break;
      while (v >= nextb) {  // the stream left `row`: store it, step to the next row
        store_row(row);
        ++row;
        const int k = (int)((row - R0) / kSub), i = (int)((row - R0) % kSub);
        if (k != sub) {
          // entering sub-tile k: its rowPtr went out with the commit of step
          // rp_step, complete from the wait of step rp_step + D on
          if (b < rp_step + kD) cp_wait<0>();
          __syncwarp(gmask);  // complete for all lanes; nobody reads sub-tile k - 1 any more
          sub = k;
          fetch_rp(k + 1);  // into the buffer sub-tile k - 1 used
          rp_step = b + 1;
        }
        nextb = rpS[(k & 1) * (kSub + 1) + i + 1];
      }
      const float w = valS[cs * kU + u];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const float4 x = bS[((bs * kU + u) * F + f) * 32 + lane];
        acc[f].x = fmaf(w, x.x, acc[f].x);
        acc[f].y = fmaf(w, x.y, acc[f].y);
        acc[f].z = fmaf(w, x.z, acc[f].z);
        acc[f].w = fmaf(w, x.w, acc[f].w);
      }
    }
  }
  cp_wait<0>();
  // the stream is exhausted: the current row and every row after it (all
  // empty) are stored
  for (; row < R1; ++row) store_row(row);
  if (a.fan.n) __threadfence_system();
}

using AsyncFn = void (*)(const AsyncArgs);

template <int F>
AsyncFn pick_g(int G, int *bytes) {
  switch (G) {
    case 2: *bytes = warp_bytes<F, 2>(); return spmm_async_kernel<F, 2>;
    case 4: *bytes = warp_bytes<F, 4>(); return spmm_async_kernel<F, 4>;
    case 8: *bytes = warp_bytes<F, 8>(); return spmm_async_kernel<F, 8>;
    case 16: *bytes = warp_bytes<F, 16>(); return spmm_async_kernel<F, 16>;
    case 32: *bytes = warp_bytes<F, 32>(); return spmm_async_kernel<F, 32>;
    default: return nullptr;
  }
}

AsyncFn pick(int F, int G, int *bytes) {
  switch (F) {
    case 1: return pick_g<1>(G, bytes);
    case 2: return pick_g<2>(G, bytes);
    case 4: return pick_g<4>(G, bytes);
    default: return nullptr;
  }
}

int ceil_pow2(int x) {
  int p = 1;
  while (p < x && p < 32) p <<= 1;
  return p;
}

}  // namespace

bool async_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                     const float *d_C, const pspmm_config &cfg) {
  return A->V == 1 && A->S == 0 && K % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0 &&
         (cfg.F == 1 || cfg.F == 2 || cfg.F == 4);
}

pspmm_status run_spmm_async(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                            float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                            int64_t u0, int64_t u1, int32_t accumulate, const Fanout &fan) {
  if (u1 <= u0) return PSPMM_OK;
  const int F = cfg.F;
  int G = cfg.G ? cfg.G : ceil_pow2((K / 4 + F - 1) / F);
  if (G < 2) G = 2;
  int wbytes = 0;
  AsyncFn fn = pick(F, G, &wbytes);
  if (!fn) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 4: F must be 1, 2 or 4 and G >= 2");
  const int W = std::min(cfg.W, 8);
  const int threads = W * 32;
  const int smem = W * wbytes;
  if (smem > 227 * 1024) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 4: W too large for smem");
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PSPMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm < 1) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 4: no resident block");
  const int64_t rows = u1 - u0;
  const int64_t per_block = (int64_t)W * (32 / G);
  int64_t bx = (int64_t)num_sms() * per_sm;
  // one contiguous row range per group, every resident group busy
  int64_t rpg = (rows + bx * per_block - 1) / (bx * per_block);
  if (rpg < 1) rpg = 1;
  bx = (rows + rpg * per_block - 1) / (rpg * per_block);
  if (rpg > 0x7fffffff) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run mode 4: too many rows");
  AsyncArgs args;
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
  args.rows_per_group = (int32_t)rpg;
  args.accumulate = accumulate;
  args.warp_bytes = wbytes;
  args.fan = fan;
  const int64_t by = (K + 4 * G * F - 1) / (4 * G * F);
  fn<<<dim3((unsigned)bx, (unsigned)by), threads, smem, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
