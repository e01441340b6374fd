// (a6, a7) The ParamSpMM computing engine (Alg. 2),
// re-designed for sm_100a.  One template instance per (V, S, F, G, vector
// width); W (warps per CTA) is a launch parameter.
//
// Mapping:
//  - a row group of G lanes (G | 32) owns one unit: a panel (S = 0) or a
//    chunk (S = 1).  A warp holds 32/G groups.  Lane l of the group owns the
//    columns col0 + (f G + l) VW, f < F, of C, VW = 4 (one float4 per f) on
//    the 128-bit path.  So a group covers 4 G F columns per pass; the paper's
//    coarsening factor F becomes F float4 accumulators per lane and
//    its blk.y segments are blockIdx.y passes.  The t-clamp of Alg. 2
//    l.3 is the per-f column mask `cok`.
//  - Alg. 2 l.5-7 (prefetch colIdx and the V values of a vector): the group
//    loads TILE = G M consecutive vectors' (colIdx, val) with coalesced
//    streaming loads, then broadcasts each one with a sub-group shuffle.
//  - Alg. 2 l.9-15 (t MACs reusing each B value V times): U vectors at a time
//    the lane issues U F independent 128-bit B-row loads (memory-level
//    parallelism), then V U F float4 FMAs into res[V][F] registers.
//  - Alg. 2 l.17-23 (S = 0): streaming 128-bit stores of V rows, rows >= n
//    skipped (c-6).  l.25-30 (S = 1, argument order fixed per c-9): a chunk
//    that is its panel's only chunk stores directly; the chunks of split
//    panels accumulate with red.global.add.v4.f32 into rows zeroed by
//    zero_split_kernel (c-12).
#include <type_traits>

#include "common.cuh"

namespace pspmm {
namespace {

struct SpmmArgs {
  const int32_t *__restrict__ rowptr;
  const int32_t *__restrict__ colidx;
  const float *__restrict__ val;
  const int32_t *__restrict__ trow;
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t n_rows, units, K;
};

__device__ __forceinline__ int ld_stream_i32(const int32_t *p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream_f32(const float *p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

template <typename T>
__device__ __forceinline__ T ld_b(const T *p) {
  return __ldg(p);
}

__device__ __forceinline__ void fma4(float4 &acc, float a, const float4 &b) {
  acc.x = fmaf(a, b.x, acc.x);
  acc.y = fmaf(a, b.y, acc.y);
  acc.z = fmaf(a, b.z, acc.z);
  acc.w = fmaf(a, b.w, acc.w);
}
__device__ __forceinline__ void fma4(float &acc, float a, const float &b) { acc = fmaf(a, b, acc); }

template <typename T>
__device__ __forceinline__ T zero_v();
template <>
__device__ __forceinline__ float4 zero_v<float4>() {
  return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <>
__device__ __forceinline__ float zero_v<float>() {
  return 0.f;
}

__device__ __forceinline__ void st_c(float4 *p, const float4 &v) { __stcs(p, v); }
__device__ __forceinline__ void st_c(float *p, const float &v) { __stcs(p, v); }
__device__ __forceinline__ void red_c(float4 *p, const float4 &v) { atomicAdd(p, v); }
__device__ __forceinline__ void red_c(float *p, const float &v) { atomicAdd(p, v); }

template <int V, int S, int F, int G, bool VEC>
__global__ void __launch_bounds__(512, 1) spmm_kernel(const SpmmArgs a) {
  using T = typename std::conditional<VEC, float4, float>::type;
  constexpr int VW = VEC ? 4 : 1;
  constexpr int GPW = 32 / G;
  constexpr int M = G >= 8 ? 1 : 8 / G;  // staged vectors per lane
  constexpr int TILE = G * M;            // vectors staged per group per round
  constexpr int U0 = (8 / F) > 0 ? (8 / F) : 1;
  constexpr int U = U0 < TILE ? U0 : TILE;  // vectors whose B rows are in flight together
  static_assert(TILE % U == 0, "tile/batch mismatch");

  const int lane = threadIdx.x & 31;
  const int g = lane / G;
  const int l = lane % G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t unit = warp * GPW + g;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
  const int col0 = blockIdx.y * (G * F * VW);

  int coff[F];
  bool cok[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    coff[f] = col0 + (f * G + l) * VW;
    cok[f] = coff[f] < a.K;
  }

  int head = 0, tail = 0;
  if (unit < a.units) {
    head = a.rowptr[unit];
    tail = a.rowptr[unit + 1];
  }

  T acc[V][F];
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int f = 0; f < F; ++f) acc[k][f] = zero_v<T>();

  for (int base = head; base < tail; base += TILE) {
    int mc[M];
    float mv[M][V];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int idx = base + m * G + l;
      if (idx < tail) {
        mc[m] = ld_stream_i32(a.colidx + idx);
#pragma unroll
        for (int k = 0; k < V; ++k) mv[m][k] = ld_stream_f32(a.val + (int64_t)idx * V + k);
      } else {
        mc[m] = 0;
#pragma unroll
        for (int k = 0; k < V; ++k) mv[m][k] = 0.f;
      }
    }
    const int cnt = min(TILE, tail - base);
#pragma unroll
    for (int j0 = 0; j0 < TILE; j0 += U) {
      if (j0 < cnt) {  // uniform inside the group
        T b[U][F];
        float vv[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u;
          const int c = __shfl_sync(gmask, mc[j / G], j % G, G);
#pragma unroll
          for (int k = 0; k < V; ++k) vv[u][k] = __shfl_sync(gmask, mv[j / G][k], j % G, G);
          const T *brow = reinterpret_cast<const T *>(a.B + (int64_t)c * a.ldb);
#pragma unroll
          for (int f = 0; f < F; ++f)
            b[u][f] = (j < cnt && cok[f]) ? ld_b(brow + coff[f] / VW) : zero_v<T>();
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < V; ++k)
#pragma unroll
            for (int f = 0; f < F; ++f) fma4(acc[k][f], vv[u][k], b[u][f]);
      }
    }
  }

  if (unit >= a.units) return;
  if (S == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t row = unit * V + k;
      if (row < a.n_rows) {
        T *crow = reinterpret_cast<T *>(a.C + row * a.ldc);
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) st_c(crow + coff[f] / VW, acc[k][f]);
      }
    }
  } else {
    const int panel = a.trow[unit];
    const bool sole = (unit == 0 || a.trow[unit - 1] != panel) &&
                      (unit + 1 == a.units || a.trow[unit + 1] != panel);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t row = (int64_t)panel * V + k;
      if (row < a.n_rows) {
        T *crow = reinterpret_cast<T *>(a.C + row * a.ldc);
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) {
            if (sole)
              st_c(crow + coff[f] / VW, acc[k][f]);
            else
              red_c(crow + coff[f] / VW, acc[k][f]);
          }
      }
    }
  }
}

// Zero the C rows of panels that own more than one chunk (S = 1, c-12).
__global__ void zero_split_kernel(const int32_t *__restrict__ split, int64_t num_split, int V,
                                  int64_t n_rows, int32_t K, float *__restrict__ C, int64_t ldc) {
  const int64_t per = (int64_t)V * K;
  const int64_t total = num_split * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / per, r = t % per;
    const int64_t row = (int64_t)split[s] * V + r / K;
    if (row < n_rows) C[row * ldc + r % K] = 0.f;
  }
}

// C = 0 (nnz_V == 0).
__global__ void zero_all_kernel(int64_t n_rows, int32_t K, float *__restrict__ C, int64_t ldc) {
  const int64_t total = n_rows * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    C[(t / K) * ldc + t % K] = 0.f;
}

using KernelFn = void (*)(const SpmmArgs);

template <int V, int S, int F, bool VEC>
KernelFn pick_g(int G) {
  switch (G) {
    case 1: return spmm_kernel<V, S, F, 1, VEC>;
    case 2: return spmm_kernel<V, S, F, 2, VEC>;
    case 4: return spmm_kernel<V, S, F, 4, VEC>;
    case 8: return spmm_kernel<V, S, F, 8, VEC>;
    case 16: return spmm_kernel<V, S, F, 16, VEC>;
    case 32: return spmm_kernel<V, S, F, 32, VEC>;
    default: return nullptr;
  }
}

template <int V, int S>
KernelFn pick(bool vec, int F, int G) {
  if (!vec) return F == 1 ? pick_g<V, S, 1, false>(G) : nullptr;
  switch (F) {
    case 1: return pick_g<V, S, 1, true>(G);
    case 2: return pick_g<V, S, 2, true>(G);
    case 3: return pick_g<V, S, 3, true>(G);
    case 4: return pick_g<V, S, 4, true>(G);
    case 5: return pick_g<V, S, 5, true>(G);
    case 6: return pick_g<V, S, 6, true>(G);
    case 7: return pick_g<V, S, 7, true>(G);
    case 8: return pick_g<V, S, 8, true>(G);
    default: return nullptr;
  }
}

KernelFn pick_kernel(int V, int S, bool vec, int F, int G) {
  if (V == 1) return S ? pick<1, 1>(vec, F, G) : pick<1, 0>(vec, F, G);
  return S ? pick<2, 1>(vec, F, G) : pick<2, 0>(vec, F, G);
}

bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

int ceil_pow2(int64_t x) {
  int p = 1;
  while (p < x && p < 32) p <<= 1;
  return p;
}

}  // namespace

pspmm_status run_spmm(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K, float *d_C,
                      int64_t ldc, const pspmm_config &cfg, cudaStream_t stream) {
  if (!A || !d_B || !d_C) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run: null handle or pointer");
  if (K < 1 || ldb < K || ldc < K)
    PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "spmm_run: need K >= 1, ldb >= K, ldc >= K");
  if (cfg.V != A->V || cfg.S != A->S || cfg.omega != A->omega)
    PSPMM_FAIL(PSPMM_ERR_CONFIG_MISMATCH, "spmm_run: cfg.V/S/omega differ from the PCSR handle");
  if (cfg.mode != 0) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: only mode 0 is implemented");
  if (!(cfg.W == 1 || cfg.W == 2 || cfg.W == 4 || cfg.W == 8 || cfg.W == 16))
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: W must be 1, 2, 4, 8 or 16");
  if (cfg.F < 1 || cfg.F > 8)
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: F must be in 1..8 (float4 units)");
  if (cfg.G != 0 && !(pow2(cfg.G) && cfg.G <= 32))
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: G must be 0 or a power of two <= 32");

  const int64_t n_rows = A->n_rows;
  if (A->nnz_v == 0) {
    int64_t total = n_rows * K;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    zero_all_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(n_rows, K, d_C, ldc);
    PSPMM_CUDA_TRY(cudaGetLastError());
    return PSPMM_OK;
  }

  const bool vec = (K % 4 == 0) && (ldb % 4 == 0) && (ldc % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(d_B) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(d_C) & 15) == 0);
  int F = cfg.F, G = cfg.G, cols_per_pass;
  if (vec) {
    if (G == 0) G = ceil_pow2((K / 4 + F - 1) / F);
    cols_per_pass = 4 * G * F;
  } else {
    // masked scalar variant: one column per lane, G = min(32, pow2 >= K)
    F = 1;
    G = ceil_pow2(K);
    cols_per_pass = G;
  }
  KernelFn fn = pick_kernel(A->V, A->S, vec, F, G);
  if (!fn) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: no kernel instance for this config");

  if (A->S == 1 && A->num_split > 0) {
    int64_t total = A->num_split * A->V * (int64_t)K;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    zero_split_kernel<<<blocks, 256, 0, stream>>>(A->d_split, A->num_split, A->V, n_rows, K, d_C,
                                                   ldc);
    PSPMM_CUDA_TRY(cudaGetLastError());
  }

  SpmmArgs args;
  args.rowptr = A->d_rowptr;
  args.colidx = A->d_colidx;
  args.val = A->d_val;
  args.trow = A->d_trow;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.n_rows = (int32_t)n_rows;
  args.units = (int32_t)A->num_chunks;
  args.K = K;
  const int threads = cfg.W * 32;
  const int64_t groups_per_block = threads / G;
  const int64_t bx = (A->num_chunks + groups_per_block - 1) / groups_per_block;
  const int64_t by = (K + cols_per_pass - 1) / cols_per_pass;
  if (bx > 0x7fffffff || by > 65535)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: grid too large for this config");
  fn<<<dim3((unsigned)bx, (unsigned)by), threads, 0, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
