// (a6, a7) The ParamSpMM computing engine — kernel template (instantiated in
// spmm_inst_v*s*.cu, one translation unit per (V, S) so they compile in
// parallel; dispatch in spmm.cu) (Alg. 2),
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
#pragma once
#include <type_traits>

#include "common.cuh"

namespace pspmm {
namespace detail {


struct SpmmArgs {
  const int32_t *__restrict__ rowptr;
  const int32_t *__restrict__ colidx;
  const float *__restrict__ val;
  const int32_t *__restrict__ trow;
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t n_rows, unit_begin, units, units_total, K;  // units = end of this launch's range
  int32_t accumulate;                                  // 1: C += A.B
  const int32_t *__restrict__ order;                   // optional unit order (nullptr = identity)
  Fanout fan;                                          // peer copies of C (f2); fan.n = 0: none
};

// L2 policies: A (colIdx / val) is streamed once -> evict_first and no L1
// allocation; B rows are re-gathered nnz/n times each -> evict_last.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ld_a(const int32_t *p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_a(const float *p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
// B gathers: L1-allocating, or (NA) L1::no_allocate — for B far larger than
// L2, whose gathers cannot hit in L1 (the allocations only thrash it); the
// NA instances are separate kernels (spmm_inst_*_na.cu), chosen per launch
template <bool NA>
__device__ __forceinline__ void ld_b(float4 &v, const char *p, uint64_t pol) {
  if constexpr (NA)
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  else
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
}
template <bool NA>
__device__ __forceinline__ void ld_b(float &v, const char *p, uint64_t pol) {
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
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

// C store; with `accumulate` (pspmm_spmm_accumulate: C += A.B) the old value
// is added first — one writer per element within a launch, so no atomics
__device__ __forceinline__ void st_c(float4 *p, float4 v, int accumulate = 0) {
  if (accumulate) {
    const float4 o = *p;
    v.x += o.x;
    v.y += o.y;
    v.z += o.z;
    v.w += o.w;
  }
  __stcs(p, v);
}
__device__ __forceinline__ void st_c(float *p, float v, int accumulate = 0) {
  if (accumulate) v += *p;
  __stcs(p, v);
}
__device__ __forceinline__ float4 add_c(const float4 &o, const float4 &v) {
  return make_float4(o.x + v.x, o.y + v.y, o.z + v.z, o.w + v.w);
}
__device__ __forceinline__ float add_c(const float &o, const float &v) { return o + v; }
__device__ __forceinline__ void red_c(float4 *p, const float4 &v) { atomicAdd(p, v); }
__device__ __forceinline__ void red_c(float *p, const float &v) { atomicAdd(p, v); }

// Write one C element group at float offset `off`: to C (store or atomic) and,
// with a fan-out, to the same offset of every peer buffer (f2).  The peer
// loop is a uniform branch on a kernel parameter: free when fan.n == 0.
template <typename T>
__device__ __forceinline__ void put_c(const SpmmArgs &a, int64_t off, const T &v, bool red) {
  T *p = reinterpret_cast<T *>(a.C + off);
  if (a.fan.mc) {  // NVLS: one multimem op reaches every bound copy (local included)
    if (red) {
      mc_red(a.fan.peer[0] + off, v);
    } else {
      T w = v;
      if (a.accumulate) w = add_c(*p, w);
      mc_st(a.fan.peer[0] + off, w);
    }
    return;
  }
  if (red)
    red_c(p, v);
  else
    st_c(p, v, a.accumulate);
#pragma unroll 1
  for (int d = 0; d < a.fan.n; ++d) {
    T *q = reinterpret_cast<T *>(a.fan.peer[d] + off);
    if (red)
      red_c(q, v);
    else
      st_c(q, v, 0);
  }
}

// Stage one tile of the unit's vectors: lane l of the group holds vectors
// base + m G + l, m < M (colIdx and the V values; Alg. 2 l.6-7).
template <int V, int M, int G>
__device__ __forceinline__ void load_tile(const SpmmArgs &a, int base, int tail, int l,
                                          uint64_t pol, int (&c)[M], float (&v)[M][V]) {
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int idx = base + m * G + l;
    if (idx < tail) {
      c[m] = ld_a(a.colidx + idx, pol);
#pragma unroll
      for (int k = 0; k < V; ++k) v[m][k] = ld_a(a.val + (int64_t)idx * V + k, pol);
    } else {
      c[m] = 0;
#pragma unroll
      for (int k = 0; k < V; ++k) v[m][k] = 0.f;
    }
  }
}

// Alg. 2 l.8-16 for one staged tile: batches of U vectors, U F independent
// B-row loads in flight per lane, then V U F FMAs.  FULL = every vector of
// the tile exists (no per-vector predicates).
// One batch: U vectors starting at tile position j0 (J0 is j0 when it is a
// compile-time constant, -1 when the batch loop is rolled; then M == 1).
template <int V, int F, int G, int M, int U, bool VEC, bool FULL, bool NA, typename T>
__device__ __forceinline__ void mac_batch(const char *__restrict__ bptr, uint32_t stride,
                                          const bool (&cok)[F], unsigned gmask, int cnt,
                                          uint64_t pol, const int (&mc)[M],
                                          const float (&mv)[M][V], T (&acc)[V][F], int j0) {
  constexpr int FSTEP = G * (VEC ? 16 : 4);  // bytes between a lane's f-th columns
  T b[U][F];
  float vv[U][V];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = j0 + u;
    const int m = M == 1 ? 0 : j / G;
    const int c = __shfl_sync(gmask, mc[m], j % G, G);
#pragma unroll
    for (int k = 0; k < V; ++k) vv[u][k] = __shfl_sync(gmask, mv[m][k], j % G, G);
    const char *row = bptr + (uint64_t)(uint32_t)c * stride;
#pragma unroll
    for (int f = 0; f < F; ++f) {
      if ((FULL || j < cnt) && cok[f])
        ld_b<NA>(b[u][f], row + f * FSTEP, pol);
      else
        b[u][f] = zero_v<T>();
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < V; ++k)
#pragma unroll
      for (int f = 0; f < F; ++f) fma4(acc[k][f], vv[u][k], b[u][f]);
}

// PSPMM_NOHOIST = 1 keeps the batch loop rolled (M == 1 tiles), so at most
// U F B loads per lane are in flight and the register footprint stays small;
// 0 lets the compiler unroll a whole tile and hoist its loads.
#ifndef PSPMM_NOHOIST
#define PSPMM_NOHOIST 0
#endif
// float4 B loads a lane keeps in flight per batch (U = PSPMM_INFLIGHT / F)
#ifndef PSPMM_INFLIGHT
#define PSPMM_INFLIGHT 8
#endif

template <int V, int F, int G, int M, int U, bool VEC, bool FULL, bool NA, typename T>
__device__ __forceinline__ void mac_tile(const char *__restrict__ bptr, uint32_t stride,
                                         const bool (&cok)[F], unsigned gmask, int cnt,
                                         uint64_t pol, const int (&mc)[M],
                                         const float (&mv)[M][V], T (&acc)[V][F]) {
  constexpr int TILE = G * M;
  if constexpr (PSPMM_NOHOIST && M == 1 && TILE > U) {
#pragma unroll 1
    for (int j0 = 0; j0 < TILE; j0 += U) {
      if (FULL || j0 < cnt)
        mac_batch<V, F, G, M, U, VEC, FULL, NA>(bptr, stride, cok, gmask, cnt, pol, mc, mv, acc, j0);
    }
  } else {
#pragma unroll
    for (int j0 = 0; j0 < TILE; j0 += U) {
      if (FULL || j0 < cnt)  // uniform inside the group
        mac_batch<V, F, G, M, U, VEC, FULL, NA>(bptr, stride, cok, gmask, cnt, pol, mc, mv, acc, j0);
    }
  }
}

// Register budget: PSPMM_MAX_THREADS x PSPMM_MIN_BLOCKS threads per SM
// 256 x 3 -> at most 85 registers, 24 warps per SM: the best of the budgets
// A/B-tested on B200 (profiles/r01/ab_variants.md); tools/variants.py builds others.
#ifndef PSPMM_MAX_THREADS
#define PSPMM_MAX_THREADS 256
#endif
#ifndef PSPMM_MIN_BLOCKS
#define PSPMM_MIN_BLOCKS 3
#endif
// grid = at most PSPMM_WAVES waves of resident blocks (0 = one group per
// unit, the default: a grid-stride variant with cross-unit prefetch measured
// 5-14 % slower, profiles/r01/ab_variants.md)
#ifndef PSPMM_WAVES
#define PSPMM_WAVES 0
#endif

template <int V, int S, int F, int G, bool VEC, bool NA = false>
__global__ void __launch_bounds__(PSPMM_MAX_THREADS, PSPMM_MIN_BLOCKS)
    spmm_kernel(const SpmmArgs a) {
  using T = typename std::conditional<VEC, float4, float>::type;
  constexpr int VW = VEC ? 4 : 1;
  constexpr int GPW = 32 / G;
  constexpr int M = G >= 8 ? 1 : 8 / G;  // staged vectors per lane
  constexpr int TILE = G * M;            // vectors staged per group per round
  constexpr int U0 = (PSPMM_INFLIGHT / F) > 0 ? (PSPMM_INFLIGHT / F) : 1;
  // vectors whose B rows are in flight together: the largest power of two
  // <= min(U0, TILE), so it divides the (power-of-two) tile
  constexpr int U1 = U0 < TILE ? U0 : TILE;
  constexpr int U = U1 >= 16 ? 16 : U1 >= 8 ? 8 : U1 >= 4 ? 4 : U1 >= 2 ? 2 : 1;
  static_assert(TILE % U == 0, "tile/batch mismatch");

  const int lane = threadIdx.x & 31;
  const int g = lane / G;
  const int l = lane % G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // with a unit order (descending vector count, built with the PCSR), the
  // groups of a warp get units of similar length (less intra-warp idling)
  // and the longest units start first (shorter tail)
  const int64_t slot = a.unit_begin + warp * GPW + g;
  const int64_t unit = (a.order && slot < a.units) ? a.order[slot] : slot;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
  const int col0 = blockIdx.y * (G * F * VW);
  const uint64_t pol_a = policy_evict_first();
  const uint64_t pol_b = policy_evict_last();

  int coff[F];
  bool cok[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    coff[f] = col0 + (f * G + l) * VW;
    cok[f] = coff[f] < a.K;
  }
  // this lane's first column of B; row r is at bptr + r * stride
  const char *bptr = reinterpret_cast<const char *>(a.B + coff[0]);
  const uint32_t stride = (uint32_t)(a.ldb * 4);

  int head = 0, tail = 0;
  if (slot < a.units) {
    head = a.rowptr[unit];
    tail = a.rowptr[unit + 1];
  }

  T acc[V][F];
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int f = 0; f < F; ++f) acc[k][f] = zero_v<T>();

  // software pipeline over tiles: the next tile's (colIdx, val) loads are in
  // flight while the current tile's B rows are gathered
  int mc[M];
  float mv[M][V];
  if (head < tail) load_tile<V, M, G>(a, head, tail, l, pol_a, mc, mv);
  for (int base = head; base < tail; base += TILE) {
    int nc[M];
    float nv[M][V];
    const bool more = base + TILE < tail;
    if (more) load_tile<V, M, G>(a, base + TILE, tail, l, pol_a, nc, nv);
    const int cnt = tail - base;
    if (cnt >= TILE)
      mac_tile<V, F, G, M, U, VEC, true, NA>(bptr, stride, cok, gmask, cnt, pol_b, mc, mv, acc);
    else
      mac_tile<V, F, G, M, U, VEC, false, NA>(bptr, stride, cok, gmask, cnt, pol_b, mc, mv, acc);
    if (more) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        mc[m] = nc[m];
#pragma unroll
        for (int k = 0; k < V; ++k) mv[m][k] = nv[m][k];
      }
    }
  }

  if (slot >= a.units) return;
  if (S == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t row = unit * V + k;
      if (row < a.n_rows) {
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) put_c(a, row * a.ldc + coff[f], acc[k][f], false);
      }
    }
  } else {
    // S = 1 is launched as a programmatic dependent of the split-row zeroing
    // kernel (PDL): the grid starts while the zeroing runs, gathers its first
    // unit, and waits for the zeroing only here, before its first write (a
    // no-op without the launch attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int panel = a.trow[unit];
    const bool sole = (unit == 0 || a.trow[unit - 1] != panel) &&
                      (unit + 1 == a.units_total || a.trow[unit + 1] != panel);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t row = (int64_t)panel * V + k;
      if (row < a.n_rows) {
#pragma unroll
        for (int f = 0; f < F; ++f)
          if (cok[f]) put_c(a, row * a.ldc + coff[f], acc[k][f], !sole);
      }
    }
  }
  if (a.fan.n) __threadfence_system();  // peers read after the caller's barrier
}

using KernelFn = void (*)(const SpmmArgs);

template <int V, int S, int F, bool VEC, bool NA = false>
KernelFn pick_g(int G) {
  switch (G) {
    case 1: return spmm_kernel<V, S, F, 1, VEC, NA>;
    case 2: return spmm_kernel<V, S, F, 2, VEC, NA>;
    case 4: return spmm_kernel<V, S, F, 4, VEC, NA>;
    case 8: return spmm_kernel<V, S, F, 8, VEC, NA>;
    case 16: return spmm_kernel<V, S, F, 16, VEC, NA>;
    case 32: return spmm_kernel<V, S, F, 32, VEC, NA>;
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

// the 128-bit instances with L1::no_allocate B gathers
template <int V, int S>
KernelFn pick_na(int F, int G) {
  switch (F) {
    case 1: return pick_g<V, S, 1, true, true>(G);
    case 2: return pick_g<V, S, 2, true, true>(G);
    case 3: return pick_g<V, S, 3, true, true>(G);
    case 4: return pick_g<V, S, 4, true, true>(G);
    case 5: return pick_g<V, S, 5, true, true>(G);
    case 6: return pick_g<V, S, 6, true, true>(G);
    case 7: return pick_g<V, S, 7, true, true>(G);
    case 8: return pick_g<V, S, 8, true, true>(G);
    default: return nullptr;
  }
}

// one per (V, S) translation unit, and one per (V, S) for the NA instances
KernelFn pick_v1s0(bool vec, int F, int G);
KernelFn pick_v1s1(bool vec, int F, int G);
KernelFn pick_v2s0(bool vec, int F, int G);
KernelFn pick_v2s1(bool vec, int F, int G);
KernelFn pick_v1s0_na(int F, int G);
KernelFn pick_v1s1_na(int F, int G);
KernelFn pick_v2s0_na(int F, int G);
KernelFn pick_v2s1_na(int F, int G);

}  // namespace detail
}  // namespace pspmm
