// (a6, a7) Engine mode 2: the same ParamSpMM computation (Alg. 2,
// P:215-267) with the B-row gather done by the Tensor Memory Accelerator.
//
// Each warp owns one unit (panel / chunk) at a time and a private ring of
// STAGES shared-memory slots.  Lane 0 issues `cp.async.bulk.tensor.2d
// .tile::gather4` — one instruction lands the 4 B rows of 4 consecutive
// nonzero vectors (4 x 4·KP floats) in a slot and completes an mbarrier —
// while all 32 lanes consume the oldest slot with LDS.128 + FMA.  The data in
// flight lives in shared memory, not registers, so a warp keeps
// STAGES x 4 rows outstanding regardless of its register budget (the LDG
// engine is register-bound, profiles/r01/ab_variants.md).
//
// Lane mapping for a slot: KP float4 per row (box = 4·KP floats, K = 4·KP
// per pass), R = 32/KP rows per LDS instruction (KP < 32) or FQ = KP/32
// float4 per lane (KP >= 32).  A lane accumulates res[V][FQ] (Alg. 2 l.2) for
// its column(s) over the rows it visits; the R row-subgroups are summed with
// shuffles at the end of the unit, then stored / red-accumulated exactly as
// in the LDG engine (Alg. 2 l.17-30, c-9, c-12).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kStages = 8;

struct TmaArgs {
  const int32_t *__restrict__ rowptr;
  const int32_t *__restrict__ colidx;
  const float *__restrict__ val;
  const int32_t *__restrict__ trow;
  float *__restrict__ C;
  int64_t ldc;
  int32_t n_rows, unit_begin, units, units_total, K;  // units = end of this launch's range
  int32_t accumulate;                                  // 1: C += A.B
  Fanout fan;                                          // peer copies of C (f2)
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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int r0, int r1, int r2, int r3,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3), "l"(policy)
      : "memory");
}
__device__ __forceinline__ int ld_stream(const int32_t *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float *p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

template <int V, int S, int KP>
__global__ void __launch_bounds__(256, 1) spmm_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                           const TmaArgs a) {
  constexpr int R = KP >= 32 ? 1 : 32 / KP;   // rows per LDS instruction
  constexpr int FQ = KP >= 32 ? KP / 32 : 1;  // float4 per lane per row
  constexpr int SLOT = 4 * KP * 16;           // bytes per slot (4 rows)
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  unsigned char *ring = smem + (size_t)warp * kStages * SLOT;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)nwarps * kStages * SLOT) +
                   warp * kStages;
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));

  const int rsub = lane / KP % R;        // which of the R rows of an LDS step
  const int q = KP >= 32 ? lane : lane % KP;  // float4 column (first of FQ)
  const int c0 = blockIdx.y * 4 * KP;    // first float column of this pass
  const int64_t unit = a.unit_begin + (int64_t)blockIdx.x * nwarps + warp;
  if (unit >= a.units) return;
  const int head = a.rowptr[unit], tail = a.rowptr[unit + 1];
  const int nvec = tail - head;
  const int nquad = (nvec + 3) >> 2;

  float4 acc[V][FQ];
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int f = 0; f < FQ; ++f) acc[k][f] = make_float4(0.f, 0.f, 0.f, 0.f);

  // colIdx of the unit, a 32-vector register window running kStages quads
  // ahead of consumption (lane i holds vector wbase + i); padding -> row 0
  int wcol = 0;
  int wbase = -1;
  // issue quad t into slot t % kStages (all lanes call; lane 0 issues)
  auto issue = [&](int t) {
    const int base = t * 4;
    if ((base & ~31) != wbase) {
      wbase = base & ~31;
      const int i = head + wbase + lane;
      wcol = i < tail ? ld_stream(a.colidx + i) : 0;
    }
    int icol[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) icol[r] = __shfl_sync(0xffffffffu, wcol, (base + r) & 31);
    if (lane == 0) {
      const int s = t % kStages;
      mbar_expect_tx(&bars[s], SLOT);
      tma_gather4(ring + s * SLOT, &map, &bars[s], c0, icol[0], icol[1], icol[2], icol[3], pol);
    }
  };
  // the V values of the 4 vectors of quad t (padding -> 0)
  float qv[V][4];
  int vbase = -1;
  float vwin[V];
  auto qvals = [&](int t) {
    const int base = t * 4;
    if ((base & ~31) != vbase) {
      const int i = head + (base & ~31) + lane;
#pragma unroll
      for (int k = 0; k < V; ++k) vwin[k] = i < tail ? ld_stream(a.val + (int64_t)i * V + k) : 0.f;
      vbase = base & ~31;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k) qv[k][r] = __shfl_sync(0xffffffffu, vwin[k], (base + r) & 31);
  };

  const int pro = nquad < kStages ? nquad : kStages;
  for (int t = 0; t < pro; ++t) issue(t);
  for (int t = 0; t < nquad; ++t) {
    const int s = t % kStages;
    const uint32_t parity = (uint32_t)(t / kStages) & 1u;
    qvals(t);
    mbar_wait(&bars[s], parity);
    const float4 *slot = reinterpret_cast<const float4 *>(ring + s * SLOT);
#pragma unroll
    for (int r0 = 0; r0 < 4; r0 += R) {
      const int r = r0 + rsub;
#pragma unroll
      for (int f = 0; f < FQ; ++f) {
        const float4 b = slot[r * KP + q + f * 32];
#pragma unroll
        for (int k = 0; k < V; ++k) {
          // r is lane-dependent: select the quad value by r
          const float v = r == 0 ? qv[k][0] : r == 1 ? qv[k][1] : r == 2 ? qv[k][2] : qv[k][3];
          acc[k][f].x = fmaf(v, b.x, acc[k][f].x);
          acc[k][f].y = fmaf(v, b.y, acc[k][f].y);
          acc[k][f].z = fmaf(v, b.z, acc[k][f].z);
          acc[k][f].w = fmaf(v, b.w, acc[k][f].w);
        }
      }
    }
    __syncwarp();
    if (t + kStages < nquad) issue(t + kStages);
  }
  // the (zero-valued) padding of the last quad gathered row icol = 0 rows: harmless

  // reduce the R row-subgroups: lanes q, q + KP, q + 2 KP, ...
#pragma unroll
  for (int off = KP; off < 32; off <<= 1)
#pragma unroll
    for (int k = 0; k < V; ++k)
#pragma unroll
      for (int f = 0; f < FQ; ++f) {
        acc[k][f].x += __shfl_xor_sync(0xffffffffu, acc[k][f].x, off);
        acc[k][f].y += __shfl_xor_sync(0xffffffffu, acc[k][f].y, off);
        acc[k][f].z += __shfl_xor_sync(0xffffffffu, acc[k][f].z, off);
        acc[k][f].w += __shfl_xor_sync(0xffffffffu, acc[k][f].w, off);
      }
  if (lane >= KP && KP < 32) return;
  int64_t prow;
  bool sole = true;
  if (S == 0) {
    prow = unit;
  } else {
    prow = a.trow[unit];
    sole = (unit == 0 || a.trow[unit - 1] != prow) &&
           (unit + 1 == a.units_total || a.trow[unit + 1] != prow);
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int64_t row = prow * V + k;
    if (row >= a.n_rows) continue;
    float4 *crow = reinterpret_cast<float4 *>(a.C + row * a.ldc + c0);
#pragma unroll
    for (int f = 0; f < FQ; ++f) {
      if (sole) {
        float4 v = acc[k][f];
        if (a.accumulate) {
          const float4 o = crow[q + f * 32];
          v.x += o.x;
          v.y += o.y;
          v.z += o.z;
          v.w += o.w;
        }
        __stcs(crow + q + f * 32, v);
#pragma unroll 1
        for (int d = 0; d < a.fan.n; ++d)
          __stcs(reinterpret_cast<float4 *>(a.fan.peer[d] + row * a.ldc + c0) + q + f * 32, v);
      } else {
        atomicAdd(crow + q + f * 32, acc[k][f]);
#pragma unroll 1
        for (int d = 0; d < a.fan.n; ++d)
          atomicAdd(reinterpret_cast<float4 *>(a.fan.peer[d] + row * a.ldc + c0) + q + f * 32,
                    acc[k][f]);
      }
    }
  }
  if (a.fan.n) __threadfence_system();
}

using TmaFn = void (*)(const CUtensorMap, const TmaArgs);

template <int V, int S>
TmaFn pick_kp(int KP) {
  switch (KP) {
    case 8: return spmm_tma_kernel<V, S, 8>;
    case 16: return spmm_tma_kernel<V, S, 16>;
    case 32: return spmm_tma_kernel<V, S, 32>;
    case 64: return spmm_tma_kernel<V, S, 64>;
    default: return nullptr;
  }
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

}  // namespace

// float4 columns per pass: the largest of {64, 32, 16, 8} dividing K/4 (0 = none)
static int tma_kp(int32_t K) {
  if (K % 4 != 0) return 0;
  for (int c : {64, 32, 16, 8})
    if ((K / 4) % c == 0) return c;
  return 0;
}

bool tma_supported(int32_t K, int64_t ldb, int64_t ldc, const float *d_B, const float *d_C) {
  return tma_kp(K) != 0 && ldb % 4 == 0 && ldc % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0;
}

// Mode 2 dispatch (called from run_spmm after validation and the S = 1 zeroing).
pspmm_status run_spmm_tma(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                          float *d_C, int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                          int64_t u0, int64_t u1, int32_t accumulate, const Fanout &fan) {
  if (!tma_supported(K, ldb, ldc, d_B, d_C))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run mode 2: unsupported K / layout");
  const int KP = tma_kp(K);
  const int passes = K / 4 / KP;
  auto encode = get_encode();
  if (!encode) PSPMM_FAIL(PSPMM_ERR_CUDA, "spmm_run mode 2: cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)A->n_cols};
  cuuint64_t strides[1] = {(cuuint64_t)ldb * 4};
  cuuint32_t box[2] = {(cuuint32_t)(4 * KP), 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(d_B), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) PSPMM_FAIL(PSPMM_ERR_CUDA, "spmm_run mode 2: tensor map encode failed");
  TmaFn fn = A->V == 1 ? (A->S ? pick_kp<1, 1>(KP) : pick_kp<1, 0>(KP))
                       : (A->S ? pick_kp<2, 1>(KP) : pick_kp<2, 0>(KP));
  if (!fn) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 2: no instance");
  const int warps = std::min(cfg.W, 8);
  const size_t smem = (size_t)warps * kStages * (4 * KP * 16) + (size_t)warps * kStages * 8;
  if (smem > 227 * 1024) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run mode 2: W too large for this K");
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TmaArgs args;
  args.rowptr = A->d_rowptr;
  args.colidx = A->d_colidx;
  args.val = A->d_val;
  args.trow = A->d_trow;
  args.C = d_C;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.unit_begin = (int32_t)u0;
  args.units = (int32_t)u1;
  args.units_total = (int32_t)A->num_chunks;
  args.K = K;
  args.accumulate = accumulate;
  args.fan = fan;
  if (u1 <= u0) return PSPMM_OK;
  const int64_t bx = (u1 - u0 + warps - 1) / warps;
  fn<<<dim3((unsigned)bx, (unsigned)passes), warps * 32, smem, stream>>>(map, args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
