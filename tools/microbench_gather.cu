// Microbenchmark: random B-row gather bandwidth on B200.
// Compares (1) the engine's LDG.128 row gather (G lanes x 16 B per row) with
// (2) a TMA tile::gather4 pipeline (4 rows per cp.async.bulk.tensor, landed
// in shared memory, consumed with LDS.128), for an L2-resident B (Reddit:
// 232965 x 64 fp32 = 60 MB) and an HBM-resident B (products: 2449029 x 128).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_gather.cu
// ./mb [rows] [K] [gathers]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// ---------------------------------------------------------------- LDG gather
template <int G, int U>
__global__ void __launch_bounds__(256, 3) ldg_gather(const float *__restrict__ B, int K,
                                                      const int *__restrict__ idx, long long m,
                                                      float *__restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane / G, l = lane % G;
  const long long groups = (long long)gridDim.x * blockDim.x / G;
  long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  float4 acc = make_float4(0, 0, 0, 0);
  const char *base = reinterpret_cast<const char *>(B) + l * 16;
  const uint32_t stride = K * 4;
  for (long long i = gid * U; i < m; i += groups * U) {
    float4 b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long j = i + u;
      int r = j < m ? __ldg(idx + j) : 0;
      b[u] = __ldg(reinterpret_cast<const float4 *>(base + (uint64_t)(uint32_t)r * stride));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x += b[u].x; acc.y += b[u].y; acc.z += b[u].z; acc.w += b[u].w;
    }
  }
  (void)g;
  if (acc.x == 12345.678f) out[0] = acc.y + acc.z + acc.w;
}

// ---------------------------------------------------------------- TMA gather4
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
                                            int c0, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2),
      "r"(r3)
      : "memory");
}

// each warp: STAGES slots of 4 rows x K floats; lane 0 produces, all lanes consume
template <int STAGES>
__global__ void __launch_bounds__(256, 1) tma_gather(const __grid_constant__ CUtensorMap map,
                                                      int K, const int *__restrict__ idx,
                                                      long long m, float *__restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int slot_bytes = 4 * K * 4;
  unsigned char *my = smem + (size_t)warp * STAGES * slot_bytes;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)nwarps * STAGES * slot_bytes) +
                   warp * STAGES;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long warps_total = (long long)gridDim.x * nwarps;
  const long long wid = (long long)blockIdx.x * nwarps + warp;
  // this warp's quads: q = wid, wid + warps_total, ...
  const long long nquads = m / 4;
  float4 acc = make_float4(0, 0, 0, 0);
  long long q_issue = wid;
  // prologue: fill the ring
  for (int s = 0; s < STAGES; ++s, q_issue += warps_total) {
    if (q_issue < nquads && lane == 0) {
      const int *p = idx + q_issue * 4;
      mbar_expect_tx(&bars[s], slot_bytes);
      tma_gather4(my + s * slot_bytes, &map, &bars[s], 0, p[0], p[1], p[2], p[3]);
    }
  }
  uint32_t phase = 0;
  int s = 0;
  for (long long q = wid; q < nquads; q += warps_total) {
    mbar_wait(&bars[s], phase);
    const float4 *rows = reinterpret_cast<const float4 *>(my + s * slot_bytes);
    const int per_row = K / 4;  // float4 per row
    for (int e = lane; e < 4 * per_row; e += 32) {
      float4 v = rows[e];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    if (q_issue < nquads && lane == 0) {
      const int *p = idx + q_issue * 4;
      mbar_expect_tx(&bars[s], slot_bytes);
      tma_gather4(my + s * slot_bytes, &map, &bars[s], 0, p[0], p[1], p[2], p[3]);
    }
    q_issue += warps_total;
    if (++s == STAGES) {
      s = 0;
      phase ^= 1;
    }
  }
  if (acc.x == 12345.678f) out[0] = acc.y + acc.z + acc.w;
}

// semantics check: gather rows {r0..r3} and copy the landed tile to global
__global__ void tma_check(const __grid_constant__ CUtensorMap map, int K, int r0, int r1, int r2,
                          int r3, float *out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 4 * K * 4);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, 4 * K * 4);
    tma_gather4(smem, &map, bar, 0, r0, r1, r2, r3);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < 4 * K; i += blockDim.x) out[i] = reinterpret_cast<float *>(smem)[i];
}

int main(int argc, char **argv) {
  long long n = argc > 1 ? atoll(argv[1]) : 232965;
  int K = argc > 2 ? atoi(argv[2]) : 64;
  long long m = argc > 3 ? atoll(argv[3]) : 114615892;
  m -= m % 4;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("rows=%lld K=%d gathers=%lld (B = %.1f MB, gathered = %.2f GB) SMs=%d\n", n, K, m,
         n * K * 4 / 1e6, m * K * 4.0 / 1e9, sms);
  std::vector<int> h(m);
  std::mt19937_64 rng(1);
  for (long long i = 0; i < m; ++i) h[i] = (int)(rng() % n);
  float *B, *out;
  int *idx;
  CK(cudaMalloc(&B, n * K * 4));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&out, 16));
  CK(cudaMemset(B, 0, n * K * 4));
  CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, const char *name) {
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    printf("%-34s %8.3f ms  %8.1f GB/s gathered\n", name, best, m * K * 4.0 / best / 1e6);
  };
  // LDG variants (G lanes x 16 B = one row; K = 64 -> G = 16, K = 128 -> G = 32)
  if (K == 64) {
    timeit([&] { ldg_gather<16, 8><<<sms * 24, 256>>>(B, K, idx, m, out); }, "ldg G16 U8");
    timeit([&] { ldg_gather<16, 16><<<sms * 24, 256>>>(B, K, idx, m, out); }, "ldg G16 U16");
    timeit([&] { ldg_gather<16, 4><<<sms * 24, 256>>>(B, K, idx, m, out); }, "ldg G16 U4");
  } else if (K == 128) {
    timeit([&] { ldg_gather<32, 8><<<sms * 24, 256>>>(B, K, idx, m, out); }, "ldg G32 U8");
    timeit([&] { ldg_gather<32, 16><<<sms * 24, 256>>>(B, K, idx, m, out); }, "ldg G32 U16");
  }
  // TMA gather4
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q));
  for (int box_rows : {1, 4}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)K * 4};
    cuuint32_t box[2] = {(cuuint32_t)(K > 256 ? 256 : K), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map box {%d, %d}: encode status %d\n", box[0], box[1], (int)r);
    if (r != CUDA_SUCCESS) continue;
    {
      // fill a probe B with B[r][c] = r * 1000 + c and check the landed rows
      std::vector<float> hb((size_t)16 * K);
      for (int rr = 0; rr < 16; ++rr)
        for (int c = 0; c < K; ++c) hb[(size_t)rr * K + c] = rr * 1000.f + c;
      CK(cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
      float *chk;
      CK(cudaMalloc(&chk, 4 * K * 4));
      CK(cudaFuncSetAttribute(tma_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * K * 4 + 16));
      tma_check<<<1, 128, 4 * K * 4 + 16>>>(map, K, 5, 1, 9, 2, chk);
      CK(cudaDeviceSynchronize());
      std::vector<float> hc(4 * K);
      CK(cudaMemcpy(hc.data(), chk, 4 * K * 4, cudaMemcpyDeviceToHost));
      const int rows[4] = {5, 1, 9, 2};
      int bad = 0;
      for (int i = 0; i < 4; ++i)
        for (int c = 0; c < K; ++c) bad += hc[i * K + c] != rows[i] * 1000.f + c;
      printf("  gather4 semantics (rows 5,1,9,2 as 4 x K row-major): %s (%d mismatches; first row "
             "starts %.0f %.0f)\n", bad ? "MISMATCH" : "ok", bad, hc[0], hc[1]);
      CK(cudaFree(chk));
      CK(cudaMemset(B, 0, n * K * 4));
    }
    for (int warps : {4, 8}) {
      constexpr int STAGES = 8;
      size_t smem = (size_t)warps * STAGES * (4 * K * 4 + 8);
      if (smem > 227 * 1024) continue;
      CK(cudaFuncSetAttribute(tma_gather<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
      int per_sm = (int)((227 * 1024) / smem);
      if (per_sm < 1) per_sm = 1;
      char name[96];
      snprintf(name, sizeof name, "tma gather4 box%d w%d s%d x%d/SM", box_rows, warps, STAGES,
               per_sm);
      timeit([&] {
        tma_gather<STAGES><<<sms * per_sm, warps * 32, smem>>>(map, K, idx, m, out);
      }, name);
    }
  }
  return 0;
}
