// Microbenchmark library (ctypes, tools/stream_ceiling.py): how fast can one
// persistent CTA per SM stream a dense n x Ki fp32 matrix X through a TMA
// ring (the dense product's load path, gemm_tc.cu), with and without a TMA
// store of every tile to T (the product's store path), against plain
// LDG.128 streaming.  No tensor cores: the ceiling of the data movement.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//      -o tools/libmb_stream.so tools/mb_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

namespace {

constexpr int kM = 128, kKc = 32, kPart = kM * kKc * 4;  // 16 KB: 128 rows x 128 B

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}

// stage = one tile's chunks: `chunks` 2-D boxes (32 columns x 128 rows) or
// one 3-D box (32 x 128 x chunks) landing as [chunk][row][128 B]
__global__ void __launch_bounds__(64, 1)
    tma_stream(const __grid_constant__ CUtensorMap xm, const __grid_constant__ CUtensorMap tm,
               int64_t n, int chunks, int stages, int box3d, int store) {
  extern __shared__ uint8_t sraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sraw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = chunks * kPart;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)stages * stage_bytes);
  uint64_t *empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = (n + kM - 1) / kM;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {  // producer
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages;
      if (it >= stages) bar_wait(&empty[s], ((it / stages) - 1) & 1);
      bar_tx(&full[s], stage_bytes);
      const uint32_t dst = su32(sm + (size_t)s * stage_bytes);
      if (box3d) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(&xm)), "r"(su32(&full[s])), "r"(0), "r"((int)(t * kM)),
            "r"(0)
            : "memory");
      } else {
        for (int c = 0; c < chunks; ++c)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst + c * kPart),
              "l"(reinterpret_cast<uint64_t>(&xm)), "r"(su32(&full[s])), "r"(c * kKc),
              "r"((int)(t * kM))
              : "memory");
      }
    }
  } else if (warp == 1 && lane == 0) {  // consumer: optional TMA store, then release
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages;
      bar_wait(&full[s], (it / stages) & 1);
      if (store) {
        for (int c = 0; c < chunks; ++c)
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&tm)),
              "r"(c * kKc), "r"((int)(t * kM)), "r"(su32(sm + (size_t)s * stage_bytes + c * kPart))
              : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      bar_arrive(&empty[s]);
    }
    if (store) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}

__global__ void ldg_stream(const float4 *__restrict__ x, int64_t n4, float *__restrict__ out) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x + i);
    a.x += v.x;
    a.y += v.y;
    a.z += v.z;
    a.w += v.w;
  }
  if (a.x + a.y + a.z + a.w == 1234.5f) out[0] = a.x;  // keep the loads
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

extern "C" int mb_tma_stream(const float *X, float *T, int64_t n, int Ki, int stages, int box3d,
                             int store, void *stream) {
  auto enc = encoder();
  if (!enc || Ki % kKc) return 1;
  const int chunks = Ki / kKc;
  CUtensorMap xm, tm;
  cuuint32_t estr[3] = {1, 1, 1};
  if (box3d) {  // dims (32 columns, rows, chunks): the box lands as [chunk][row][32]
    cuuint64_t dims[3] = {(cuuint64_t)kKc, (cuuint64_t)n, (cuuint64_t)chunks};
    cuuint64_t strides[2] = {(cuuint64_t)Ki * 4, (cuuint64_t)kKc * 4};
    cuuint32_t box[3] = {(cuuint32_t)kKc, (cuuint32_t)kM, (cuuint32_t)chunks};
    if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(X), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 2;
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)Ki, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)Ki * 4};
    cuuint32_t box[2] = {(cuuint32_t)kKc, (cuuint32_t)kM};
    if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 2;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)Ki, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)Ki * 4};
    cuuint32_t box[2] = {(cuuint32_t)kKc, (cuuint32_t)kM};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, T, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 3;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 1024 + (size_t)stages * chunks * kPart + 16 * stages + 64;
  if (smem > 227 * 1024) return 4;
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tiles = (n + kM - 1) / kM;
  tma_stream<<<(int)(tiles < sms ? tiles : sms), 64, smem, (cudaStream_t)stream>>>(
      xm, tm, n, chunks, stages, box3d, store);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" int mb_ldg_stream(const float *X, int64_t nfloats, float *out, int blocks, void *stream) {
  ldg_stream<<<blocks, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4 *>(X),
                                                      nfloats / 4, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
