// (f3) GNN layer on top of the engine (GCN /
// GIN layers are H' = A . H . W): the dense product with the layer weight
// and the SpMM, ordered so the SpMM runs on the narrower side.
//
// dense_gemm: T = X . W.  Shapes the tensor-core product takes (Ki % 32,
// Ko % 16, Ko <= 256, W's TF32 image in shared memory) run gemm_tc.cu's
// 3xTF32 tcgen05 kernel; the rest run dense_gemm_kernel below.
//
// dense_gemm_kernel: T = X . W in fp32 on CUDA cores.  X is n x Ki (row
// major, ldx), W is Ki x Ko (row major, ldw), T is n x Ko.  This is an
// HBM-bound skinny product (Ki, Ko <= 256, n ~ 10^5..10^6: 2 n Ki Ko flops
// against 4 n (Ki + Ko) bytes), so it is written for bandwidth, not for the
// tensor cores: a block stages a Ko-tile of W (Ki x 64 floats) in shared
// memory once, then each thread computes RT = 4 rows x one float4 of T,
// streaming its rows of X (each X element is read by the 16 threads of a
// row, an L1 broadcast) and reusing every W float4 four times.  fp32 with
// sequential accumulation over Ki (error <= Ki 2^-24 sum |x||w|).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kRT = 4;        // rows per thread
constexpr int kTileCols = 64; // Ko columns per block (16 float4)

__global__ void __launch_bounds__(256) dense_gemm_kernel(int64_t n, int Ki, int Ko,
                                                         const float *__restrict__ X, int64_t ldx,
                                                         const float *__restrict__ W, int64_t ldw,
                                                         float *__restrict__ T, int64_t ldt) {
  extern __shared__ __align__(16) float ws[];  // [Ki][kTileCols]
  const int c0 = blockIdx.y * kTileCols;
  const int ncols = min(kTileCols, Ko - c0);
  for (int i = threadIdx.x; i < Ki * kTileCols; i += blockDim.x) {
    const int k = i / kTileCols, c = i % kTileCols;
    ws[i] = c < ncols ? W[(int64_t)k * ldw + c0 + c] : 0.f;
  }
  __syncthreads();
  const int q = threadIdx.x % 16;  // float4 column of the tile
  const int rsub = threadIdx.x / 16;  // 16 row slots per block pass
  const bool col_ok = q * 4 < ncols;
  const int64_t rows_per_pass = (int64_t)gridDim.x * 16 * kRT;
  for (int64_t r0 = ((int64_t)blockIdx.x * 16 + rsub) * kRT; r0 < n; r0 += rows_per_pass) {
    float4 acc[kRT];
#pragma unroll
    for (int t = 0; t < kRT; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < Ki; ++k) {
      const float4 w = reinterpret_cast<const float4 *>(ws + k * kTileCols)[q];
#pragma unroll
      for (int t = 0; t < kRT; ++t) {
        const float x = r0 + t < n ? __ldg(X + (r0 + t) * ldx + k) : 0.f;
        acc[t].x = fmaf(x, w.x, acc[t].x);
        acc[t].y = fmaf(x, w.y, acc[t].y);
        acc[t].z = fmaf(x, w.z, acc[t].z);
        acc[t].w = fmaf(x, w.w, acc[t].w);
      }
    }
    if (!col_ok) continue;
#pragma unroll
    for (int t = 0; t < kRT; ++t) {
      if (r0 + t >= n) break;
      float *dst = T + (r0 + t) * ldt + c0 + q * 4;
      if (q * 4 + 4 <= ncols && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        __stcs(reinterpret_cast<float4 *>(dst), acc[t]);
      } else {
        const float v[4] = {acc[t].x, acc[t].y, acc[t].z, acc[t].w};
        for (int e = 0; e < 4 && q * 4 + e < ncols; ++e) dst[e] = v[e];
      }
    }
  }
}

}  // namespace

pspmm_status dense_gemm(int64_t n, int32_t Ki, int32_t Ko, const float *d_X, int64_t ldx,
                        const float *d_W, int64_t ldw, float *d_T, int64_t ldt,
                        cudaStream_t stream) {
  if (!d_X || !d_W || !d_T) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "dense_gemm: null pointer");
  if (n < 0 || Ki < 1 || Ko < 1 || ldx < Ki || ldw < Ko || ldt < Ko)
    PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "dense_gemm: need Ki, Ko >= 1 and ld >= width");
  // the tensor-core product (gemm_tc.cu) where its shape rules hold; the
  // CUDA-core kernel below for every other shape (PSPMM_GEMM_CC=1 forces it,
  // an A/B knob for the tools)
  const char *cc = std::getenv("PSPMM_GEMM_CC");
  if (!(cc && cc[0] == '1') && gemm_tc_supported(Ki, Ko, d_X, ldx, d_W, ldw, d_T, ldt))
    return gemm_tc(n, Ki, Ko, d_X, ldx, d_W, ldw, d_T, ldt, stream);
  const size_t smem = (size_t)Ki * kTileCols * sizeof(float);
  if (smem > 200 * 1024) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "dense_gemm: Ki > 800");
  if (n == 0) return PSPMM_OK;
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(dense_gemm_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t row_blocks = (n + 16 * kRT - 1) / (16 * kRT);
  const int by = (Ko + kTileCols - 1) / kTileCols;
  const int64_t bx = std::min<int64_t>(row_blocks, (int64_t)num_sms() * 8);
  dense_gemm_kernel<<<dim3((unsigned)bx, (unsigned)by), 256, smem, stream>>>(n, Ki, Ko, d_X, ldx,
                                                                            d_W, ldw, d_T, ldt);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace pspmm
