// Microbenchmark library (ctypes, tools/gather_ceiling.py): the bare B-row
// gather with the workload's OWN column stream and the
// narrow-row gathers a K-sliced engine would issue (SURVEY
// §8(d) "K-slicing").  No A values, no FMAs, no C: a group of G lanes reads
// F float4 of row idx[j] (row_bytes = 16 G F) at `stride` bytes per row, U
// rows in flight per group, and folds them into a register sum.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//      -o tools/libmb_gather.so tools/mb_gather.cu
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int G, int F, int U>
__global__ void __launch_bounds__(256, 3)
    gather(const char *__restrict__ B, uint32_t stride, const int *__restrict__ idx,
           long long m, float *__restrict__ out) {
  const int lane = threadIdx.x & 31, l = lane % G;
  const long long groups = (long long)gridDim.x * blockDim.x / G;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const char *base = B + l * 16;
  for (long long i = gid * U; i < m; i += groups * U) {
    float4 b[U][F];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = i + u;
      const int r = j < m ? __ldg(idx + j) : 0;
      const char *row = base + (uint64_t)(uint32_t)r * stride;
#pragma unroll
      for (int f = 0; f < F; ++f)
        b[u][f] = __ldg(reinterpret_cast<const float4 *>(row + f * G * 16));
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int f = 0; f < F; ++f) {
        acc.x += b[u][f].x;
        acc.y += b[u][f].y;
        acc.z += b[u][f].z;
        acc.w += b[u][f].w;
      }
  }
  if (acc.x == 12345.678f) out[0] = acc.y + acc.z + acc.w;
}

using Fn = void (*)(const char *, uint32_t, const int *, long long, float *);

template <int G, int F>
Fn pick_u(int U) {
  switch (U) {
    case 2: return gather<G, F, 2>;
    case 4: return gather<G, F, 4>;
    case 8: return gather<G, F, 8>;
    case 16: return gather<G, F, 16>;
    default: return nullptr;
  }
}

template <int G>
Fn pick_f(int F, int U) {
  switch (F) {
    case 1: return pick_u<G, 1>(U);
    case 2: return pick_u<G, 2>(U);
    default: return nullptr;
  }
}

Fn pick(int G, int F, int U) {
  switch (G) {
    case 1: return pick_f<1>(F, U);
    case 2: return pick_f<2>(F, U);
    case 4: return pick_f<4>(F, U);
    case 8: return pick_f<8>(F, U);
    case 16: return pick_f<16>(F, U);
    case 32: return pick_f<32>(F, U);
    default: return nullptr;
  }
}

}  // namespace

extern "C" int mb_gather(const float *B, int64_t stride_bytes, const int32_t *idx, int64_t m,
                         int32_t G, int32_t F, int32_t U, float *out, void *stream) {
  Fn fn = pick(G, F, U);
  if (!fn) return 1;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  fn<<<sms * 3, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const char *>(B), (uint32_t)stride_bytes, idx, (long long)m, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
