// (a6, a7) Host dispatch of the ParamSpMM computing engine (Alg. 2,
// P:215-267) and its two helper kernels.  The kernel template and its
// design notes are in spmm_kernel.cuh.
#include <algorithm>

#include "spmm_kernel.cuh"

namespace pspmm {
namespace {
using namespace detail;

// Zero the C rows of panels that own more than one chunk (S = 1, c-12).
// mc = 1: C is a multicast address, zeroed with multimem stores (every
// bound copy at once).
__global__ void zero_split_kernel(const int32_t *__restrict__ split, int64_t num_split, int V,
                                  int64_t n_rows, int32_t K, float *__restrict__ C, int64_t ldc,
                                  int mc, int vec4) {
  // the engine (a programmatic dependent) may launch now; it waits for this
  // grid's completion before its first write
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t q = vec4 ? K / 4 : K;  // stores per row
  const int64_t per = (int64_t)V * q;
  const int64_t total = num_split * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / per, r = t - s * per;
    const int64_t k = r / q, j = r - k * q;
    const int64_t row = (int64_t)split[s] * V + k;
    if (row >= n_rows) continue;
    float *p = C + row * ldc + (vec4 ? 4 * j : j);
    if (vec4 && !mc) {
      *reinterpret_cast<float4 *>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int e = 0; e < (vec4 ? 4 : 1); ++e) {
        if (mc)
          mc_st(p + e, 0.f);
        else
          p[e] = 0.f;
      }
    }
  }
}

// C = 0 (nnz_V == 0).
__global__ void zero_all_kernel(int64_t n_rows, int32_t K, float *__restrict__ C, int64_t ldc,
                                int mc) {
  const int64_t total = n_rows * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (mc)
      mc_st(C + (t / K) * ldc + t % K, 0.f);
    else
      C[(t / K) * ldc + t % K] = 0.f;
  }
}

KernelFn pick_kernel(int V, int S, bool vec, int F, int G, bool na) {
  if (vec && na) {
    if (V == 1) return S ? pick_v1s1_na(F, G) : pick_v1s0_na(F, G);
    return S ? pick_v2s1_na(F, G) : pick_v2s0_na(F, G);
  }
  if (V == 1) return S ? pick_v1s1(vec, F, G) : pick_v1s0(vec, F, G);
  return S ? pick_v2s1(vec, F, G) : pick_v2s0(vec, F, G);
}

bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

int ceil_pow2(int64_t x) {
  int p = 1;
  while (p < x && p < 32) p <<= 1;
  return p;
}

}  // namespace

namespace {

// Validated launch plan of one engine call.
struct Plan {
  KernelFn fn = nullptr;
  int threads = 0, G = 1;
  int64_t by = 1;
};

pspmm_status make_plan(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                       const float *d_C, int64_t ldc, const pspmm_config &cfg, Plan *plan) {
  if (!A || !d_B || !d_C) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run: null handle or pointer");
  if (K < 1 || ldb < K || ldc < K)
    PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "spmm_run: need K >= 1, ldb >= K, ldc >= K");
  if (cfg.V != A->V || cfg.S != A->S || cfg.omega != A->omega)
    PSPMM_FAIL(PSPMM_ERR_CONFIG_MISMATCH, "spmm_run: cfg.V/S/omega differ from the PCSR handle");
  if (cfg.mode != 0 && cfg.mode != 2 && cfg.mode != 3)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run: mode must be 0 (LDG engine), 1 (dense tiles on tensor cores), "
               "2 (TMA gather), 3 (short rows), 5 (row blocks) or 6 (staged bands)");
  if (!(cfg.W == 1 || cfg.W == 2 || cfg.W == 4 || cfg.W == 8))
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: W must be 1, 2, 4 or 8");
  if (cfg.W * 32 > PSPMM_MAX_THREADS)
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: W exceeds this build's launch bounds");
  if (cfg.F < 1 || cfg.F > 8)
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: F must be in 1..8 (float4 units)");
  if (cfg.G != 0 && !(pow2(cfg.G) && cfg.G <= 32))
    PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: G must be 0 or a power of two <= 32");
  if ((uint64_t)ldb * 4 >= (1ull << 32))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: ldb * 4 bytes must be < 2^32");
  if (cfg.order != 0 && cfg.order != 1) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: order must be 0 or 1");
  if (cfg.mode == 2) {
    if (!tma_supported(K, ldb, ldc, d_B, d_C))
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
                 "spmm_run mode 2: needs K % 32 == 0, ld % 4 == 0 and 16-B aligned B and C");
    return PSPMM_OK;
  }
  if (cfg.mode == 3) {
    if (!short_supported(A, K, ldb, ldc, d_B, d_C, cfg))
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
                 "spmm_run mode 3: needs V = 1, S = 0, F in {1, 2, 4}, K and ld % 4 == 0, "
                 "16-B aligned B and C");
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
  // B far larger than L2 (> 2x): its gathers cannot hit in L1, so they skip
  // L1 allocation (A/B: products-shaped -5 %)
  // (Reddit, B = 0.45 x L2: no_allocate measured 1.6067 vs 1.6067 ms, so the
  // rule stays at 2 x L2; profiles/r02/gemm_r3/reddit_b_na_ab.jsonl)
  const bool na = (double)A->n_cols * (double)ldb * 4.0 > 2.0 * (double)l2_bytes();
  plan->fn = pick_kernel(A->V, A->S, vec, F, G, na);
  if (!plan->fn) PSPMM_FAIL(PSPMM_ERR_CONFIG, "spmm_run: no kernel instance for this config");
  plan->threads = cfg.W * 32;
  plan->G = G;
  plan->by = (K + cols_per_pass - 1) / cols_per_pass;
  if (plan->by > 65535) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: too many column passes");
  return PSPMM_OK;
}

// C rows of split panels = 0 (S = 1, c-12); everything else is overwritten.
// With a fan-out the peer copies are zeroed the same way.
pspmm_status prepare_c(const pspmm_pcsr_s *A, int32_t K, float *d_C, int64_t ldc,
                       cudaStream_t stream, const Fanout &fan) {
  for (int d = fan.mc ? 0 : -1; d < fan.n; ++d) {  // multicast: the one mc address
    float *C = d < 0 ? d_C : fan.peer[d];
    if (A->nnz_v == 0) {
      const int64_t total = A->n_rows * K;
      const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
      zero_all_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(A->n_rows, K, C, ldc,
                                                                    fan.mc);
      PSPMM_CUDA_TRY(cudaGetLastError());
    } else if (A->S == 1 && A->num_split > 0) {
      // float4 stores when every row start is 16-B aligned
      const int vec4 = K % 4 == 0 && ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
      const int64_t total = A->num_split * A->V * (int64_t)(vec4 ? K / 4 : K);
      const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
      zero_split_kernel<<<blocks, 256, 0, stream>>>(A->d_split, A->num_split, A->V, A->n_rows,
                                                     K, C, ldc, fan.mc, vec4);
      PSPMM_CUDA_TRY(cudaGetLastError());
    }
  }
  return PSPMM_OK;
}

// The engine over units [u0, u1).
pspmm_status launch_range(const pspmm_pcsr_s *A, const Plan &plan, const float *d_B,
                          int64_t ldb, int32_t K, float *d_C, int64_t ldc,
                          const pspmm_config &cfg, cudaStream_t stream, int64_t u0, int64_t u1,
                          int32_t accumulate, const Fanout &fan, bool pdl = false) {
  if (A->nnz_v == 0 || u1 <= u0) return PSPMM_OK;
  if (cfg.mode == 2)
    return run_spmm_tma(A, d_B, ldb, K, d_C, ldc, cfg, stream, u0, u1, accumulate, fan);
  if (cfg.mode == 3)
    return run_spmm_short(A, d_B, ldb, K, d_C, ldc, cfg, stream, u0, u1, accumulate, fan);
  SpmmArgs args;
  args.rowptr = A->d_rowptr;
  args.colidx = A->d_colidx;
  args.val = A->d_val;
  args.trow = A->d_trow;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.unit_begin = (int32_t)u0;
  args.units = (int32_t)u1;
  args.units_total = (int32_t)A->num_chunks;
  args.K = K;
  args.accumulate = accumulate;
  args.fan = fan;
  // the length-sorted unit order applies to whole-matrix launches only (the
  // host entry's slices are contiguous unit ranges)
  args.order = (cfg.order && u0 == 0 && u1 == A->num_chunks) ? A->d_order : nullptr;
  const int64_t groups_per_block = plan.threads / plan.G;
  // groups loop over units (grid-stride): cap the grid at PSPMM_WAVES waves of
  // resident blocks so each group pipelines several units
  int64_t bx = (u1 - u0 + groups_per_block - 1) / groups_per_block;
  const int64_t resident =
      std::min<int64_t>(32, (PSPMM_MAX_THREADS * PSPMM_MIN_BLOCKS) / plan.threads);
  if (PSPMM_WAVES > 0) bx = std::min<int64_t>(bx, (int64_t)num_sms() * resident * PSPMM_WAVES);
  if (bx > 0x7fffffff) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run: grid too large");
  if (pdl && A->S == 1) {  // overlap this launch with the zeroing kernel before it
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)bx, (unsigned)plan.by);
    lc.blockDim = dim3(plan.threads);
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    PSPMM_CUDA_TRY(cudaLaunchKernelEx(&lc, plan.fn, args));
    return PSPMM_OK;
  }
  plan.fn<<<dim3((unsigned)bx, (unsigned)plan.by), plan.threads, 0, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace

pspmm_status run_spmm(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K, float *d_C,
                      int64_t ldc, const pspmm_config &cfg, cudaStream_t stream,
                      int32_t accumulate, const Fanout *fan) {
  Fanout f{};
  if (fan) {
    if (fan->n < 0 || fan->n > kMaxPeers)
      PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run_fanout: npeers must be in 0..PSPMM_MAX_PEERS");
    if (fan->n > 0 && accumulate)
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run_fanout: no accumulate with peer copies");
    for (int d = 0; d < fan->n; ++d) {
      if (!fan->peer[d]) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run_fanout: null peer pointer");
      // peer copies take the same vector width as C
      if ((reinterpret_cast<uintptr_t>(fan->peer[d]) & 15) !=
          (reinterpret_cast<uintptr_t>(d_C) & 15))
        PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run_fanout: peer alignment differs from C's");
    }
    if (fan->mc && fan->n != 1)
      PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run_multicast: exactly one multicast address");
    if (fan->mc && cfg.mode == 2)
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
                 "spmm_run_multicast: engine modes 0, 3, 5 and 6 take the multicast epilogue");
    f = *fan;
  }
  if (cfg.mode == 1) {  // dense tiles on the tensor cores + the rest (spmm_dense.cu)
    if (f.n > 0) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "spmm_run_fanout: no peer copies in mode 1");
    if (A && (cfg.V != A->V || cfg.S != A->S || cfg.omega != A->omega))
      PSPMM_FAIL(PSPMM_ERR_CONFIG_MISMATCH, "spmm_run: cfg.V/S/omega differ from the PCSR handle");
    return run_spmm_dense(A, d_B, ldb, K, d_C, ldc, cfg, stream, accumulate);
  }
  if (cfg.mode == 5 || cfg.mode == 6) {  // row blocks / staged bands (spmm_block.cu, spmm_band.cu)
    if (!A || !d_B || !d_C) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run: null handle or pointer");
    if (K < 1 || ldb < K || ldc < K)
      PSPMM_FAIL(PSPMM_ERR_DIM_MISMATCH, "spmm_run: need K >= 1, ldb >= K, ldc >= K");
    if (cfg.V != A->V || cfg.S != A->S || cfg.omega != A->omega)
      PSPMM_FAIL(PSPMM_ERR_CONFIG_MISMATCH, "spmm_run: cfg.V/S/omega differ from the PCSR handle");
    if (cfg.mode == 6) return run_spmm_band(A, d_B, ldb, K, d_C, ldc, stream, accumulate, f);
    return run_spmm_block(A, d_B, ldb, K, d_C, ldc, stream, accumulate, f);
  }
  Plan plan;
  pspmm_status st = make_plan(A, d_B, ldb, K, d_C, ldc, cfg, &plan);
  if (st != PSPMM_OK) return st;
  if (!accumulate) {  // C = A.B: zero what the atomics accumulate into (c-12)
    st = prepare_c(A, K, d_C, ldc, stream, f);
    if (st != PSPMM_OK) return st;
  }
  const bool zeroed = !accumulate && A->S == 1 && A->num_split > 0 && A->nnz_v > 0 &&
                      cfg.mode == 0;
  return launch_range(A, plan, d_B, ldb, K, d_C, ldc, cfg, stream, 0, A->num_chunks, accumulate,
                      f, zeroed);
}

namespace {

// Slicing the engine into kSlices unit ranges overlaps the D2H copy with the
// compute, but each slice lasts at least as long as its longest unit (one
// row group works through it).  When the longest unit holds more vectors
// than a slice's fair share per resident row group, slices would serialise
// on their hub rows: run the engine whole (with its unit order) instead.
bool slices_balanced(const pspmm_pcsr_s *A, const Plan &plan) {
  const int64_t groups = (int64_t)num_sms() * (PSPMM_MAX_THREADS * PSPMM_MIN_BLOCKS / 32) *
                         (32 / std::max(1, plan.G));
  return A->max_unit_len * kSlices * groups <= A->nnz_v;
}

}  // namespace

pspmm_status run_spmm_host(pspmm_pcsr_s *A, const float *h_B, int64_t ldb, int32_t K, float *h_C,
                           int64_t ldc, const pspmm_config &cfg, float *d_Bbuf, float *d_Cbuf,
                           cudaStream_t stream) {
  if (!A || !h_B || !h_C)
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "spmm_run_host: null handle or host pointer");
  if (cfg.mode == 1 || cfg.mode == 5 || cfg.mode == 6) {  // one whole-matrix product, no slices
    PSPMM_CUDA_TRY(cudaMemcpyAsync(d_Bbuf, h_B, (size_t)A->n_cols * ldb * sizeof(float),
                                   cudaMemcpyHostToDevice, stream));
    pspmm_status st = run_spmm(A, d_Bbuf, ldb, K, d_Cbuf, ldc, cfg, stream);
    if (st != PSPMM_OK) return st;
    PSPMM_CUDA_TRY(cudaMemcpyAsync(h_C, d_Cbuf, (size_t)A->n_rows * ldc * sizeof(float),
                                   cudaMemcpyDeviceToHost, stream));
    PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
    return PSPMM_OK;
  }
  Plan plan;
  pspmm_status st = make_plan(A, d_Bbuf, ldb, K, d_Cbuf, ldc, cfg, &plan);
  if (st != PSPMM_OK) return st;
  const Fanout none{};
  if (cfg.mode == 0 && !slices_balanced(A, plan)) {
    PSPMM_CUDA_TRY(cudaMemcpyAsync(d_Bbuf, h_B, (size_t)A->n_cols * ldb * sizeof(float),
                                   cudaMemcpyHostToDevice, stream));
    st = prepare_c(A, K, d_Cbuf, ldc, stream, none);
    if (st != PSPMM_OK) return st;
    st = launch_range(A, plan, d_Bbuf, ldb, K, d_Cbuf, ldc, cfg, stream, 0, A->num_chunks, 0,
                      none);
    if (st != PSPMM_OK) return st;
    PSPMM_CUDA_TRY(cudaMemcpyAsync(h_C, d_Cbuf, (size_t)A->n_rows * ldc * sizeof(float),
                                   cudaMemcpyDeviceToHost, stream));
    PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
    return PSPMM_OK;
  }
  if (!A->copy_stream) {
    PSPMM_CUDA_TRY(cudaStreamCreateWithFlags(&A->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < kSlices; ++k)
      PSPMM_CUDA_TRY(cudaEventCreateWithFlags(&A->slice_done[k], cudaEventDisableTiming));
  }
  PSPMM_CUDA_TRY(cudaMemcpyAsync(d_Bbuf, h_B, (size_t)A->n_cols * ldb * sizeof(float),
                                 cudaMemcpyHostToDevice, stream));
  st = prepare_c(A, K, d_Cbuf, ldc, stream, none);
  if (st != PSPMM_OK) return st;
  for (int k = 0; k < kSlices; ++k) {
    st = launch_range(A, plan, d_Bbuf, ldb, K, d_Cbuf, ldc, cfg, stream, A->slice_units[k],
                      A->slice_units[k + 1], 0, none);
    if (st != PSPMM_OK) return st;
    PSPMM_CUDA_TRY(cudaEventRecord(A->slice_done[k], stream));
    PSPMM_CUDA_TRY(cudaStreamWaitEvent(A->copy_stream, A->slice_done[k], 0));
    const int64_t r0 = A->slice_rows[k], r1 = A->slice_rows[k + 1];
    if (r1 > r0)
      PSPMM_CUDA_TRY(cudaMemcpyAsync(h_C + r0 * ldc, d_Cbuf + r0 * ldc,
                                     (size_t)(r1 - r0) * ldc * sizeof(float),
                                     cudaMemcpyDeviceToHost, A->copy_stream));
  }
  // the caller's stream observes the copies' completion, then the host waits
  PSPMM_CUDA_TRY(cudaEventRecord(A->slice_done[0], A->copy_stream));
  PSPMM_CUDA_TRY(cudaStreamWaitEvent(stream, A->slice_done[0], 0));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  return PSPMM_OK;
}

pspmm_status run_spmm_host_batch(pspmm_pcsr_s *A, const float *const *h_B, int64_t ldb, int32_t K,
                                 float *const *h_C, int64_t ldc, int32_t count,
                                 const pspmm_config &cfg, float *const *d_B, float *const *d_C,
                                 cudaStream_t stream) {
  Plan plan[2];
  for (int b = 0; b < 2 && cfg.mode != 1 && cfg.mode != 5 && cfg.mode != 6; ++b) {
    pspmm_status st = make_plan(A, d_B[b], ldb, K, d_C[b], ldc, cfg, &plan[b]);
    if (st != PSPMM_OK) return st;
  }
  if (!A->h2d_stream) {
    PSPMM_CUDA_TRY(cudaStreamCreateWithFlags(&A->h2d_stream, cudaStreamNonBlocking));
    PSPMM_CUDA_TRY(cudaStreamCreateWithFlags(&A->d2h_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      PSPMM_CUDA_TRY(cudaEventCreateWithFlags(&A->h2d_done[b], cudaEventDisableTiming));
      PSPMM_CUDA_TRY(cudaEventCreateWithFlags(&A->comp_done[b], cudaEventDisableTiming));
      PSPMM_CUDA_TRY(cudaEventCreateWithFlags(&A->d2h_done[b], cudaEventDisableTiming));
    }
    PSPMM_CUDA_TRY(cudaEventCreateWithFlags(&A->batch_start, cudaEventDisableTiming));
  }
  // the copy streams start after the work already queued on `stream`
  PSPMM_CUDA_TRY(cudaEventRecord(A->batch_start, stream));
  PSPMM_CUDA_TRY(cudaStreamWaitEvent(A->h2d_stream, A->batch_start, 0));
  PSPMM_CUDA_TRY(cudaStreamWaitEvent(A->d2h_stream, A->batch_start, 0));
  const Fanout none{};
  const size_t b_bytes = (size_t)A->n_cols * ldb * sizeof(float);
  const size_t c_bytes = (size_t)A->n_rows * ldc * sizeof(float);
  for (int32_t i = 0; i < count; ++i) {
    const int b = i & 1;
    // buffer set b is free once product i - 2 has been computed / copied out
    if (i >= 2) PSPMM_CUDA_TRY(cudaStreamWaitEvent(A->h2d_stream, A->comp_done[b], 0));
    PSPMM_CUDA_TRY(cudaMemcpyAsync(d_B[b], h_B[i], b_bytes, cudaMemcpyHostToDevice,
                                   A->h2d_stream));
    PSPMM_CUDA_TRY(cudaEventRecord(A->h2d_done[b], A->h2d_stream));
    PSPMM_CUDA_TRY(cudaStreamWaitEvent(stream, A->h2d_done[b], 0));
    if (i >= 2) PSPMM_CUDA_TRY(cudaStreamWaitEvent(stream, A->d2h_done[b], 0));
    pspmm_status st;
    if (cfg.mode == 1 || cfg.mode == 5 || cfg.mode == 6) {  // whole-matrix modes
      st = run_spmm(A, d_B[b], ldb, K, d_C[b], ldc, cfg, stream);
    } else {
      st = prepare_c(A, K, d_C[b], ldc, stream, none);
      if (st != PSPMM_OK) return st;
      st = launch_range(A, plan[b], d_B[b], ldb, K, d_C[b], ldc, cfg, stream, 0, A->num_chunks, 0,
                        none);
    }
    if (st != PSPMM_OK) return st;
    PSPMM_CUDA_TRY(cudaEventRecord(A->comp_done[b], stream));
    PSPMM_CUDA_TRY(cudaStreamWaitEvent(A->d2h_stream, A->comp_done[b], 0));
    PSPMM_CUDA_TRY(cudaMemcpyAsync(h_C[i], d_C[b], c_bytes, cudaMemcpyDeviceToHost,
                                   A->d2h_stream));
    PSPMM_CUDA_TRY(cudaEventRecord(A->d2h_done[b], A->d2h_stream));
  }
  for (int b = 0; b < 2 && b < count; ++b)
    PSPMM_CUDA_TRY(cudaStreamWaitEvent(stream, A->d2h_done[b], 0));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  return PSPMM_OK;
}

}  // namespace pspmm
