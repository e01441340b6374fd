// (a4, a5) PCSR generation on the device (PAPER.md P:208 data representation,
// P:211 generation, Eq. 3).  Count -> exclusive scan -> fill, so
// every output position is a pure function of the input and the integer
// arrays are bit-identical to the oracle's (no atomics decide an order).
//
//   V = 1: panels are rows; rowPtr/colIdx/val are copies of the CSR.
//   V = 2: panel p = rows {2p, 2p+1}.  The panel's vectors are the ascending
//          union of the two rows' columns.  With a = row 2p, b = row 2p+1:
//            pos(x in a)       = i_a(x) + U_b(x)
//            pos(y in b \ a)   = i_a(y) + U_b(y)
//          where i_a(x) = #a-columns < x and U_b(x) = #b-only columns < x
//          (a prefix count of the "not in a" flags of b, one warp ballot per
//          32 columns).  val[2 pos + k] = A[2p+k, col] or +0.0f (c-7).
//   S = 1: SG = ceil(nnz_V / (P^ omega)) omega (c-3a) or sg_override;
//          panel p with L vectors -> max(1, ceil(L/SG)) chunks (c-5) at
//          offsets 0, SG, 2SG ...; TRow[c] = p.
#include <algorithm>

#include <cub/cub.cuh>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ int lower_bound_dev(const int32_t *__restrict__ a, int len, int x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

int grid_for(int64_t items, int per_block) {
  int64_t b = (items + per_block - 1) / per_block;
  int64_t cap = (int64_t)num_sms() * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// L[p] = vectors of panel p (V = 1: the row degree).  L[P] = 0 (scan sentinel).
__global__ void counts_v1_kernel(int64_t n_rows, const int32_t *__restrict__ rowptr,
                                 int64_t *__restrict__ L) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_rows;
       i += (int64_t)gridDim.x * blockDim.x)
    L[i] = i < n_rows ? (int64_t)(rowptr[i + 1] - rowptr[i]) : 0;
}

// V = 2 counts: |a u b| = |a| + #(b not in a).  One warp per panel.
template <typename OutT>
__global__ void __launch_bounds__(kBlock) counts_v2_kernel(int64_t n_rows, int64_t P,
                                                           const int32_t *__restrict__ rowptr,
                                                           const int32_t *__restrict__ colidx,
                                                           OutT *__restrict__ L) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p <= P; p += warps) {
    if (p == P) {
      if (lane == 0) L[P] = 0;
      continue;
    }
    const int64_t ra = 2 * p, rb = 2 * p + 1;
    const int a0 = rowptr[ra], a1 = rowptr[ra + 1];
    const int b0 = rb < n_rows ? rowptr[rb] : 0, b1 = rb < n_rows ? rowptr[rb + 1] : 0;
    const int la = a1 - a0;
    int only_b = 0;
    for (int j = b0 + lane; j < b1; j += 32) {
      const int y = colidx[j];
      const int i = lower_bound_dev(colidx + a0, la, y);
      only_b += (i < la && colidx[a0 + i] == y) ? 0 : 1;
    }
    only_b = __reduce_add_sync(0xffffffffu, only_b);
    if (lane == 0) L[p] = (OutT)(la + only_b);
  }
}

// V = 2 fill.  bpre[j] (j indexes colidx of the b rows) = #b-only columns
// before position j within its row.
__global__ void __launch_bounds__(kBlock) fill_v2_kernel(int64_t n_rows, int64_t P,
                                                         const int32_t *__restrict__ rowptr,
                                                         const int32_t *__restrict__ colidx,
                                                         const float *__restrict__ val,
                                                         const int64_t *__restrict__ panelptr,
                                                         int32_t *__restrict__ bpre,
                                                         int32_t *__restrict__ out_col,
                                                         float *__restrict__ out_val) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += warps) {
    const int64_t ra = 2 * p, rb = 2 * p + 1;
    const int a0 = rowptr[ra], a1 = rowptr[ra + 1];
    const int b0 = rb < n_rows ? rowptr[rb] : 0, b1 = rb < n_rows ? rowptr[rb + 1] : 0;
    const int la = a1 - a0, lb = b1 - b0;
    const int64_t base = panelptr[p];
    // pass 1: b-only flags -> exclusive prefix (bpre), b-only vectors written
    int running = 0;
    for (int t = 0; t < lb; t += 32) {
      const int j = t + lane;
      int flag = 0, ia = 0, y = 0;
      if (j < lb) {
        y = colidx[b0 + j];
        ia = lower_bound_dev(colidx + a0, la, y);
        flag = (ia < la && colidx[a0 + ia] == y) ? 0 : 1;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, flag);
      const int before = running + __popc(bal & ((1u << lane) - 1u));
      if (j < lb) {
        bpre[b0 + j] = before;
        if (flag) {
          const int64_t pos = base + ia + before;
          out_col[pos] = y;
          out_val[2 * pos] = 0.0f;
          out_val[2 * pos + 1] = val[b0 + j];
        }
      }
      running += __popc(bal);
    }
    __syncwarp();
    // pass 2: every a column, paired with b's value when b has it
    for (int i = lane; i < la; i += 32) {
      const int x = colidx[a0 + i];
      const int jb = lower_bound_dev(colidx + b0, lb, x);
      const bool both = jb < lb && colidx[b0 + jb] == x;
      const int ub = jb < lb ? bpre[b0 + jb] : running;
      const int64_t pos = base + i + ub;
      out_col[pos] = x;
      out_val[2 * pos] = val[a0 + i];
      out_val[2 * pos + 1] = both ? val[b0 + jb] : 0.0f;
    }
  }
}

__global__ void nonempty_kernel(int64_t P, const int64_t *__restrict__ L,
                                unsigned long long *__restrict__ count) {
  unsigned long long c = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    c += L[p] > 0 ? 1ull : 0ull;
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// nch[p] = max(1, ceil(L/SG)); split flag = nch > 1.  nch[P] = split[P] = 0.
__global__ void chunk_counts_kernel(int64_t P, int64_t SG, const int64_t *__restrict__ L,
                                    int64_t *__restrict__ nch, int64_t *__restrict__ split) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= P;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (p == P) {
      nch[P] = 0;
      split[P] = 0;
      continue;
    }
    const int64_t l = L[p];
    const int64_t c = l == 0 ? 1 : (l + SG - 1) / SG;
    nch[p] = c;
    split[p] = c > 1 ? 1 : 0;
  }
}

__global__ void chunk_fill_kernel(int64_t P, int64_t SG, int64_t nnz_v,
                                  const int64_t *__restrict__ panelptr,
                                  const int64_t *__restrict__ choff,
                                  const int64_t *__restrict__ splitoff,
                                  int32_t *__restrict__ rowptr, int32_t *__restrict__ trow,
                                  int32_t *__restrict__ split_ids) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t start = panelptr[p], L = panelptr[p + 1] - start;
    const int64_t c0 = choff[p], nc = choff[p + 1] - c0;
    for (int64_t j = 0; j < nc; ++j) {
      rowptr[c0 + j] = (int32_t)(start + j * SG);
      trow[c0 + j] = (int32_t)p;
    }
    if (nc > 1) split_ids[splitoff[p]] = (int32_t)p;
    (void)L;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t total = choff[P];
    rowptr[total] = (int32_t)nnz_v;
  }
}

__global__ void narrow_kernel(int64_t count, const int64_t *__restrict__ in,
                              int32_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

// Exclusive scan of `count` int64 values (CUB); temp storage from the stream pool.
pspmm_status exclusive_scan(const int64_t *d_in, int64_t *d_out, int64_t count,
                            cudaStream_t stream) {
  size_t bytes = 0;
  PSPMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, bytes, d_in, d_out, (int)count, stream));
  void *tmp = nullptr;
  PSPMM_CUDA_TRY(cudaMallocAsync(&tmp, bytes > 0 ? bytes : 16, stream));
  PSPMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, bytes, d_in, d_out, (int)count, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(tmp, stream));
  return PSPMM_OK;
}

__global__ void unit_len_kernel(int64_t units, const int32_t *__restrict__ rowptr,
                                int32_t *__restrict__ len, int32_t *__restrict__ ids) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units;
       u += (int64_t)gridDim.x * blockDim.x) {
    len[u] = rowptr[u + 1] - rowptr[u];
    ids[u] = (int32_t)u;
  }
}

}  // namespace

// Engine schedule (not part of the PCSR contract): unit ids by descending
// vector count, ties in ascending id (stable radix sort -> deterministic).
pspmm_status build_unit_order(pspmm_pcsr_s *A, cudaStream_t stream) {
  const int64_t units = A->num_chunks;
  if (units < 1) return PSPMM_OK;
  int32_t *len = nullptr, *len_sorted = nullptr, *ids = nullptr;
  void *tmp = nullptr;
  size_t bytes = 0;
  PSPMM_CUDA_TRY(cudaMalloc(&A->d_order, (size_t)units * sizeof(int32_t)));
  PSPMM_CUDA_TRY(cudaMallocAsync(&len, (size_t)units * sizeof(int32_t), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&len_sorted, (size_t)units * sizeof(int32_t), stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&ids, (size_t)units * sizeof(int32_t), stream));
  unit_len_kernel<<<grid_for(units, kBlock), kBlock, 0, stream>>>(units, A->d_rowptr, len, ids);
  PSPMM_CUDA_TRY(cudaGetLastError());
  PSPMM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, len, len_sorted, ids,
                                                           A->d_order, (int)units, 0, 32, stream));
  PSPMM_CUDA_TRY(cudaMallocAsync(&tmp, bytes > 0 ? bytes : 16, stream));
  PSPMM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(tmp, bytes, len, len_sorted, ids,
                                                           A->d_order, (int)units, 0, 32, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(tmp, stream));
  // the longest unit's vector count (its id leads the order)
  int32_t lmax = 0;
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&lmax, len_sorted, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  A->max_unit_len = lmax;
  PSPMM_CUDA_TRY(cudaFreeAsync(len, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(len_sorted, stream));
  PSPMM_CUDA_TRY(cudaFreeAsync(ids, stream));
  return PSPMM_OK;
}

namespace {

struct Scratch {
  cudaStream_t s;
  void *ptrs[8] = {};
  int n = 0;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <typename T>
  cudaError_t get(T **p, size_t count) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(p), count * sizeof(T) + 16, s);
    if (e == cudaSuccess) ptrs[n++] = *p;
    return e;
  }
  ~Scratch() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], s);
  }
};

}  // namespace

pspmm_status panel_counts_v2(int64_t n_rows, const int32_t *d_rowptr, const int32_t *d_colidx,
                             int32_t *d_L, cudaStream_t stream) {
  const int64_t P = (n_rows + 1) / 2;
  counts_v2_kernel<int32_t><<<grid_for((P + 1) * 32, kBlock), kBlock, 0, stream>>>(
      n_rows, P, d_rowptr, d_colidx, d_L);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

pspmm_status build_pcsr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t *d_rowptr,
                        const int32_t *d_colidx, const float *d_val, int32_t V, int32_t S,
                        int32_t omega, int32_t sg_override, cudaStream_t stream,
                        pspmm_pcsr_s *A) {
  if (V != 1 && V != 2) PSPMM_FAIL(PSPMM_ERR_CONFIG, "pcsr_build: V must be 1 or 2 (P:91)");
  if (S != 0 && S != 1) PSPMM_FAIL(PSPMM_ERR_CONFIG, "pcsr_build: S must be 0 or 1");
  if (omega < 1 || sg_override < 0) PSPMM_FAIL(PSPMM_ERR_CONFIG, "pcsr_build: bad omega / SG");
  if (nnz > 0 && !d_val) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_build: null val");
  pspmm_status st = validate_csr(n_rows, n_cols, nnz, d_rowptr, d_colidx, stream);
  if (st != PSPMM_OK) return st;

  A->n_rows = n_rows;
  A->n_cols = n_cols;
  A->nnz = nnz;
  A->V = V;
  A->S = S;
  A->omega = omega;
  const int64_t P = (n_rows + V - 1) / V;
  A->num_panels = P;

  Scratch scr(stream);
  int64_t *L = nullptr, *panelptr = nullptr;
  unsigned long long *d_cnt = nullptr;
  PSPMM_CUDA_TRY(scr.get(&L, P + 1));
  PSPMM_CUDA_TRY(scr.get(&panelptr, P + 1));
  PSPMM_CUDA_TRY(scr.get(&d_cnt, 2));
  PSPMM_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned long long), stream));

  // step 1-2 counts, step 3 scan
  if (V == 1)
    counts_v1_kernel<<<grid_for(P + 1, kBlock), kBlock, 0, stream>>>(n_rows, d_rowptr, L);
  else
    counts_v2_kernel<int64_t><<<grid_for((P + 1) * 32, kBlock), kBlock, 0, stream>>>(
        n_rows, P, d_rowptr, d_colidx, L);
  PSPMM_CUDA_TRY(cudaGetLastError());
  st = exclusive_scan(L, panelptr, P + 1, stream);
  if (st != PSPMM_OK) return st;
  nonempty_kernel<<<grid_for(P, kBlock), kBlock, 0, stream>>>(P, L, d_cnt);
  PSPMM_CUDA_TRY(cudaGetLastError());
  int64_t nnz_v = 0;
  unsigned long long h_cnt[2] = {0, 0};
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&nnz_v, panelptr + P, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 stream));
  PSPMM_CUDA_TRY(cudaMemcpyAsync(h_cnt, d_cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  if (nnz_v >= INT32_MAX) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "pcsr_build: nnz_V >= 2^31");
  const int64_t nonempty = (int64_t)h_cnt[0];
  A->nnz_v = nnz_v;
  A->pr = nnz_v > 0 ? 1.0 - (double)nnz / ((double)nnz_v * (double)V) : __builtin_nan("");

  // step 2 fill (colIdx, val)
  if (nnz_v > 0) {
    PSPMM_CUDA_TRY(cudaMalloc(&A->d_colidx, (size_t)nnz_v * sizeof(int32_t)));
    PSPMM_CUDA_TRY(cudaMalloc(&A->d_val, (size_t)nnz_v * V * sizeof(float)));
    if (V == 1) {
      PSPMM_CUDA_TRY(cudaMemcpyAsync(A->d_colidx, d_colidx, (size_t)nnz * sizeof(int32_t),
                                     cudaMemcpyDeviceToDevice, stream));
      PSPMM_CUDA_TRY(cudaMemcpyAsync(A->d_val, d_val, (size_t)nnz * sizeof(float),
                                     cudaMemcpyDeviceToDevice, stream));
    } else {
      int32_t *bpre = nullptr;
      PSPMM_CUDA_TRY(scr.get(&bpre, nnz > 0 ? nnz : 1));
      fill_v2_kernel<<<grid_for(P * 32, kBlock), kBlock, 0, stream>>>(
          n_rows, P, d_rowptr, d_colidx, d_val, panelptr, bpre, A->d_colidx, A->d_val);
      PSPMM_CUDA_TRY(cudaGetLastError());
    }
  }

  if (S == 0) {
    // step 4
    A->rowptr_len = P + 1;
    A->num_chunks = P;
    A->sg = 0;
    A->sr = 1.0;
    PSPMM_CUDA_TRY(cudaMalloc(&A->d_rowptr, (size_t)(P + 1) * sizeof(int32_t)));
    narrow_kernel<<<grid_for(P + 1, kBlock), kBlock, 0, stream>>>(P + 1, panelptr, A->d_rowptr);
    PSPMM_CUDA_TRY(cudaGetLastError());
    st = build_unit_order(A, stream);
    if (st != PSPMM_OK) return st;
    PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
    for (int k = 0; k <= kSlices; ++k) {
      const int64_t p = P * k / kSlices;
      A->slice_units[k] = p;
      A->slice_rows[k] = std::min<int64_t>(p * V, n_rows);
    }
    return PSPMM_OK;
  }

  // step 5: Eq. 3
  int64_t SG;
  if (sg_override > 0) {
    SG = sg_override;
  } else {
    if (nonempty == 0) PSPMM_FAIL(PSPMM_ERR_EMPTY, "pcsr_build: SG undefined, all panels empty");
    const int64_t denom = nonempty * (int64_t)omega;
    SG = ((nnz_v + denom - 1) / denom) * omega;
  }
  A->sg = SG;
  int64_t *nch = nullptr, *choff = nullptr, *split = nullptr, *splitoff = nullptr;
  PSPMM_CUDA_TRY(scr.get(&nch, P + 1));
  PSPMM_CUDA_TRY(scr.get(&choff, P + 1));
  PSPMM_CUDA_TRY(scr.get(&split, P + 1));
  PSPMM_CUDA_TRY(scr.get(&splitoff, P + 1));
  chunk_counts_kernel<<<grid_for(P + 1, kBlock), kBlock, 0, stream>>>(P, SG, L, nch, split);
  PSPMM_CUDA_TRY(cudaGetLastError());
  st = exclusive_scan(nch, choff, P + 1, stream);
  if (st != PSPMM_OK) return st;
  st = exclusive_scan(split, splitoff, P + 1, stream);
  if (st != PSPMM_OK) return st;
  int64_t totals[2] = {0, 0};
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&totals[0], choff + P, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 stream));
  PSPMM_CUDA_TRY(cudaMemcpyAsync(&totals[1], splitoff + P, sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, stream));
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t chunks = totals[0];
  if (chunks >= INT32_MAX) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "pcsr_build: chunks >= 2^31");
  A->num_chunks = chunks;
  A->rowptr_len = chunks + 1;
  A->num_split = totals[1];
  A->sr = (double)(chunks + 1) / (double)(P + 1);
  PSPMM_CUDA_TRY(cudaMalloc(&A->d_rowptr, (size_t)(chunks + 1) * sizeof(int32_t)));
  PSPMM_CUDA_TRY(cudaMalloc(&A->d_trow, (size_t)chunks * sizeof(int32_t)));
  PSPMM_CUDA_TRY(cudaMalloc(&A->d_split, (size_t)(A->num_split > 0 ? A->num_split : 1) *
                                             sizeof(int32_t)));
  chunk_fill_kernel<<<grid_for(P, kBlock), kBlock, 0, stream>>>(
      P, SG, nnz_v, panelptr, choff, splitoff, A->d_rowptr, A->d_trow, A->d_split);
  PSPMM_CUDA_TRY(cudaGetLastError());
  st = build_unit_order(A, stream);
  if (st != PSPMM_OK) return st;
  // slice bounds at panel boundaries: unit = first chunk of the panel
  for (int k = 0; k <= kSlices; ++k) {
    const int64_t p = P * k / kSlices;
    PSPMM_CUDA_TRY(cudaMemcpyAsync(&A->slice_units[k], choff + p, sizeof(int64_t),
                                   cudaMemcpyDeviceToHost, stream));
    A->slice_rows[k] = std::min<int64_t>(p * V, n_rows);
  }
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  return PSPMM_OK;
}

}  // namespace pspmm
