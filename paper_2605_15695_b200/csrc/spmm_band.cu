// (a6, a7) Engine mode 6: staged-band engine for locality-ordered graphs.
//
// The paper's locality step (§4.4: reordering so that "rows with
// similar column sets are close") leaves each block of consecutive rows
// touching a few contiguous column ranges (a road lattice: the rows
// themselves and the rows one lattice width above and below).  The mode-0 /
// mode-3 engines gather every B row with a dependent rowPtr -> colIdx ->
// B-row chain per row, which keeps them latency-bound on such graphs
// (roadNet: 58 % of the HBM roofline, long-scoreboard stalls).  Here every
// byte a block needs moves by bulk copy, issued from one descriptor:
//
//  - pack (pspmm_pcsr_attach_band, once per graph): rows in blocks of R =
//    128 / 64 / 32 / 16 rows (k_max <= 16 / 32 / 64 / 128, so the band of a lattice
//    block fits the budget at any K); per block a descriptor {first range,
//    ranges, first nonzero, end nonzero} and its staged-row count; per range
//    {first B row, rows, slot in the band}, where a range is a run of the
//    block's sorted distinct columns with gaps of at most kGap rows; per
//    nonzero the pair (slot in the band, value bits), 8 B, in CSR order; a
//    padded copy of rowPtr.  A block whose band exceeds kBandBytes keeps the
//    global column in its pairs and gathers B from L2 / HBM;
//  - kernel (persistent, 3 CTAs per SM, two stages each): a producer warp
//    reads a block's descriptor, arms the stage's mbarrier with the total
//    byte count and issues every copy at once, one range per lane
//    (cp.async.bulk: the band's ranges, the block's pair run, its rowPtr
//    slice), so the next block's data is in flight while four compute warps
//    finish the current one; after the mbarrier completes, every row group
//    (G lanes = K / 4 columns, one float4 each) walks its rows' pairs in
//    shared memory: a
//    broadcast LDS.64 of (slot, value) and one LDS.128 of the staged B row
//    per nonzero (Alg. 2 l.9-15); one streaming 128-bit store per lane and
//    row (l.17-23, one writer per element).
//
// The pack is derived data, not part of the bit-exact PCSR contract.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr int kThreads = 128;
constexpr int kGap = 8;              // merge column ranges separated by <= kGap rows
constexpr int kPairCap = 512;        // pairs staged per block (4 KB); more: read from global

constexpr int kMaxRows = 128;  // rows per block at most (the stage's rowPtr slice)
int block_rows(int k_max) {
  return k_max <= 16 ? 128 : k_max <= 32 ? 64 : k_max <= 64 ? 32 : 16;
}

struct BandArgs {
  const int4 *__restrict__ desc;        // blocks: {first range, ranges, p0, p1}
  const int32_t *__restrict__ staged;   // blocks: staged band rows (-1: over budget)
  const int4 *__restrict__ rng;         // ranges: {first B row, rows, band slot, 0}
  const int2 *__restrict__ pairs;       // nnz (+2 pad): (slot or column, value bits)
  const int32_t *__restrict__ rowptr;   // padded copy (n + 1 + kMaxRows)
  const float *__restrict__ B;
  float *__restrict__ C;
  int64_t ldb, ldc;
  int32_t n_rows, K, R, accumulate;
  int64_t nblk;
  int32_t stages;  // stage ring depth (2 by default: 3 CTAs per SM)
  Fanout fan;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk(uint32_t dst, const void *src, uint32_t bytes,
                                     uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void fma4(float4 &acc, float v, const float4 &b) {
  acc.x = fmaf(v, b.x, acc.x);
  acc.y = fmaf(v, b.y, acc.y);
  acc.z = fmaf(v, b.z, acc.z);
  acc.w = fmaf(v, b.w, acc.w);
}

// G lanes per row (K <= 4 G).  Persistent CTAs: warp 4 is the producer —
// per block (b = blockIdx.x, + gridDim.x, ...) it reads the descriptor,
// writes the block's info into the stage, arms the stage's mbarrier with the
// byte count and issues every copy (one range per lane); warps 0-3 (128
// threads = 128 / G row groups) compute the block of the other stage.  Two
// stages, so the next block's copies are in flight while this one computes.
constexpr int kMaxStages = 4;
constexpr int kRPG = 4;  // rows per row group in one block (R = kRPG x 128 / G at K = 4 G)
constexpr int kStageBytes = kBandBytes + kPairCap * 8 + kMaxRows * 4 + 32;  // + info

template <int G>
__global__ void __launch_bounds__(kThreads + 32, 3) spmm_band_kernel(const BandArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int GROUPS = kThreads / G;
  const int S = a.stages;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * kStageBytes);
  uint64_t *empty = full + kMaxStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rowb = (uint32_t)a.ldb * 4u;  // staged row pitch = B's row pitch
  const int64_t nblk = a.nblk;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])),
                   "r"(kThreads));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kThreads / 32) {  // producer warp
    // the next block's descriptor, staged-row count and range entries are
    // loaded before waiting for its stage, so only the copy issue waits
    int64_t blk = blockIdx.x;
    int4 d = blk < nblk ? a.desc[blk] : make_int4(0, 0, 0, 0);
    int staged = blk < nblk ? a.staged[blk] : 0;
    int4 r = (blk < nblk && staged > 0 && lane < d.y) ? a.rng[d.x + lane] : make_int4(0, 0, 0, 0);
    for (int it = 0; blk < nblk; ++it) {
      const int s = it % S;
      const int64_t nb = blk + gridDim.x;  // prefetch the next block's metadata
      const int4 dn = nb < nblk ? a.desc[nb] : make_int4(0, 0, 0, 0);
      const int stn = nb < nblk ? a.staged[nb] : 0;
      unsigned char *st = smem + s * kStageBytes;
      int *info = reinterpret_cast<int *>(st + kBandBytes + kPairCap * 8 + kMaxRows * 4);
      const int64_t r0 = blk * a.R;
      const int rows = (int)(a.n_rows - r0 < a.R ? a.n_rows - r0 : a.R);
      const int pb = d.z & ~1, pcnt = (d.w - pb + 1) & ~1;  // 16-B aligned pair run
      const bool pairs_in = pcnt <= kPairCap;
      const int rp_cnt = (rows + 3) & ~3;
      if (it >= S) mbar_wait_parity(&empty[s], ((it / S) - 1) & 1);
      if (lane == 0) {
        info[0] = staged;
        info[1] = pairs_in ? pb : -1;
        info[2] = d.w;
        info[3] = rows;
        const uint32_t bytes = (staged > 0 ? (uint32_t)staged * rowb : 0u) +
                               (pairs_in ? (uint32_t)pcnt * 8u : 0u) + (uint32_t)rp_cnt * 4u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&full[s])),
                     "r"(bytes)
                     : "memory");
      }
      __syncwarp();
      const uint32_t bar = smem_u32(&full[s]);
      if (staged > 0) {
        if (lane < d.y)
          bulk(smem_u32(st) + (uint32_t)r.z * rowb, a.B + (int64_t)r.x * a.ldb,
               (uint32_t)r.y * rowb, bar);
        for (int i = lane + 32; i < d.y; i += 32) {  // blocks with > 32 ranges
          const int4 q = a.rng[d.x + i];
          bulk(smem_u32(st) + (uint32_t)q.z * rowb, a.B + (int64_t)q.x * a.ldb,
               (uint32_t)q.y * rowb, bar);
        }
      }
      if (lane == 0 && pairs_in && pcnt > 0)
        bulk(smem_u32(st + kBandBytes), a.pairs + pb, (uint32_t)pcnt * 8u, bar);
      if (lane == 1)
        bulk(smem_u32(st + kBandBytes + kPairCap * 8), a.rowptr + r0, (uint32_t)rp_cnt * 4u, bar);
      blk = nb;
      d = dn;
      staged = stn;
      r = (blk < nblk && staged > 0 && lane < d.y) ? a.rng[d.x + lane] : make_int4(0, 0, 0, 0);
    }
    return;
  }

  const int g = tid / G, l = tid % G;
  const bool cok = l * 4 < a.K;
  const float *gb = a.B + l * 4;
  int it = 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
    const int s = it % S;
    unsigned char *st = smem + s * kStageBytes;
    const int2 *spairs = reinterpret_cast<const int2 *>(st + kBandBytes);
    const int32_t *srp = reinterpret_cast<const int32_t *>(st + kBandBytes + kPairCap * 8);
    const int *info = reinterpret_cast<const int *>(st + kBandBytes + kPairCap * 8 + kMaxRows * 4);
    mbar_wait_parity(&full[s], (it / S) & 1);
    const int staged = info[0], pb = info[1], p_end = info[2], rows = info[3];
    const int64_t r0 = blk * a.R;
    const uint32_t sb = smem_u32(st) + l * 16;
    if (pb >= 0 && staged > 0 && rows <= GROUPS * kRPG) {
      // the fast path: the group's (up to kRPG) rows walked together, one
      // nonzero of each per step, so their LDS chains overlap
      int q0[kRPG], n[kRPG];
      float4 acc[kRPG];
      int nmax = 0;
#pragma unroll
      for (int u = 0; u < kRPG; ++u) {
        const int i = g + u * GROUPS;
        const bool ok = i < rows;
        q0[u] = ok ? srp[i] - pb : 0;
        n[u] = ok ? (i + 1 < rows ? srp[i + 1] : p_end) - pb - q0[u] : 0;
        nmax = max(nmax, n[u]);
        acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (cok) {
        for (int j = 0; j < nmax; ++j) {
#pragma unroll
          for (int u = 0; u < kRPG; ++u)
            if (j < n[u]) {
              const int2 x = spairs[q0[u] + j];
              fma4(acc[u], __int_as_float(x.y), lds4(sb + (uint32_t)x.x * rowb));
            }
        }
#pragma unroll
        for (int u = 0; u < kRPG; ++u) {
          const int i = g + u * GROUPS;
          if (i < rows) {
            const int64_t off = (r0 + i) * a.ldc + l * 4;
            float4 v = acc[u];
            if (a.accumulate) {
              const float4 o = *reinterpret_cast<const float4 *>(a.C + off);
              v.x += o.x;
              v.y += o.y;
              v.z += o.z;
              v.w += o.w;
            }
            fan_store4(a.C, a.fan, off, v);
          }
        }
      }
    } else {
    for (int i = g; i < rows; i += GROUPS) {
      if (!cok) break;
      const int q0 = srp[i], q1 = i + 1 < rows ? srp[i + 1] : p_end;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = q0; j < q1; ++j) {  // a pair run over the stage or a band over budget
        const int2 x = pb >= 0 ? spairs[j - pb] : __ldg(a.pairs + j);
        const float4 b = staged > 0
                             ? lds4(sb + (uint32_t)x.x * rowb)
                             : __ldg(reinterpret_cast<const float4 *>(gb + (int64_t)x.x * a.ldb));
        fma4(acc, __int_as_float(x.y), b);
      }
      const int64_t off = (r0 + i) * a.ldc + l * 4;
      if (a.accumulate) {
        const float4 o = *reinterpret_cast<const float4 *>(a.C + off);
        acc.x += o.x;
        acc.y += o.y;
        acc.z += o.z;
        acc.w += o.w;
      }
      fan_store4(a.C, a.fan, off, acc);
    }
    }
    // the stage is refilled by bulk copies (async proxy): order this thread's
    // generic reads before its release (WAR across proxies)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
  if (a.fan.n) __threadfence_system();
}

template <typename T>
pspmm_status upload(T **dst, const std::vector<T> &src) {
  PSPMM_CUDA_TRY(cudaMalloc(dst, std::max<size_t>(1, src.size()) * sizeof(T)));
  if (!src.empty())
    PSPMM_CUDA_TRY(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return PSPMM_OK;
}

int lanes_for(int K) {
  int G = 4;
  while (G * 4 < K) G <<= 1;
  return G;
}

template <int G>
pspmm_status launch_band(const BandArgs &args, int64_t nblk, cudaStream_t stream) {
  const int kSmem = args.stages * kStageBytes + 2 * kMaxStages * 8;
  PSPMM_CUDA_TRY(cudaFuncSetAttribute(spmm_band_kernel<G>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  int per_sm = 0;
  PSPMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmm_band_kernel<G>,
                                                               kThreads + 32, kSmem));
  const int64_t grid = std::min<int64_t>(nblk, (int64_t)num_sms() * std::max(1, per_sm));
  spmm_band_kernel<G><<<(unsigned)grid, kThreads + 32, kSmem, stream>>>(args);
  PSPMM_CUDA_TRY(cudaGetLastError());
  return PSPMM_OK;
}

}  // namespace

void destroy_band(Band *D) {
  if (!D) return;
  cudaFree(D->d_desc);
  cudaFree(D->d_staged);
  cudaFree(D->d_rng);
  cudaFree(D->d_pairs);
  cudaFree(D->d_rowptr);
  delete D;
}

// Host pack (blocks split over host threads).  Synchronises `stream`.
pspmm_status attach_band(pspmm_pcsr_s *A, int32_t k_max, cudaStream_t stream, double *staged_frac) {
  if (!A) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "attach_band: null handle");
  if (A->V != 1 || A->S != 0)
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "attach_band: needs a V = 1, S = 0 handle (CSR order)");
  if (k_max < 4 || k_max > kBandMaxK || k_max % 4 != 0)
    PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "attach_band: k_max must be a multiple of 4 in [4, 128]");
  const int64_t n = A->n_rows, nnz = A->nnz;
  if (nnz >= 0x7ffffff0ll) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "attach_band: nnz >= 2^31");
  const int R = block_rows(k_max);
  const int64_t nblk = (n + R - 1) / R;
  const int64_t max_rows = kBandBytes / ((int64_t)k_max * 4);  // staged rows per block
  PSPMM_CUDA_TRY(cudaStreamSynchronize(stream));
  std::vector<int32_t> rp(n + 1 + kMaxRows), ci(nnz);
  std::vector<float> vl(nnz);
  PSPMM_CUDA_TRY(cudaMemcpy(rp.data(), A->d_rowptr, (n + 1) * 4, cudaMemcpyDeviceToHost));
  for (int k = 0; k < kMaxRows; ++k) rp[n + 1 + k] = rp[n];
  if (nnz) {
    PSPMM_CUDA_TRY(cudaMemcpy(ci.data(), A->d_colidx, nnz * 4, cudaMemcpyDeviceToHost));
    PSPMM_CUDA_TRY(cudaMemcpy(vl.data(), A->d_val, nnz * 4, cudaMemcpyDeviceToHost));
  }
  std::vector<int2> pairs(nnz + 2, make_int2(0, 0));
  std::vector<int4> desc(nblk);
  std::vector<int32_t> staged(nblk);
  std::vector<std::vector<int4>> rng_t(nblk);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t)
    th.emplace_back([&, t] {
      std::vector<int32_t> cols;
      for (int64_t b = t; b < nblk; b += nth) {
        const int64_t q0 = rp[b * R], q1 = rp[std::min(n, (b + 1) * R)];
        cols.assign(ci.begin() + q0, ci.begin() + q1);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        std::vector<int4> &rg = rng_t[b];
        int64_t rows = 0;
        for (size_t i = 0; i < cols.size();) {
          size_t j = i;
          while (j + 1 < cols.size() && cols[j + 1] - cols[j] <= kGap + 1) ++j;
          rg.push_back(make_int4(cols[i], cols[j] - cols[i] + 1, (int)rows, 0));
          rows += cols[j] - cols[i] + 1;
          i = j + 1;
        }
        const bool fits = rows > 0 && rows <= max_rows;
        staged[b] = rows == 0 ? 0 : fits ? (int32_t)rows : -1;
        if (!fits) rg.clear();
        for (int64_t p = q0; p < q1; ++p) {
          int32_t s = ci[p];
          if (fits) {  // column -> band slot (ranges sorted by first row)
            size_t lo = 0, hi = rg.size();
            while (hi - lo > 1) {
              const size_t mid = (lo + hi) / 2;
              if (rg[mid].x <= s)
                lo = mid;
              else
                hi = mid;
            }
            s = rg[lo].z + (s - rg[lo].x);
          }
          int32_t bits;
          std::memcpy(&bits, &vl[p], 4);
          pairs[p] = make_int2(s, bits);
        }
      }
    });
  for (auto &x : th) x.join();
  std::vector<int4> rng;
  int64_t staged_blocks = 0, nonempty = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t q0 = rp[b * R], q1 = rp[std::min(n, (b + 1) * R)];
    desc[b] = make_int4((int)rng.size(), (int)rng_t[b].size(), (int)q0, (int)q1);
    rng.insert(rng.end(), rng_t[b].begin(), rng_t[b].end());
    if (staged[b] != 0) ++nonempty;
    if (staged[b] > 0) ++staged_blocks;
  }
  Band *D = new Band();
  struct Guard {
    Band *d;
    ~Guard() { destroy_band(d); }
  } guard{D};
  D->num_blocks = nblk;
  D->k_max = k_max;
  D->rows = R;
  D->staged_frac = nonempty ? (double)staged_blocks / nonempty : 1.0;
  pspmm_status st;
  if ((st = upload(&D->d_desc, desc)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_staged, staged)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_rng, rng)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_pairs, pairs)) != PSPMM_OK) return st;
  if ((st = upload(&D->d_rowptr, rp)) != PSPMM_OK) return st;
  destroy_band(A->band);
  A->band = D;
  guard.d = nullptr;
  if (staged_frac) *staged_frac = D->staged_frac;
  return PSPMM_OK;
}

bool band_supported(const pspmm_pcsr_s *A, int32_t K, int64_t ldb, int64_t ldc, const float *d_B,
                    const float *d_C) {
  return A && A->band && A->V == 1 && A->S == 0 && K % 4 == 0 && K <= A->band->k_max &&
         ldb % 4 == 0 && ldb <= A->band->k_max && ldc % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(d_B) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(d_C) & 15) == 0;
}

pspmm_status run_spmm_band(const pspmm_pcsr_s *A, const float *d_B, int64_t ldb, int32_t K,
                           float *d_C, int64_t ldc, cudaStream_t stream, int32_t accumulate,
                           const Fanout &fan) {
  if (!band_supported(A, K, ldb, ldc, d_B, d_C))
    PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED,
               "spmm_run mode 6: needs pspmm_pcsr_attach_band on a V = 1, S = 0 handle, "
               "K % 4 == 0, K <= ldb <= the pack's k_max, ldc % 4 == 0, 16-B aligned B and C");
  const Band *D = A->band;
  if (D->num_blocks == 0) return PSPMM_OK;
  BandArgs args;
  args.desc = D->d_desc;
  args.staged = D->d_staged;
  args.rng = D->d_rng;
  args.pairs = D->d_pairs;
  args.rowptr = D->d_rowptr;
  args.B = d_B;
  args.C = d_C;
  args.ldb = ldb;
  args.ldc = ldc;
  args.n_rows = (int32_t)A->n_rows;
  args.K = K;
  args.R = D->rows;
  args.accumulate = accumulate;
  args.nblk = D->num_blocks;
  args.stages = 2;
  if (const char *e = std::getenv("PSPMM_BAND_STAGES"))  // A/B knob for the tools (2..4)
    args.stages = std::max(2, std::min(kMaxStages, std::atoi(e)));
  args.fan = fan;
  switch (lanes_for(K)) {
    case 4: return launch_band<4>(args, D->num_blocks, stream);
    case 8: return launch_band<8>(args, D->num_blocks, stream);
    case 16: return launch_band<16>(args, D->num_blocks, stream);
    default: return launch_band<32>(args, D->num_blocks, stream);
  }
}

}  // namespace pspmm
