// (f4) PCSR binary file (External Interfaces of the pcsr
// module): little-endian header with the SPEC's fields in the SPEC's order,
// then this library's extension fields, then the four arrays.  Layout
// (format version 1; byte offsets):
//    0  char[4] "PCSR"          4  u32 version = 1
//    8  u64 n (rows)           16  u64 numPanels      24  u64 nnzV
//   32  u8  V                  33  u8  S              34  u16 omega
//   --- extension (version 1) ---
//   36  u32 reserved = 0       40  u64 numChunks (= numPanels when S = 0)
//   48  u64 SG (0 when S = 0)  56  u64 nnz (true nonzeros, for PR)
//   64  u64 nCols
//   72  rowPtr u64[numChunks + 1], colIdx u32[nnzV], val f32[nnzV V],
//       TRow u32[numChunks] iff S = 1
// The derived engine data (split-panel list, unit order, slice bounds) is
// rebuilt on load.  Loading validates every structural invariant of the
// PCSR (c-2) and rejects the file otherwise.
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"

namespace pspmm {
namespace {

constexpr uint32_t kVersion = 1;
constexpr size_t kHeader = 72;

template <typename T>
void put(unsigned char *h, size_t off, T v) {
  memcpy(h + off, &v, sizeof(T));
}
template <typename T>
T get(const unsigned char *h, size_t off) {
  T v;
  memcpy(&v, h + off, sizeof(T));
  return v;
}

struct File {
  FILE *f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

bool little_endian() {
  const uint16_t x = 1;
  unsigned char c;
  memcpy(&c, &x, 1);
  return c == 1;
}

}  // namespace
}  // namespace pspmm

using namespace pspmm;

extern "C" pspmm_status pspmm_pcsr_save(pspmm_pcsr A, const char *path) {
  return pspmm::guarded("pcsr_save", [&]() -> pspmm_status {
    if (!A || !path) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_save: null argument");
    if (!little_endian()) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "pcsr_save: big-endian host");
    const int64_t units = A->num_chunks, rl = A->rowptr_len, nv = A->nnz_v;
    std::vector<int32_t> rp(rl), ci(nv), tr(A->S ? units : 0);
    std::vector<float> val(nv * A->V);
    if (rl) PSPMM_CUDA_TRY(cudaMemcpy(rp.data(), A->d_rowptr, rl * 4, cudaMemcpyDeviceToHost));
    if (nv) {
      PSPMM_CUDA_TRY(cudaMemcpy(ci.data(), A->d_colidx, nv * 4, cudaMemcpyDeviceToHost));
      PSPMM_CUDA_TRY(cudaMemcpy(val.data(), A->d_val, nv * A->V * 4, cudaMemcpyDeviceToHost));
    }
    if (A->S && units)
      PSPMM_CUDA_TRY(cudaMemcpy(tr.data(), A->d_trow, units * 4, cudaMemcpyDeviceToHost));
    unsigned char h[kHeader] = {};
    memcpy(h, "PCSR", 4);
    put<uint32_t>(h, 4, kVersion);
    put<uint64_t>(h, 8, (uint64_t)A->n_rows);
    put<uint64_t>(h, 16, (uint64_t)A->num_panels);
    put<uint64_t>(h, 24, (uint64_t)nv);
    put<uint8_t>(h, 32, (uint8_t)A->V);
    put<uint8_t>(h, 33, (uint8_t)A->S);
    put<uint16_t>(h, 34, (uint16_t)A->omega);
    put<uint64_t>(h, 40, (uint64_t)units);
    put<uint64_t>(h, 48, (uint64_t)A->sg);
    put<uint64_t>(h, 56, (uint64_t)A->nnz);
    put<uint64_t>(h, 64, (uint64_t)A->n_cols);
    std::vector<uint64_t> rp64(rp.begin(), rp.end());
    File out;
    out.f = fopen(path, "wb");
    if (!out.f) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_save: cannot open the output file");
    bool ok = fwrite(h, 1, kHeader, out.f) == kHeader;
    ok = ok && fwrite(rp64.data(), 8, rl, out.f) == (size_t)rl;
    ok = ok && fwrite(ci.data(), 4, nv, out.f) == (size_t)nv;
    ok = ok && fwrite(val.data(), 4, nv * A->V, out.f) == (size_t)(nv * A->V);
    if (A->S) ok = ok && fwrite(tr.data(), 4, units, out.f) == (size_t)units;
    ok = fclose(out.f) == 0 && ok;
    out.f = nullptr;
    if (!ok) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_save: write failed");
    return PSPMM_OK;
  });
}

extern "C" pspmm_status pspmm_pcsr_load(const char *path, void *stream, pspmm_pcsr *out) {
  return pspmm::guarded("pcsr_load", [&]() -> pspmm_status {
    if (!path || !out) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: null argument");
    *out = nullptr;
    if (!little_endian()) PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "pcsr_load: big-endian host");
    File in;
    in.f = fopen(path, "rb");
    if (!in.f) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: cannot open the file");
    unsigned char h[kHeader];
    if (fread(h, 1, kHeader, in.f) != kHeader || memcmp(h, "PCSR", 4) != 0)
      PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: not a PCSR file (magic)");
    if (get<uint32_t>(h, 4) != kVersion)
      PSPMM_FAIL(PSPMM_ERR_UNSUPPORTED, "pcsr_load: unknown format version");
    const int64_t n = (int64_t)get<uint64_t>(h, 8), P = (int64_t)get<uint64_t>(h, 16);
    const int64_t nv = (int64_t)get<uint64_t>(h, 24), units = (int64_t)get<uint64_t>(h, 40);
    const int V = get<uint8_t>(h, 32), S = get<uint8_t>(h, 33), omega = get<uint16_t>(h, 34);
    const int64_t sg = (int64_t)get<uint64_t>(h, 48), nnz = (int64_t)get<uint64_t>(h, 56);
    const int64_t n_cols = (int64_t)get<uint64_t>(h, 64);
    const bool header_ok =
        (V == 1 || V == 2) && (S == 0 || S == 1) && omega >= 1 && n >= 0 && n < INT32_MAX &&
        n_cols >= 0 && n_cols < INT32_MAX && P == (n + V - 1) / V && nv >= 0 && nv < INT32_MAX &&
        units >= 0 && units < INT32_MAX && (S == 1 || (units == P && sg == 0)) &&
        (S == 0 || (sg >= 1 && units >= P)) && nnz >= 0 && nnz <= nv * V &&
        get<uint32_t>(h, 36) == 0;
    if (!header_ok) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: inconsistent header");
    // the file must be exactly as long as the header says, checked BEFORE any
    // header-sized allocation (a crafted header cannot trigger a huge one)
    const int64_t expect = (int64_t)kHeader + (units + 1) * 8 + nv * 4 + nv * V * 4 +
                           (S ? units * 4 : 0);
    if (fseeko(in.f, 0, SEEK_END) != 0)
      PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: cannot seek the file");
    const int64_t fsize = (int64_t)ftello(in.f);
    if (fsize != expect)
      PSPMM_FAIL(PSPMM_ERR_INVALID_ARG,
                 "pcsr_load: file size does not match the header (truncated or oversized)");
    if (fseeko(in.f, (off_t)kHeader, SEEK_SET) != 0)
      PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: cannot seek the file");
    std::vector<uint64_t> rp64(units + 1);
    std::vector<int32_t> ci(nv), tr(S ? units : 0);
    std::vector<float> val(nv * V);
    bool ok = fread(rp64.data(), 8, units + 1, in.f) == (size_t)(units + 1);
    ok = ok && fread(ci.data(), 4, nv, in.f) == (size_t)nv;
    ok = ok && fread(val.data(), 4, nv * V, in.f) == (size_t)(nv * V);
    if (S) ok = ok && fread(tr.data(), 4, units, in.f) == (size_t)units;
    unsigned char extra;
    ok = ok && fread(&extra, 1, 1, in.f) == 0;  // nothing after the arrays
    if (!ok) PSPMM_FAIL(PSPMM_ERR_INVALID_ARG, "pcsr_load: truncated or oversized file");
  
    // structural invariants: rowPtr monotone from 0 to nnzV; ascending columns
    // inside each panel (c-8) below nCols; TRow non-decreasing panel ids, each
    // panel owning >= 1 chunk (c-5), chunks of <= SG vectors cut at multiples
    // of SG from the panel start (Eq. 4 reading)
    std::vector<int32_t> rp(units + 1);
    if (rp64[0] != 0 || rp64[units] != (uint64_t)nv)
      PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: rowPtr must run from 0 to nnzV");
    for (int64_t u = 0; u <= units; ++u) {
      if (u && rp64[u] < rp64[u - 1])
        PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: rowPtr decreases");
      rp[u] = (int32_t)rp64[u];
    }
    std::vector<int64_t> first(P + 1, -1);  // first chunk of each panel
    if (S) {
      for (int64_t u = 0; u < units; ++u) {
        const int32_t p = tr[u];
        if (p < 0 || p >= P || (u && p < tr[u - 1]) || (u && p > tr[u - 1] + 1) ||
            (u == 0 && p != 0))
          PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: TRow must list every panel in order");
        if (first[p] < 0) first[p] = u;
        if (rp[u + 1] - rp[u] > sg)
          PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: chunk longer than SG");
      }
      if (units && tr[units - 1] != P - 1)
        PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: TRow must end at the last panel");
      for (int64_t u = 0; u < units; ++u)  // interior chunks are exactly SG long
        if (u + 1 < units && tr[u + 1] == tr[u] && rp[u + 1] - rp[u] != sg)
          PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: split chunk shorter than SG");
    } else {
      for (int64_t p = 0; p < P; ++p) first[p] = p;
    }
    first[P] = units;
    for (int64_t p = 0; p < P; ++p) {
      const int64_t a = rp[first[p]], b = rp[first[p + 1]];
      for (int64_t i = a; i < b; ++i)
        if (ci[i] < 0 || ci[i] >= n_cols || (i > a && ci[i] <= ci[i - 1]))
          PSPMM_FAIL(PSPMM_ERR_NOT_CANONICAL, "pcsr_load: panel columns not ascending / in range");
    }
  
    pspmm_pcsr_s *A = new (std::nothrow) pspmm_pcsr_s();
    if (!A) PSPMM_FAIL(PSPMM_ERR_OOM, "pcsr_load: host allocation failed");
    struct Guard {
      pspmm_pcsr_s *a;
      ~Guard() {
        if (a) pspmm_pcsr_destroy(a);
      }
    } guard{A};
    A->n_rows = n;
    A->n_cols = n_cols;
    A->num_panels = P;
    A->nnz = nnz;
    A->nnz_v = nv;
    A->num_chunks = units;
    A->sg = sg;
    A->rowptr_len = units + 1;
    A->V = V;
    A->S = S;
    A->omega = omega;
    A->pr = nv > 0 ? 1.0 - (double)nnz / ((double)nv * (double)V) : __builtin_nan("");
    A->sr = S ? (double)(units + 1) / (double)(P + 1) : 1.0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PSPMM_CUDA_TRY(cudaMalloc(&A->d_rowptr, (size_t)(units + 1) * 4));
    PSPMM_CUDA_TRY(cudaMemcpy(A->d_rowptr, rp.data(), (units + 1) * 4, cudaMemcpyHostToDevice));
    if (nv) {
      PSPMM_CUDA_TRY(cudaMalloc(&A->d_colidx, (size_t)nv * 4));
      PSPMM_CUDA_TRY(cudaMalloc(&A->d_val, (size_t)nv * V * 4));
      PSPMM_CUDA_TRY(cudaMemcpy(A->d_colidx, ci.data(), nv * 4, cudaMemcpyHostToDevice));
      PSPMM_CUDA_TRY(cudaMemcpy(A->d_val, val.data(), nv * V * 4, cudaMemcpyHostToDevice));
    }
    if (S) {
      std::vector<int32_t> split;
      for (int64_t p = 0; p < P; ++p)
        if (first[p + 1] - first[p] > 1) split.push_back((int32_t)p);
      A->num_split = (int64_t)split.size();
      PSPMM_CUDA_TRY(cudaMalloc(&A->d_trow, (size_t)(units > 0 ? units : 1) * 4));
      PSPMM_CUDA_TRY(cudaMalloc(&A->d_split, (size_t)(split.empty() ? 1 : split.size()) * 4));
      if (units)
        PSPMM_CUDA_TRY(cudaMemcpy(A->d_trow, tr.data(), units * 4, cudaMemcpyHostToDevice));
      if (!split.empty())
        PSPMM_CUDA_TRY(cudaMemcpy(A->d_split, split.data(), split.size() * 4,
                                  cudaMemcpyHostToDevice));
    }
    for (int k = 0; k <= kSlices; ++k) {
      const int64_t p = P * k / kSlices;
      A->slice_units[k] = first[p];
      A->slice_rows[k] = std::min<int64_t>(p * V, n);
    }
    pspmm_status st = build_unit_order(A, s);
    if (st != PSPMM_OK) return st;
    PSPMM_CUDA_TRY(cudaStreamSynchronize(s));
    guard.a = nullptr;
    *out = A;
    return PSPMM_OK;
  });
}
