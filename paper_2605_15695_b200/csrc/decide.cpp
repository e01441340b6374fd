// (a3) SpMM-decider stand-in (§5.2): a pure host
// function of (Table-3 features, K) -> <W, F, V, S> (+ G).  The paper uses a
// random forest trained on A6000 timings; here a decision tree trained on this
// repo's own B200 sweep is compiled in (decider_model.h).
// Before a model exists a rule derived from the paper's observations is used:
//   V = 2 iff PR_2 < 0.30      (T1: V = 2 wins at PR 26.8-30.6 %,
//                               loses at 47.8-49 %)
//   S = 1 iff d_max > 8 d^     (balancing pays on skewed degrees)
//   F: smallest coarsening whose row group fits in a warp with no MAC-job gap
//      (Eq. 1 generalised to 4G lanes).
#include "guard.h"
#include <algorithm>
#include <cmath>

#include "decider_model.h"
#include "pspmm.h"

namespace {

// B200 L2 (cudaDevAttrL2CacheSize on the target; the decider is a pure host
// function of (features, K), so the target's value is a constant here)
constexpr double kL2Bytes = 132644864.0;
// resident mode-0 warps: 148 SMs x 24 warps (the engine's launch bounds,
// 256 threads x 3 blocks per SM)
constexpr double kSMs = 148.0, kWarpsPerSM = 24.0;

int ceil_pow2(int x) {
  int p = 1;
  while (p < x && p < 32) p <<= 1;
  return p;
}

// float4 columns per lane F and lanes G covering K with the least waste.
void pick_fg(int K, int F_hint, int *F, int *G) {
  const int q = (K + 3) / 4;  // float4 columns (scalar path ignores F)
  if (F_hint >= 1 && F_hint <= 8) {
    *F = F_hint;
    *G = ceil_pow2((q + F_hint - 1) / F_hint);
    return;
  }
  int bestF = 1, bestG = ceil_pow2(q), bestWaste = 1 << 30;
  for (int f = 1; f <= 8; ++f) {
    const int g = ceil_pow2((q + f - 1) / f);
    const int cover = g * f;
    const int passes = (q + cover - 1) / cover;
    const int waste = passes * cover - q;
    // prefer zero waste, then one pass, then the smallest F (fewer registers)
    const int score = waste * 16 + (passes - 1) * 4;
    if (score < bestWaste) {
      bestWaste = score;
      bestF = f;
      bestG = g;
    }
  }
  *F = bestF;
  *G = bestG;
}

// model feature idx: 0..15 = the Table-3 fields in header order, 16 =
// log2(K), 17 = log2(n K 4 / L2 bytes) (B's footprint against the L2; the
// signal of the single-pass guard, learned from the sweep since round 2)
double feature_value(const pspmm_features *f, int idx, int K) {
  const double *v = reinterpret_cast<const double *>(f);
  if (idx >= 0 && idx < 16) return v[idx];
  if (idx == 17) return std::log2(std::max(f->n, 1.0) * (double)K * 4.0 / kL2Bytes);
  return std::log2((double)K);
}

}  // namespace

extern "C" pspmm_status pspmm_decide_config(const pspmm_features *f, int32_t K,
                                            pspmm_config *out) {
  return pspmm::guarded("decide_config", [&]() -> pspmm_status {
    if (!f || !out || K < 1) return PSPMM_ERR_INVALID_ARG;
    if (!(f->nnz > 0)) return PSPMM_ERR_EMPTY;
    pspmm_config c{};
    c.omega = 32;
    c.sg_override = 0;
    c.mode = 0;
  #if PSPMM_DECIDER_TRAINED
    // random forest: every tree votes for its leaf's label; the label
    // with the most votes wins, ties to the lowest label id
    int votes[pspmm_model::kNumLabels] = {};
    for (int t = 0; t < pspmm_model::kTrees; ++t) {
      int node = pspmm_model::kRoot[t];
      while (pspmm_model::kFeature[node] >= 0) {
        const double x = feature_value(f, pspmm_model::kFeature[node], K);
        node = x <= pspmm_model::kThreshold[node] ? pspmm_model::kLeft[node]
                                                  : pspmm_model::kRight[node];
      }
      votes[pspmm_model::kLeafLabel[node]]++;
    }
    int best = 0;
    for (int l = 1; l < pspmm_model::kNumLabels; ++l)
      if (votes[l] > votes[best]) best = l;
    const int *lab = pspmm_model::kLabel[best];
    c.mode = lab[0];
    c.V = lab[1];
    c.S = lab[2];
    c.W = lab[3];
    c.order = c.mode == 0 ? lab[6] : 0;
    if (c.mode == 2 && K % 32 != 0) c.mode = 0;  // TMA engine needs K % 32 == 0
    if (c.mode == 3 && K % 4 != 0) c.mode = 0;  // short-row engines: 128-bit only
    // the short-row engines walk a row's vectors beyond the staged window one
    // dependent load at a time: a hub row serialises its group (K sweep,
    // Cora K = 128, mode 3 0.059 ms vs cuSPARSE 0.023), so
    // graphs with rows longer than 64 vectors stay on mode 0
    if (c.mode == 3 && f->d_max > 64.0) c.mode = 0;
    // vectorized blocking only where it saves B reads: at PR_2 ~ 0.5 a V = 2
    // vector is a padded single value (the paper's T1: V = 2 loses
    // at PR 47.8-49 %); the forest's V = 2 there extrapolates a noise-level
    // label (products K = 128) to other graphs (Reddit K = 128: 4.46 ms with
    // V = 2 vs 3.22 ms with V = 1)
    if (c.V == 2 && f->pr2 >= 0.45) c.V = 1;
    if (c.mode == 2) {
      pick_fg(K, 0, &c.F, &c.G);  // unused by mode 2; a valid mode-0 fallback
    } else if (lab[0] == 2) {
      pick_fg(K, 0, &c.F, &c.G);
    } else {
      // G from the label's column-pass count P: the smallest power of two with
      // 4 G F P >= K (capped at 32 lanes)
      c.F = lab[4];
      const int P = lab[5];
      const int q = (K + 3) / 4;
      c.G = ceil_pow2((q + c.F * P - 1) / (c.F * P));
      // B far beyond L2 (the training corpus has no such graph at large K):
      // every column pass re-gathers one B segment per nonzero, and the
      // gather cost is per segment, so take one pass of 32 lanes (K sweep,
      // products K = 256, 4 passes 27.8 ms vs cuSPARSE 23.4)
      const int passes = (K + 4 * c.G * c.F - 1) / (4 * c.G * c.F);
      if (c.mode == 0 && passes > 1 && f->n * (double)K * 4.0 > 2.0 * kL2Bytes &&
          (q + 31) / 32 <= 8) {
        c.F = (q + 31) / 32;
        c.G = ceil_pow2((q + c.F - 1) / c.F);
      }
    }
    // sub-wave hub rows: when every S = 0 unit fits in one wave of resident
    // row groups (148 SMs x 24 warps x 32 / G), the launch lasts as long as
    // its longest row, so rows of >= 4 SG nonzeros (Eq. 3) are split (S = 1,
    // P:130).  On the training corpus this regime holds 18 (graph, K) points;
    // S = 1 is the sweep's best on all 18 and the forest already picks it on
    // all 18 (the guard changes no corpus decision); it covers graphs outside
    // the corpus such as Cora (d_max = 4.5-5 SG: K = 32 S = 0 20.5 us vs
    // S = 1 13.3 us)
    if (c.mode == 0 && c.V == 1 && c.S == 0 && c.G >= 1) {
      const double sg = std::ceil(f->d_hat / 32.0) * 32.0;
      const double groups = kSMs * kWarpsPerSM * (32.0 / c.G);
      if (f->n <= groups && f->d_max >= 4.0 * sg) c.S = 1;
    }
    *out = c;
    return PSPMM_OK;
  #else
    (void)feature_value;
    c.V = f->pr2 < 0.30 ? 2 : 1;
    c.S = f->d_max > 8.0 * f->d_hat ? 1 : 0;
    c.W = 4;
    pick_fg(K, 0, &c.F, &c.G);
    *out = c;
    return PSPMM_OK;
  #endif
  });
}
