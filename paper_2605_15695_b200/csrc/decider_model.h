// Random-forest model of the SpMM-decider.
// PLACEHOLDER: no sweep has been run yet, so the decider uses the
// hand-written rule in decide.cpp.  tools/train_decider.py overwrites this
// file with a forest trained on the repo's own B200 autotune sweep.
#pragma once
#define PSPMM_DECIDER_TRAINED 0
#define PSPMM_DECIDER_SOURCE "rule (untrained)"
namespace pspmm_model {
constexpr int kTrees = 1;
constexpr int kNodes = 1;
constexpr int kNumLabels = 1;
// feature index: 0..15 = pspmm_features fields in header order, 16 = log2(K)
constexpr int kRoot[kTrees] = {0};
constexpr int kFeature[kNodes] = {-1};
constexpr double kThreshold[kNodes] = {0.0};
constexpr int kLeft[kNodes] = {-1};
constexpr int kRight[kNodes] = {-1};
// leaf -> label id (-1 for inner nodes)
constexpr int kLeafLabel[kNodes] = {0};
// label: {mode, V, S, W, F, P (column passes)}
constexpr int kLabel[kNumLabels][6] = {{0, 1, 0, 4, 1, 1}};
}  // namespace pspmm_model
