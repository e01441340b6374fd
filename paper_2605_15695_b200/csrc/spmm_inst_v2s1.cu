// Kernel instances of the engine for V = 2, S = 1 (see spmm_kernel.cuh).
#include "spmm_kernel.cuh"

namespace pspmm {
namespace detail {
KernelFn pick_v2s1(bool vec, int F, int G) { return pick<2, 1>(vec, F, G); }
}  // namespace detail
}  // namespace pspmm
