// Kernel instances of the engine for V = 1, S = 1 (see spmm_kernel.cuh).
#include "spmm_kernel.cuh"

namespace pspmm {
namespace detail {
KernelFn pick_v1s1(bool vec, int F, int G) { return pick<1, 1>(vec, F, G); }
}  // namespace detail
}  // namespace pspmm
