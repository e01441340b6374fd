// Kernel instances of the engine for V = 1, S = 0 (see spmm_kernel.cuh).
#include "spmm_kernel.cuh"

namespace pspmm {
namespace detail {
KernelFn pick_v1s0(bool vec, int F, int G) { return pick<1, 0>(vec, F, G); }
}  // namespace detail
}  // namespace pspmm
