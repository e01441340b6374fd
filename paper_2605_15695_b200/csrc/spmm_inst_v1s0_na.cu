// Kernel instances of the engine for V = 1, S = 0 with L1::no_allocate B
// gathers (see spmm_kernel.cuh).
#include "spmm_kernel.cuh"

namespace pspmm {
namespace detail {
KernelFn pick_v1s0_na(int F, int G) { return pick_na<1, 0>(F, G); }
}  // namespace detail
}  // namespace pspmm
