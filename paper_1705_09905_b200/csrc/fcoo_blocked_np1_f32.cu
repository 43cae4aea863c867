// Explicit instantiation of the blocked SpMTTKRP kernels for 1 product modes, float accumulation
// (one translation unit per (count, accumulator) so nvcc compiles them in parallel; see
// fcoo_blocked.cuh).
#include "fcoo_blocked_kernels.cuh"

namespace fcoo {
template cudaError_t launch_blocked_np<1, float>(const BlockedParams&, int, bool, cudaStream_t);
}  // namespace fcoo
