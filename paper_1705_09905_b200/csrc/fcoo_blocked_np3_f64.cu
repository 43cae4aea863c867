// Explicit instantiation of the blocked SpMTTKRP kernels for 3 product modes, double accumulation
// (one translation unit per (count, accumulator) so nvcc compiles them in parallel; see
// fcoo_blocked.cuh).
#include "fcoo_blocked_kernels.cuh"

namespace fcoo {
template cudaError_t launch_blocked_np<3, double>(const BlockedParams&, int, bool, cudaStream_t);
}  // namespace fcoo
