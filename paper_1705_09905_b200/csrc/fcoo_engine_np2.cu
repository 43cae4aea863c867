// Instances of the engine kernels for 2 product mode(s).
#include "fcoo_engine_kernels.cuh"

namespace fcoo {
template cudaError_t launch_np<2, float>(const EngineParams&, bool, cudaStream_t);
template cudaError_t launch_np<2, double>(const EngineParams&, bool, cudaStream_t);
}  // namespace fcoo
