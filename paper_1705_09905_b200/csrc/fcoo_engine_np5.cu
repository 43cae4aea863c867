// Instances of the engine kernels for 5 product mode(s).
#include "fcoo_engine_kernels.cuh"

namespace fcoo {
template cudaError_t launch_np<5, float>(const EngineParams&, bool, cudaStream_t);
template cudaError_t launch_np<5, double>(const EngineParams&, bool, cudaStream_t);
}  // namespace fcoo
