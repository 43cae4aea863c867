// gather_ceiling.cu — X1: the on-chip roofline of the MTTKRP hot loop.  Random
// R-wide fp32 row gathers (float4 per lane, R/4 lanes per row, like k_segreduce) from a table
// of `rows` rows, indices from a device array.  Sweeping the table size separates the L1-resident
// and L2-resident gather bandwidths.  Measurement tooling only (not part of libfcoo).
#include <cuda_runtime.h>
#include <stdint.h>

template <int G>
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ table, const uint32_t* __restrict__ idx,
                                                int64_t n_per_group, int R, float* __restrict__ out) {
  const int gl = threadIdx.x % G;
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const uint32_t* ix = idx + grp * n_per_group;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t e = 0; e < n_per_group; e += 8) {
    uint4 a = __ldg(reinterpret_cast<const uint4*>(ix + e));
    uint4 b = __ldg(reinterpret_cast<const uint4*>(ix + e + 4));
    uint32_t k[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    float4 r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(table + (int64_t)k[q] * R + gl * 4));
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc.x += r[q].x; acc.y += r[q].y; acc.z += r[q].z; acc.w += r[q].w;
    }
  }
  if (acc.x == 1234.5f) out[grp] = acc.x + acc.y + acc.z + acc.w;  // keep the loads alive
}

extern "C" int gather_bench(const float* table, const uint32_t* idx, int64_t n_idx, int R, float* out,
                            void* stream, int reps, float* ms_out) {
  const int G = R / 4;
  const int64_t per = 256;
  int64_t groups = n_idx / per;
  int64_t threads = groups * G;
  unsigned blocks = (unsigned)((threads + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  auto launch = [&]() {
    switch (G) {
      case 4: k_gather<4><<<blocks, 256, 0, s>>>(table, idx, per, R, out); break;
      case 8: k_gather<8><<<blocks, 256, 0, s>>>(table, idx, per, R, out); break;
      case 16: k_gather<16><<<blocks, 256, 0, s>>>(table, idx, per, R, out); break;
      default: return;
    }
  };
  cudaFuncSetAttribute(k_gather<4>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
  cudaFuncSetAttribute(k_gather<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
  cudaFuncSetAttribute(k_gather<16>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms_out, e0, e1);
  *ms_out /= reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}
