// gather_ceiling.cu — X1 (SURVEY §2.3 / VERDICT r1 item 1a): the on-chip roofline of the MTTKRP hot
// loop as a HARDWARE property, measured per access shape and per data path.  Each lane-group of G
// lanes gathers random R-wide fp32 rows (the factor-row access of the SpMTTKRP, Eq.(6))
// and accumulates them; indices come from a per-lane LCG (one IMAD per row; no index loads, so
// the only memory traffic is the gathers themselves).  Measurement tooling only (not part of libfcoo).
//
// PATH (template):
//   0 LDG  : ld.global.nc, VEC floats per lane (VEC = 4/2/1 -> G = R/4, R/2, R lanes per row)
//   1 TEX  : tex1Dfetch<float4> on a linear texture object over the same table (TEX pipe)
//   2 LDS  : ld.shared from a shared-memory copy of the first SROWS rows
//   3 LDG+TEX : rows alternate between the two paths (one of each per step)
//   4 LDG+LDS : idem
//   5 LDS+TEX : idem
//   6 LDG+LDS+TEX : three rows per step, one per path
// ACT: fraction of lane-groups (out of 4 per warp, in 1/4 steps) that issue the gathers (the rest
// are predicated off) — mimics per-group reuse that skips a row.
// SHARE (1, 2, 4, 8): consecutive lane-groups of a warp, SHARE at a time, draw the SAME shared-memory
// row (LDS paths; LDG rows stay distinct per group) — does an LDS.128 whose quarter-warps read one
// row cost fewer data-pipe wavefronts (warp-cooperative fibre reuse)?
#include <cuda_runtime.h>
#include <stdint.h>



// Predicated loads (inline PTX) so an inactive lane-group issues nothing and the compiler keeps the
// kernel parameters in registers.
__device__ __forceinline__ float4 ldg4(bool q, const float* p) {
  float4 r = make_float4(0, 0, 0, 0);
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %4, 0; @q ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%5]; }"
               : "+f"(r.x), "+f"(r.y), "+f"(r.z), "+f"(r.w) : "r"((int)q), "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldg2(bool q, const float* p) {
  float4 r = make_float4(0, 0, 0, 0);
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.nc.v2.f32 {%0,%1}, [%3]; }"
               : "+f"(r.x), "+f"(r.y) : "r"((int)q), "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldg1(bool q, const float* p) {
  float4 r = make_float4(0, 0, 0, 0);
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %1, 0; @q ld.global.nc.f32 %0, [%2]; }" : "+f"(r.x) : "r"((int)q), "l"(p));
  return r;
}
__device__ __forceinline__ float4 lds4(bool q, uint32_t a) {
  float4 r = make_float4(0, 0, 0, 0);
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %4, 0; @q ld.shared.v4.f32 {%0,%1,%2,%3}, [%5]; }"
               : "+f"(r.x), "+f"(r.y), "+f"(r.z), "+f"(r.w) : "r"((int)q), "r"(a));
  return r;
}
__device__ __forceinline__ float4 lds2(bool q, uint32_t a) {
  float4 r = make_float4(0, 0, 0, 0);
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.f32 {%0,%1}, [%3]; }"
               : "+f"(r.x), "+f"(r.y) : "r"((int)q), "r"(a));
  return r;
}
__device__ __forceinline__ float4 lds1(bool q, uint32_t a) {
  float4 r = make_float4(0, 0, 0, 0);
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %1, 0; @q ld.shared.f32 %0, [%2]; }" : "+f"(r.x) : "r"((int)q), "r"(a));
  return r;
}

template <int R, int VEC, int PATH, int U>
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ table, cudaTextureObject_t tex, uint32_t rows,
                                                uint32_t srows, int steps, int act4, int share, float* __restrict__ out) {
  extern __shared__ float4 smraw[];
  constexpr bool use_lds = PATH == 2 || PATH == 4 || PATH == 5 || PATH == 6;
  if (use_lds) {
    const int n4 = (int)srows * R / 4;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) smraw[k] = __ldg(reinterpret_cast<const float4*>(table) + k);
    __syncthreads();
  }
  constexpr int G = R / VEC;
  const int gl = threadIdx.x % G;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool active = ((grp & 3) < (uint32_t)act4);
  const int col = gl * VEC;
  const float* tb = table + col;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smraw) + col * 4;
  float4 acc = make_float4(0, 0, 0, 0);
  uint32_t x = grp * 0x9e3779b9u + 12345u;
  uint32_t xs = (grp / (uint32_t)share) * 0x9e3779b9u + 777u;  // shared-memory row draws
  for (int s = 0; s < steps; ++s) {
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x = x * 1664525u + 1013904223u;  // LCG: one IMAD per row
      xs = xs * 1664525u + 1013904223u;
      int path = PATH;
      if (PATH == 3) path = (u & 1) ? 1 : 0;
      if (PATH == 4) path = (u & 1) ? 2 : 0;
      if (PATH == 5) path = (u & 1) ? 1 : 2;
      if (PATH == 6) path = u % 3 == 0 ? 0 : u % 3 == 1 ? 2 : 1;
      if (path == 0) {
        const float* p = tb + (size_t)__umulhi(x, rows) * R;
        r[u] = VEC == 4 ? ldg4(active, p) : VEC == 2 ? ldg2(active, p) : ldg1(active, p);
      } else if (path == 2) {
        const uint32_t a = sb + __umulhi(xs, srows) * (R * 4);
        r[u] = VEC == 4 ? lds4(active, a) : VEC == 2 ? lds2(active, a) : lds1(active, a);
      } else {  // texture: float4 texels, G = R/4 lanes per row (VEC == 4 only)
        r[u] = active ? tex1Dfetch<float4>(tex, (int)(__umulhi(x, rows) * (uint32_t)(R / 4) + gl)) : make_float4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += r[u].x; acc.y += r[u].y; acc.z += r[u].z; acc.w += r[u].w; }
  }
  if (acc.x == 1234.5f) out[grp] = acc.x + acc.y + acc.z + acc.w;  // keep the loads alive
}

template <int R, int VEC, int PATH>
static void launch(const float* table, cudaTextureObject_t tex, uint32_t rows, uint32_t srows, int steps,
                   int act4, int share, float* out, unsigned blocks, size_t smem, cudaStream_t s) {
  constexpr int U = (PATH == 6) ? 12 : 8;
  auto k = k_gather<R, VEC, PATH, U>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, smem ? 100 : 0);
  k<<<blocks, 256, smem, s>>>(table, tex, rows, srows, steps, act4, share, out);
}

template <int R>
static void go_r(int vec, int path, const float* table, cudaTextureObject_t tex, uint32_t rows, uint32_t srows,
                 int steps, int act4, int share, float* out, unsigned blocks, size_t smem, cudaStream_t s) {
#define GO(VV, PP) launch<R, VV, PP>(table, tex, rows, srows, steps, act4, share, out, blocks, smem, s)
  if (vec == 4) {
    switch (path) {
      case 0: GO(4, 0); break; case 1: GO(4, 1); break; case 2: GO(4, 2); break; case 3: GO(4, 3); break;
      case 4: GO(4, 4); break; case 5: GO(4, 5); break; default: GO(4, 6); break;
    }
  } else if constexpr (R / 2 <= 32) {
    if (vec == 2) {
      switch (path) { case 0: GO(2, 0); break; case 2: GO(2, 2); break; default: GO(2, 4); break; }
    } else if constexpr (R <= 32) {
      switch (path) { case 0: GO(1, 0); break; case 2: GO(1, 2); break; default: GO(1, 4); break; }
    }
  }
#undef GO
}

// Returns the number of row gathers issued per launch in *n_rows and the mean launch time in *ms_out.
extern "C" int gather_bench3(const float* table, uint32_t rows, int R, int vec, int path, uint32_t srows, int act4,
                             int share, int blocks_per_sm, int steps, float* out, void* stream, int reps, float* ms_out,
                             double* n_rows) {
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaTextureObject_t tex = 0;
  if (path == 1 || path == 3 || path == 5 || path == 6) {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<float*>(table);
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = (size_t)rows * R * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) return -1;
  }
  const unsigned blocks = (unsigned)(nsm * blocks_per_sm);
  const bool lds = path == 2 || path == 4 || path == 5 || path == 6;
  const size_t smem = lds ? (size_t)srows * R * 4 : 0;
  auto go = [&]() {
    if (R == 16) go_r<16>(vec, path, table, tex, rows, srows, steps, act4, share, out, blocks, smem, s);
    else if (R == 32) go_r<32>(vec, path, table, tex, rows, srows, steps, act4, share, out, blocks, smem, s);
    else go_r<64>(vec, path, table, tex, rows, srows, steps, act4, share, out, blocks, smem, s);
  };
  go();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms_out, e0, e1);
  *ms_out /= reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (tex) cudaDestroyTextureObject(tex);
  const int G = R / vec;
  const double groups = (double)blocks * 256 / G;
  const int U = path == 6 ? 12 : 8;
  *n_rows = groups * act4 / 4.0 * steps * U;
  return (int)cudaGetLastError();
}
