// umma_tf32_probe.cu — prototype (measurement tooling, not part of libfcoo): does a hand-written
// tcgen05.mma kind::tf32 with A in TMEM and an MN-major B tile in shared memory compute
// D(128 x 32) += A(128 x 8) * B(8 x 32)^T the way the SpTTMc kernel would use it (A rows = the
// segment's v * U_a rows transposed, B = U_b rows), and where does D land in TMEM?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_tf32_probe.cu && ./umma_probe
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <math.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// instruction descriptor (cute::UMMA::InstrDescriptor): c F32, a/b TF32, a K-major (TMEM), b MN-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// shared-memory matrix descriptor (cute::UMMA::SmemDescriptor), SWIZZLE_NONE, version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;
}

__global__ void k_probe(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ D, int M, int N,
                        int K, int mode, uint32_t sbo, uint32_t lbo, int a_src, int roundtrip, uint32_t a_lbo = 128,
                        uint32_t a_sbo = 256) {
  // A: M x K row-major (A[m][k]); B: N x K (B[n][k]); D: M x N; one CTA of 128 threads (4 warps)
  __shared__ __align__(1024) float bt[2048];
  __shared__ __align__(1024) float at[2048];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // B tile, MN-major interleaved: element (n, k) at byte (n/4)*sbo + k*16 + (n%4)*4
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    if (mode == 1)  // MN-major interleaved
      *reinterpret_cast<float*>(reinterpret_cast<char*>(bt) + (n / 4) * sbo + k * 16 + (n % 4) * 4) = B[n * K + k];
    else  // K-major interleaved: core = 8 n-rows x 16 B (4 k), next k-core at lbo, next n-group at sbo
      *reinterpret_cast<float*>(reinterpret_cast<char*>(bt) + (n / 8) * sbo + (k / 4) * lbo + (n % 8) * 16 + (k % 4) * 4) =
          B[n * K + k];
  }
  // A tile in shared memory, K-major interleaved: element (m, k) at byte (m/8)*256 + (k/4)*128 + (m%8)*16 + (k%4)*4
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(at) + (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4) =
        A[m * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;  // columns [0,32): D, [32,40): A
  const uint32_t tD = tm, tA = tm + 32;
  // A into TMEM: lane m = row m, column k (warp w owns lanes 32w..32w+31)
  {
    uint32_t r[8];
    const int m = warp * 32 + lane;
    for (int k = 0; k < 8; ++k) r[k] = __float_as_uint(m < M && k < K ? A[m * K + k] : 0.f);
    const uint32_t addr = tA + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (roundtrip) {  // D region <- known values by tcgen05.st (roundtrip 1: read back; 2: then accumulate MMA)
    uint32_t r[8];
    for (int c = 0; c < 32; c += 8) {
      for (int k = 0; k < 8; ++k) r[k] = __float_as_uint((float)((warp * 32 + lane) * 100 + c + k));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       tD + ((uint32_t)(warp * 32) << 16) + c), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
                   "r"(r[5]), "r"(r[6]), "r"(r[7])
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    if (roundtrip == 1 && tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mbar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (roundtrip != 1 && tid == 0) {
    const uint64_t bd = sdesc(smem_u32(bt), lbo, sbo);
    const uint32_t id = idesc_tf32(128, N, mode);
    if (a_src == 0) {
      asm volatile(
          "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
          "  tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }" ::"r"(tD),
          "r"(tA), "l"(bd), "r"(id), "r"(roundtrip == 2 ? 1 : 0)
          : "memory");
    } else {
      const uint64_t ad = sdesc(smem_u32(at), a_lbo, a_sbo);
      asm volatile(
          "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
          "  tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(tD),
          "l"(ad), "l"(bd), "r"(id), "r"(roundtrip == 2 ? 1 : 0)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  __syncwarp();
  {  // every thread waits for the MMA
    const uint32_t mb = smem_u32(&mbar);
    asm volatile(
        "{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(mb), "r"(0)
        : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {  // D out: lane = row, 32 columns
    uint32_t v[32];
    const uint32_t addr = tD + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = warp * 32 + lane;
    for (int n = 0; n < 32; ++n) D[m * 32 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(64));
}

int main() {
  const int M = 128, N = 32, K = 8;
  float hA[M * K], hB[N * K], hD[M * 32];
  for (int i = 0; i < M * K; ++i) hA[i] = (float)((i * 7) % 13) - 6.0f;   // small integers: exact in tf32
  for (int i = 0; i < N * K; ++i) hB[i] = (float)((i * 5) % 11) - 5.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  // 1. st/ld roundtrip
  cudaMemset(dD, 0, sizeof hD);
  k_probe<<<1, 128>>>(dA, dB, dD, M, N, K, 1, 128, 1024, 0, 1);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("roundtrip: CUDA error\n"); return 1; }
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int rbad = 0;
  for (int m = 0; m < M; ++m) for (int n = 0; n < 32; ++n) rbad += hD[m * 32 + n] != (float)(m * 100 + n);
  printf("roundtrip: %d of %d wrong; D[1][0..2] = %g %g %g\n", rbad, M * 32, hD[32], hD[33], hD[34]);
  // 1b. prefill + accumulating MMA (A from smem): does the MMA write at all?
  for (int a_src = 1; a_src >= 0; --a_src) {
    cudaMemset(dD, 0, sizeof hD);
    k_probe<<<1, 128>>>(dA, dB, dD, M, N, K, 1, 128, 1024, a_src, 2);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("accumulate: CUDA error\n"); return 1; }
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    printf("prefill+acc a_src=%d: D[0][0..3] = %g %g %g %g  D[1][0..1] = %g %g  D[64][0] = %g\n", a_src, hD[0], hD[1],
           hD[2], hD[3], hD[32], hD[33], hD[64 * 32]);
  }
  // 1c. everything K-major (A smem, B smem), both (lbo, sbo) conventions
  for (int sw = 0; sw < 2; ++sw) {
    const uint32_t lb = sw ? 256 : 128, sb = sw ? 128 : 256;
    cudaMemset(dD, 0, sizeof hD);
    // A fill uses (m/8)*256 + (k/4)*128: descriptor (lbo, sbo) = (128, 256) describes it; sw swaps the fields
    k_probe<<<1, 128>>>(dA, dB, dD, M, N, K, 0, sb, lb, 1, 0, lb, sb);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("kmajor: CUDA error\n"); return 1; }
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double r00 = 0;
    for (int k = 0; k < K; ++k) r00 += (double)hA[k] * hB[k];
    int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)hA[m * K + k] * hB[n * K + k];
        bad += fabs(ref - hD[m * 32 + n]) > 1e-3;
      }
    printf("K-major A,B desc(lbo=%u,sbo=%u): bad %d; D[0][0..3] = %g %g %g %g (ref %g)\n", lb, sb, bad, hD[0], hD[1], hD[2], hD[3], r00);
  }
  // 1d. A from TMEM, B K-major (desc lbo=128, sbo=256), idesc b_major = 0
  {
    cudaMemset(dD, 0, sizeof hD);
    k_probe<<<1, 128>>>(dA, dB, dD, M, N, K, 0, 256, 128, 0, 0);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("tmem-A: CUDA error\n"); return 1; }
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)hA[m * K + k] * hB[n * K + k];
        bad += fabs(ref - hD[m * 32 + n]) > 1e-3;
      }
    printf("A in TMEM, B K-major: bad %d; D[0][0..3] = %g %g %g %g\n", bad, hD[0], hD[1], hD[2], hD[3]);
  }
  // 2. MMA, A from shared memory (K-major) and from TMEM; B MN-major with candidate strides
  const uint32_t cands[][2] = {{128, 1024}, {1024, 128}};
  for (int a_src = 1; a_src >= 0; --a_src)
    for (auto& c : cands) {
      cudaMemset(dD, 0, sizeof hD);
      k_probe<<<1, 128>>>(dA, dB, dD, M, N, K, 1, c[0], c[1], a_src, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("a_src=%d sbo=%u lbo=%u: CUDA error %s\n", a_src, c[0], c[1], cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      int bad = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)hA[m * K + k] * hB[n * K + k];
          const double err = fabs(ref - hD[m * 32 + n]);
          if (err > 1e-3) ++bad;
          if (err > maxerr) maxerr = err;
        }
      double r00 = 0;
      for (int k = 0; k < K; ++k) r00 += (double)hA[k] * hB[k];
      printf("a_src=%s sbo=%u lbo=%u: max abs err %g, bad %d of %d; D[0][0..3] = %g %g %g %g (ref D[0][0] %g)\n",
             a_src ? "smem" : "tmem", c[0], c[1], maxerr, bad, M * N, hD[0], hD[1], hD[2], hD[3], r00);
    }
  return 0;
}
