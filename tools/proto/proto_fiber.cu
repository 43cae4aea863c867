// proto_fiber.cu — EXPERIMENT ONLY (not part of libfcoo): the SpMTTKRP hot loop on an F-COO
// stream whose order is blocked on the outer product mode, with
//   VAR 1: fibre factoring (outer row once per fibre, via LDG), unblocked order;
//   VAR 2: blocked order, fibre factoring, outer rows from a shared-memory block;
//   VAR 3: blocked order, outer row from shared memory for every nonzero (no fibre factoring);
//   VAR 4: blocked order, outer row via LDG for every nonzero (control).
// 3-order only (NP = 2), float4 lanes, G = R/4.  The stream is staged with cp.async like the
// library kernel.  Driven by tools/proto/proto_fiber.py.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

struct PP {
  const uint32_t* po;   // outer product index per nonzero (padded stream)
  const uint32_t* pi;   // inner product index
  const float* val;
  const uint32_t* bf;   // segment heads
  const uint32_t* ff;   // fibre heads (superset of bf)
  const uint32_t* sf;
  const uint32_t* seg_base;
  const uint32_t* seg_row;
  const int* item_blk;
  const int* item_t0;
  const int* item_nt;
  const float* Uo;
  const float* Ui;
  float* out;
  int64_t ntiles;
  int T, R, BR, Io;
};

__device__ __forceinline__ void cp16(void* d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void cp4(void* d, const void* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void red4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void red4_if(bool q, float* p, float4 v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.global.add.v4.f32 [%1], {%2,%3,%4,%5}; }" ::"r"((int)q), "l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds_if(bool q, uint32_t a, float4 old) {
  float4 r = old;
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %4, 0; @q ld.shared.v4.f32 {%0,%1,%2,%3}, [%5]; }"
               : "+f"(r.x), "+f"(r.y), "+f"(r.z), "+f"(r.w)
               : "r"((int)q), "r"(a));
  return r;
}
__device__ __forceinline__ float4 ldg_if(bool q, const float* p, float4 old) {
  float4 r = old;
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %4, 0; @q ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%5]; }"
               : "+f"(r.x), "+f"(r.y), "+f"(r.z), "+f"(r.w)
               : "r"((int)q), "l"(p));
  return r;
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ float4 f4fma(float a, float4 b, float4 c) {
  return make_float4(fmaf(a, b.x, c.x), fmaf(a, b.y, c.y), fmaf(a, b.z, c.z), fmaf(a, b.w, c.w));
}
__device__ __forceinline__ float4 f4fma4(float4 a, float4 b, float4 c) {
  return make_float4(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y), fmaf(a.z, b.z, c.z), fmaf(a.w, b.w, c.w));
}
__device__ __forceinline__ float4 f4mul(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }
__device__ __forceinline__ float4 sel4(bool q, float4 a, float4 b) { return q ? a : b; }

// stage: per group 2 x [po(32) pi(32) val(32) bf ff pad2]
constexpr int WORDS = 3 * 32 + 4;
constexpr int STRIDE = 2 * WORDS + 4;  // 204 words: 204 % 32 = 12 -> groups spread over banks

template <int G, int TB, int VAR>
__global__ void __launch_bounds__(TB, 512 / TB) k_proto(const PP P) {
  extern __shared__ float4 sm[];
  const bool blocked = VAR >= 2;
  const bool fiber = VAR <= 2;
  const bool smem_outer = VAR == 2 || VAR == 3;
  const int item = blockIdx.x;
  const int b = blocked ? P.item_blk[item] : 0;
  const int R = P.R;
  float* blk = reinterpret_cast<float*>(sm);
  const int rows_smem = smem_outer ? P.BR : 0;
  uint32_t* stg_all = reinterpret_cast<uint32_t*>(blk + (size_t)rows_smem * R);
  if (smem_outer) {  // cooperative copy of outer rows [b*BR, min((b+1)*BR, Io))
    const int r0 = b * P.BR;
    const int nr = min(P.BR, P.Io - r0);
    const float4* src = reinterpret_cast<const float4*>(P.Uo + (size_t)r0 * R);
    float4* dst = reinterpret_cast<float4*>(blk);
    const int n4 = nr * R / 4;
    for (int k = threadIdx.x; k < n4; k += TB) dst[k] = __ldg(src + k);
    __syncthreads();
  }
  const int g = threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int nt = blocked ? P.item_nt[item] : 0;
  const int64_t t = blocked ? (int64_t)P.item_t0[item] + g : (int64_t)item * (TB / G) + g;
  if ((blocked && g >= nt) || t >= P.ntiles) return;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  uint32_t* my = stg_all + g * STRIDE;
  const int col = gl * 4;
  const char* ubo = reinterpret_cast<const char*>(P.Uo + col);
  const char* ubi = reinterpret_cast<const char*>(P.Ui + col);
  const uint32_t rowb = (uint32_t)R * 4u;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(blk) + col * 4 - (uint32_t)(b * P.BR) * rowb;

  const int64_t p0 = t * (int64_t)P.T;
  const int nchunk = P.T / 32;
  const bool left_open = !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = P.seg_base[t] - 1u;
  uint32_t row = left_open ? P.seg_row[s] : 0u;
  float4 acc = make_float4(0, 0, 0, 0), run = acc, u = acc;

  auto issue = [&](int64_t pc, int st) {
    uint32_t* d = my + st * WORDS;
    const uint32_t* bases[3] = {P.po, P.pi, reinterpret_cast<const uint32_t*>(P.val)};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int k = 0; k < (8 + G - 1) / G; ++k) {
        const int q = gl + k * G;
        if (q < 8) cp16(d + a * 32 + q * 4, bases[a] + pc + q * 4);
      }
    if (gl == 0) cp4(d + 96, P.bf + (pc >> 5));
    if (gl == 1 % G) cp4(d + 97, P.ff + (pc >> 5));
  };
  issue(p0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int ci = 0; ci < nchunk; ++ci) {
    if (ci + 1 < nchunk) issue(p0 + (int64_t)(ci + 1) * 32, (ci + 1) & 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp(gmask);
    const uint32_t* st = my + (ci & 1) * WORDS;
    const uint32_t bfw = st[96];
    uint32_t ffw = st[97];
    if (ci == 0) ffw |= 1u;  // the tile's first nonzero always (re)loads its fibre's outer row
#pragma unroll
    for (int bi = 0; bi < 4; ++bi) {
      uint32_t io[8], ii[8], vb[8];
      {
        uint4 a0 = reinterpret_cast<const uint4*>(st + bi * 8)[0], a1 = reinterpret_cast<const uint4*>(st + bi * 8)[1];
        io[0] = a0.x; io[1] = a0.y; io[2] = a0.z; io[3] = a0.w; io[4] = a1.x; io[5] = a1.y; io[6] = a1.z; io[7] = a1.w;
        uint4 c0 = reinterpret_cast<const uint4*>(st + 32 + bi * 8)[0], c1 = reinterpret_cast<const uint4*>(st + 32 + bi * 8)[1];
        ii[0] = c0.x; ii[1] = c0.y; ii[2] = c0.z; ii[3] = c0.w; ii[4] = c1.x; ii[5] = c1.y; ii[6] = c1.z; ii[7] = c1.w;
        uint4 d0 = reinterpret_cast<const uint4*>(st + 64 + bi * 8)[0], d1 = reinterpret_cast<const uint4*>(st + 64 + bi * 8)[1];
        vb[0] = d0.x; vb[1] = d0.y; vb[2] = d0.z; vb[3] = d0.w; vb[4] = d1.x; vb[5] = d1.y; vb[6] = d1.z; vb[7] = d1.w;
      }
      const uint32_t heads = (bfw >> (bi * 8)) & 0xffu;
      const uint32_t fh = (ffw >> (bi * 8)) & 0xffu;
      float4 wi[8], wo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) wi[e] = __ldg(reinterpret_cast<const float4*>(ubi + (size_t)ii[e] * rowb));
      if constexpr (fiber) {
        // outer rows only at fibre heads (predicated loads into per-nonzero registers)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool q = (fh >> e) & 1u;
          if constexpr (smem_outer) wo[e] = lds_if(q, sbase + io[e] * rowb, make_float4(0, 0, 0, 0));
          else wo[e] = ldg_if(q, reinterpret_cast<const float*>(ubo + (size_t)io[e] * rowb), make_float4(0, 0, 0, 0));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if constexpr (smem_outer) wo[e] = lds4(sbase + io[e] * rowb);
          else wo[e] = __ldg(reinterpret_cast<const float4*>(ubo + (size_t)io[e] * rowb));
        }
      }
      const bool first = (ci == 0 && bi == 0);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool hd = (heads >> e) & 1u;
        const float v = __uint_as_float(vb[e]);
        if constexpr (fiber) {
          const bool f = (fh >> e) & 1u;
          // close the running fibre: acc += run * u (u = its outer row)
          if (f) acc = f4fma4(run, u, acc);
          if (hd && !(e == 0 && first)) {
            red4(P.out + (size_t)row * R + col, acc);
          }
          if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
          run = f ? make_float4(0, 0, 0, 0) : run;
          u = f ? wo[e] : u;
          run = f4fma(v, wi[e], run);
        } else {
          if (hd && !(e == 0 && first)) red4(P.out + (size_t)row * R + col, acc);
          if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
          acc = f4fma(v, f4mul(wo[e], wi[e]), acc);
        }
      }
    }
    __syncwarp(gmask);
  }
  if constexpr (fiber) acc = f4fma4(run, u, acc);
  red4(P.out + (size_t)row * R + col, acc);
}

template <int G, int TB, int VAR>
static int launch(const PP& P, int nitems, size_t smem, cudaStream_t s) {
  auto k = k_proto<G, TB, VAR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k<<<nitems, TB, smem, s>>>(P);
  return (int)cudaGetLastError();
}

template <int G, int TB>
static int launch_var(int var, const PP& P, int nitems, size_t smem, cudaStream_t s) {
  switch (var) {
    case 1: return launch<G, TB, 1>(P, nitems, smem, s);
    case 2: return launch<G, TB, 2>(P, nitems, smem, s);
    case 3: return launch<G, TB, 3>(P, nitems, smem, s);
    default: return launch<G, TB, 4>(P, nitems, smem, s);
  }
}

extern "C" int proto_run(int var, int tb, const PP* P, int nitems, void* stream) {
  const int G = P->R / 4;
  const bool so = var == 2 || var == 3;
  size_t smem = (size_t)(so ? P->BR : 0) * P->R * 4 + (size_t)(tb / G) * STRIDE * 4;
  cudaStream_t s = (cudaStream_t)stream;
  if (tb == 512) {
    switch (G) {
      case 4: return launch_var<4, 512>(var, *P, nitems, smem, s);
      case 8: return launch_var<8, 512>(var, *P, nitems, smem, s);
      default: return launch_var<16, 512>(var, *P, nitems, smem, s);
    }
  }
  switch (G) {
    case 4: return launch_var<4, 256>(var, *P, nitems, smem, s);
    case 8: return launch_var<8, 256>(var, *P, nitems, smem, s);
    default: return launch_var<16, 256>(var, *P, nitems, smem, s);
  }
}
extern "C" int proto_sizeof() { return (int)sizeof(PP); }

// ---------------------------------------------------------------------------------------------
// Lean blocked kernel (VAR 5: no fibre factoring, VAR 6: fibre factoring): packed stream word
// pk = (outer_local << IB) | inner, zero padding after each block's real nonzeros (blk_end),
// outer rows from shared memory (TMA bulk copy), inner rows LDG, packed f32x2 arithmetic.
struct PB {
  const uint32_t* pk;
  const float* val;
  const uint32_t* bf;
  const uint32_t* ff;
  const uint32_t* sf;
  const uint32_t* seg_base;
  const uint32_t* seg_row;
  const int* item_blk;
  const int* item_t0;
  const int* item_nt;
  const int64_t* blk_end;
  const float* Uo;
  const float* Ui;
  float* out;
  int64_t ntiles;
  int T, BR, Io, IB;
};

struct f2 { float x, y; };
__device__ __forceinline__ unsigned long long u64of(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ void split(unsigned long long r, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
// acc(4) += v * (a(4) * b(4)) with FMUL2/FFMA2
__device__ __forceinline__ void had_acc(float4& acc, float v, const float4& a, const float4& b) {
  unsigned long long h0, h1, a0 = u64of(acc.x, acc.y), a1 = u64of(acc.z, acc.w), vv = u64of(v, v);
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(h0) : "l"(u64of(a.x, a.y)), "l"(u64of(b.x, b.y)));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(h1) : "l"(u64of(a.z, a.w)), "l"(u64of(b.z, b.w)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(vv), "l"(h0));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a1) : "l"(vv), "l"(h1));
  split(a0, acc.x, acc.y); split(a1, acc.z, acc.w);
}
// acc(4) += a(4) * b(4)
__device__ __forceinline__ void fma4x2(float4& acc, const float4& a, const float4& b) {
  unsigned long long a0 = u64of(acc.x, acc.y), a1 = u64of(acc.z, acc.w);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(u64of(a.x, a.y)), "l"(u64of(b.x, b.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a1) : "l"(u64of(a.z, a.w)), "l"(u64of(b.z, b.w)));
  split(a0, acc.x, acc.y); split(a1, acc.z, acc.w);
}
// r(4) = v * w(4) + k * r(4)   (k = 0 or 1)
__device__ __forceinline__ void axpk(float4& r, float v, const float4& w, float k) {
  unsigned long long r0 = u64of(r.x, r.y), r1 = u64of(r.z, r.w), vv = u64of(v, v), kk = u64of(k, k);
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(r0) : "l"(kk));
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(r1) : "l"(kk));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r0) : "l"(vv), "l"(u64of(w.x, w.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r1) : "l"(vv), "l"(u64of(w.z, w.w)));
  split(r0, r.x, r.y); split(r1, r.z, r.w);
}

__device__ __forceinline__ void mbar_init(uint64_t* m, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(mb), "r"(parity)
      : "memory");
}

// One nonzero of the fibre-factored product, branch-free: at a fibre head (f != 0) fold the
// finished fibre (acc += run * u), restart run and load the new fibre's outer row into u from
// shared memory; then run += v * w.
__device__ __forceinline__ void fiber_step(uint32_t f, float v, const float4& w, uint32_t saddr, float4& acc,
                                           float4& run, float4& u) {
  asm volatile(
      "{ .reg .pred p; .reg .b64 a0, a1, r0, r1, u0, u1, w0, w1, vv;\n"
      "  setp.ne.b32 p, %12, 0;\n"
      "  mov.b64 a0, {%0, %1}; mov.b64 a1, {%2, %3};\n"
      "  mov.b64 r0, {%4, %5}; mov.b64 r1, {%6, %7};\n"
      "  mov.b64 u0, {%8, %9}; mov.b64 u1, {%10, %11};\n"
      "  mov.b64 w0, {%14, %15}; mov.b64 w1, {%16, %17}; mov.b64 vv, {%13, %13};\n"
      "  @p fma.rn.f32x2 a0, r0, u0, a0;\n"
      "  @p fma.rn.f32x2 a1, r1, u1, a1;\n"
      "  @p mov.b64 r0, 0; @p mov.b64 r1, 0;\n"
      "  @p ld.shared.v4.f32 {%8, %9, %10, %11}, [%18];\n"
      "  fma.rn.f32x2 r0, vv, w0, r0;\n"
      "  fma.rn.f32x2 r1, vv, w1, r1;\n"
      "  mov.b64 {%0, %1}, a0; mov.b64 {%2, %3}, a1;\n"
      "  mov.b64 {%4, %5}, r0; mov.b64 {%6, %7}, r1; }"
      : "+f"(acc.x), "+f"(acc.y), "+f"(acc.z), "+f"(acc.w), "+f"(run.x), "+f"(run.y), "+f"(run.z), "+f"(run.w),
        "+f"(u.x), "+f"(u.y), "+f"(u.z), "+f"(u.w)
      : "r"(f), "f"(v), "f"(w.x), "f"(w.y), "f"(w.z), "f"(w.w), "r"(saddr)
      : "memory");
}

constexpr int BW = 2 * 32 + 4;          // per stage: pk(32) val(32) bf ff pad(2)
constexpr int BSTRIDE = 2 * BW;         // 136 words: groups at bank offsets 0, 8, 16, 24

template <int POL>
__device__ __forceinline__ float4 ldgp(const void* p) {
  float4 r;
  if constexpr (POL == 0) r = __ldg(reinterpret_cast<const float4*>(p));
  else if constexpr (POL == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else if constexpr (POL == 2)
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else if constexpr (POL == 3)
    asm volatile("ld.global.nc.L1::evict_first.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

template <int G, int TB, int MINB, int FIBER, int POL = 0>
__global__ void __launch_bounds__(TB, MINB) k_blk(const PB P) {
  constexpr int R = 4 * G;
  extern __shared__ float4 sm[];
  __shared__ uint64_t mbar;
  const int item = blockIdx.x;
  const int b = P.item_blk[item];
  float* blk = reinterpret_cast<float*>(sm);
  uint32_t* stg_all = reinterpret_cast<uint32_t*>(blk + (size_t)P.BR * R);
  const int g = threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int nt = P.item_nt[item];
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int r0 = b * P.BR;
    const int nr = min(P.BR, P.Io - r0);
    bulk_g2s(blk, P.Uo + (size_t)r0 * R, (uint32_t)nr * R * 4u, &mbar);
  }
  const int64_t t = (int64_t)P.item_t0[item] + g;
  const bool live = g < nt;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  uint32_t* my = stg_all + g * BSTRIDE;
  const int col = gl * 4;
  const char* ubi = reinterpret_cast<const char*>(P.Ui + col);
  constexpr uint32_t rowb = R * 4u;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(blk) + col * 4;
  const uint32_t imask = (1u << P.IB) - 1u;
  const int IB = P.IB;

  const int64_t p0 = t * (int64_t)P.T;
  const int64_t pend = live ? min(p0 + (int64_t)P.T, P.blk_end[b]) : p0;
  const int nchunk = (int)((pend - p0) / 32);
  const bool left_open = live && !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = live ? P.seg_base[t] - 1u : 0u;
  uint32_t row = left_open ? P.seg_row[s] : 0u;
  float4 acc = make_float4(0, 0, 0, 0), run = acc, u = acc;

  auto issue = [&](int64_t pc, int st) {
    uint32_t* d = my + st * BW;
#pragma unroll
    for (int k = 0; k < (16 + G - 1) / G; ++k) {
      const int q = gl + k * G;
      if (q < 8) cp16(d + q * 4, P.pk + pc + q * 4);
      else if (q < 16) cp16(d + 32 + (q - 8) * 4, reinterpret_cast<const uint32_t*>(P.val) + pc + (q - 8) * 4);
    }
    if (gl == 0) cp4(d + 64, P.bf + (pc >> 5));
    if (gl == (1 % G)) cp4(d + 65, P.ff + (pc >> 5));
  };
  if (nchunk > 0) issue(p0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  mbar_wait(&mbar, 0);  // outer block resident
  auto flush = [&](float4 a) { red4(P.out + (size_t)row * R + col, a); };
  for (int ci = 0; ci < nchunk; ++ci) {
    if (ci + 1 < nchunk) issue(p0 + (int64_t)(ci + 1) * 32, (ci + 1) & 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp(gmask);
    const uint32_t* st = my + (ci & 1) * BW;
    const uint32_t bfw = st[64];
    uint32_t ffw = st[65];
    if (ci == 0) ffw |= 1u;
#pragma unroll
    for (int bi = 0; bi < 4; ++bi) {
      uint32_t pk[8], vb[8];
      {
        uint4 a0 = reinterpret_cast<const uint4*>(st + bi * 8)[0], a1 = reinterpret_cast<const uint4*>(st + bi * 8)[1];
        pk[0] = a0.x; pk[1] = a0.y; pk[2] = a0.z; pk[3] = a0.w; pk[4] = a1.x; pk[5] = a1.y; pk[6] = a1.z; pk[7] = a1.w;
        uint4 d0 = reinterpret_cast<const uint4*>(st + 32 + bi * 8)[0], d1 = reinterpret_cast<const uint4*>(st + 32 + bi * 8)[1];
        vb[0] = d0.x; vb[1] = d0.y; vb[2] = d0.z; vb[3] = d0.w; vb[4] = d1.x; vb[5] = d1.y; vb[6] = d1.z; vb[7] = d1.w;
      }
      const uint32_t heads = (bfw >> (bi * 8)) & 0xffu;
      const uint32_t fh = (ffw >> (bi * 8)) & 0xffu;
      float4 wi[8], wo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) wi[e] = ldgp<POL>(ubi + (size_t)(pk[e] & imask) * rowb);
      if constexpr (FIBER == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) wo[e] = lds4(sbase + (pk[e] >> IB) * rowb);
      } else if constexpr (FIBER == 2) {  // outer row loaded at fibre heads only
#pragma unroll
        for (int e = 0; e < 8; ++e) wo[e] = lds_if((fh >> e) & 1u, sbase + (pk[e] >> IB) * rowb, make_float4(0, 0, 0, 0));
#pragma unroll
        for (int e = 0; e < 8; ++e) { u = ((fh >> e) & 1u) ? wo[e] : u; wo[e] = u; }
      }
      const bool first = (ci == 0 && bi == 0);
      if (FIBER != 1 && heads == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) had_acc(acc, __uint_as_float(vb[e]), wo[e], wi[e]);
      } else if (FIBER == 1 && heads == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          fiber_step((fh >> e) & 1u, __uint_as_float(vb[e]), wi[e], sbase + (pk[e] >> IB) * rowb, acc, run, u);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool hd = (heads >> e) & 1u;
          if constexpr (FIBER == 1) {
            const uint32_t f = (fh >> e) & 1u;
            if (f) { fma4x2(acc, run, u); run = make_float4(0, 0, 0, 0); }  // fold before a segment flush
            if (hd && !(e == 0 && first)) flush(acc);
            if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
            fiber_step(f, __uint_as_float(vb[e]), wi[e], sbase + (pk[e] >> IB) * rowb, acc, run, u);
          } else {
            if (hd && !(e == 0 && first)) flush(acc);
            if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
            had_acc(acc, __uint_as_float(vb[e]), wo[e], wi[e]);
          }
        }
      }
    }
    __syncwarp(gmask);
  }
  if (!live) return;
  // ragged end of the block's last tile: one nonzero at a time
  for (int64_t p = p0 + (int64_t)nchunk * 32; p < pend; ++p) {
    const uint32_t hd = (P.bf[p >> 5] >> (p & 31)) & 1u;
    uint32_t f = (P.ff[p >> 5] >> (p & 31)) & 1u;
    if (p == p0) f = 1;
    const uint32_t k = P.pk[p];
    const float v = P.val[p];
    const float4 wi1 = __ldg(reinterpret_cast<const float4*>(ubi + (size_t)(k & imask) * rowb));
    const float4 wo1 = lds4(sbase + (k >> IB) * rowb);
    if constexpr (FIBER == 1) {
      if (f) fma4x2(acc, run, u);
      if (hd && p != p0) flush(acc);
      if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
      axpk(run, v, wi1, f ? 0.f : 1.f);
      u = f ? wo1 : u;
    } else {
      if (hd && p != p0) flush(acc);
      if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
      had_acc(acc, v, wo1, wi1);
    }
  }
  if constexpr (FIBER == 1) fma4x2(acc, run, u);
  flush(acc);
}

template <int G, int TB, int MINB, int FIBER>
static int launch_blk(const PB& P, int nitems, size_t smem, cudaStream_t s) {
  static int pol = getenv("PROTO_POL") ? atoi(getenv("PROTO_POL")) : 0;
  auto k = pol == 1 ? k_blk<G, TB, MINB, FIBER, 1> : pol == 2 ? k_blk<G, TB, MINB, FIBER, 2> : pol == 3 ? k_blk<G, TB, MINB, FIBER, 3>
         : pol == 4 ? k_blk<G, TB, MINB, FIBER, 4> : k_blk<G, TB, MINB, FIBER, 0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<nitems, TB, smem, s>>>(P);
  return (int)cudaGetLastError();
}

extern "C" int proto_blk(int fiber, int R, int tb, const PB* P, int nitems, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int G = R / 4;
  size_t smem = (size_t)P->BR * R * 4 + (size_t)(tb / G) * BSTRIDE * 4;
#define L(GG, TT, MB) return fiber == 1 ? launch_blk<GG, TT, MB, 1>(*P, nitems, smem, s) : fiber == 2 ? launch_blk<GG, TT, MB, 2>(*P, nitems, smem, s) : launch_blk<GG, TT, MB, 0>(*P, nitems, smem, s)
  if (tb == 256) {
    if (G == 4) L(4, 256, 2);
    if (G == 8) L(8, 256, 2);
    L(16, 256, 1);
  }
  if (G == 4) L(4, 512, 1);
  if (G == 8) L(8, 512, 1);
  L(16, 512, 1);
#undef L
}
extern "C" int proto_blk_sizeof() { return (int)sizeof(PB); }

// VAR 8: as VAR 5 (no fibre reuse), but the stream is loaded straight into registers: each lane of
// the group holds one 16-byte quarter... of the chunk's pk and val (lane gl: nonzeros 4gl..4gl+3 of
// an 8*G... ) and the words are broadcast within the group with SHFL.
template <int G, int TB, int MINB, int POL>
__global__ void __launch_bounds__(TB, MINB) k_blk2(const PB P) {
  constexpr int R = 4 * G;
  constexpr int CH = 4 * G;  // nonzeros per chunk: one uint4 per lane
  extern __shared__ float4 sm[];
  __shared__ uint64_t mbar;
  const int item = blockIdx.x;
  const int b = P.item_blk[item];
  float* blk = reinterpret_cast<float*>(sm);
  const int g = threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int nt = P.item_nt[item];
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int r0 = b * P.BR;
    const int nr = min(P.BR, P.Io - r0);
    bulk_g2s(blk, P.Uo + (size_t)r0 * R, (uint32_t)nr * R * 4u, &mbar);
  }
  const int64_t t = (int64_t)P.item_t0[item] + g;
  const bool live = g < nt;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int col = gl * 4;
  const char* ubi = reinterpret_cast<const char*>(P.Ui + col);
  constexpr uint32_t rowb = R * 4u;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(blk) + col * 4;
  const uint32_t imask = (1u << P.IB) - 1u;
  const int IB = P.IB;

  const int64_t p0 = t * (int64_t)P.T;
  const int64_t pend = live ? min(p0 + (int64_t)P.T, P.blk_end[b]) : p0;
  const int nchunk = (int)((pend - p0) / CH);
  const bool left_open = live && !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = live ? P.seg_base[t] - 1u : 0u;
  uint32_t row = left_open ? P.seg_row[s] : 0u;
  float4 acc = make_float4(0, 0, 0, 0);
  auto flush = [&](float4 a) { red4(P.out + (size_t)row * R + col, a); };
  // prefetch chunk 0
  uint4 kq = make_uint4(0, 0, 0, 0), vq = kq;
  uint32_t bq = 0;
  auto fetch = [&](int64_t pc, uint4& k, uint4& v, uint32_t& bw) {
    k = *reinterpret_cast<const uint4*>(P.pk + pc + 4 * gl);  // plain loads: L1::no_allocate via asm below
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(k.x), "=r"(k.y), "=r"(k.z), "=r"(k.w) : "l"(P.pk + pc + 4 * gl));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(reinterpret_cast<const uint32_t*>(P.val) + pc + 4 * gl));
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(bw) : "l"(P.bf + (pc >> 5) + (gl * 4) / 32));
  };
  if (nchunk > 0) fetch(p0, kq, vq, bq);
  mbar_wait(&mbar, 0);
  for (int ci = 0; ci < nchunk; ++ci) {
    const uint4 kc = kq, vc = vq;
    const uint32_t bc = bq;
    if (ci + 1 < nchunk) fetch(p0 + (int64_t)(ci + 1) * CH, kq, vq, bq);
#pragma unroll
    for (int bi = 0; bi < CH / 8; ++bi) {
      uint32_t pk[8], vb[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int q = bi * 8 + e;  // nonzero within the chunk: lane q/4, component q%4
        const uint32_t kk = (q % 4 == 0) ? kc.x : (q % 4 == 1) ? kc.y : (q % 4 == 2) ? kc.z : kc.w;
        const uint32_t vv = (q % 4 == 0) ? vc.x : (q % 4 == 1) ? vc.y : (q % 4 == 2) ? vc.z : vc.w;
        pk[e] = __shfl_sync(gmask, kk, q / 4, G);
        vb[e] = __shfl_sync(gmask, vv, q / 4, G);
      }
      // bf word covering nonzeros [bi*8, bi*8+8) of the chunk: held by lane (bi*8)/4 /... (word index (bi*8)/32)
      const uint32_t bw = __shfl_sync(gmask, bc, ((bi * 8) / 32) * 8 % G, G);
      const uint32_t heads = (bw >> ((p0 + (int64_t)ci * CH + bi * 8) & 31)) & 0xffu;
      float4 wi[8], wo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) wi[e] = ldgp<POL>(ubi + (size_t)(pk[e] & imask) * rowb);
#pragma unroll
      for (int e = 0; e < 8; ++e) wo[e] = lds4(sbase + (pk[e] >> IB) * rowb);
      const bool first = (ci == 0 && bi == 0);
      if (heads == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) had_acc(acc, __uint_as_float(vb[e]), wo[e], wi[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool hd = (heads >> e) & 1u;
          if (hd && !(e == 0 && first)) flush(acc);
          if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
          had_acc(acc, __uint_as_float(vb[e]), wo[e], wi[e]);
        }
      }
    }
  }
  if (!live) return;
  for (int64_t p = p0 + (int64_t)nchunk * CH; p < pend; ++p) {
    const uint32_t hd = (P.bf[p >> 5] >> (p & 31)) & 1u;
    const uint32_t k = P.pk[p];
    const float v = P.val[p];
    const float4 wi1 = __ldg(reinterpret_cast<const float4*>(ubi + (size_t)(k & imask) * rowb));
    const float4 wo1 = lds4(sbase + (k >> IB) * rowb);
    if (hd && p != p0) flush(acc);
    if (hd) { acc = make_float4(0, 0, 0, 0); ++s; row = P.seg_row[s]; }
    had_acc(acc, v, wo1, wi1);
  }
  flush(acc);
}

template <int G, int TB, int MINB>
static int launch_blk2(const PB& P, int nitems, size_t smem, cudaStream_t s) {
  auto k = k_blk2<G, TB, MINB, 2>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<nitems, TB, smem, s>>>(P);
  return (int)cudaGetLastError();
}
extern "C" int proto_blk2(int R, int tb, const PB* P, int nitems, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int G = R / 4;
  size_t smem = (size_t)P->BR * R * 4;
  if (tb == 256) {
    if (G == 4) return launch_blk2<4, 256, 3>(*P, nitems, smem, s);
    if (G == 8) return launch_blk2<8, 256, 2>(*P, nitems, smem, s);
    return launch_blk2<16, 256, 1>(*P, nitems, smem, s);
  }
  if (G == 4) return launch_blk2<4, 512, 1>(*P, nitems, smem, s);
  if (G == 8) return launch_blk2<8, 512, 1>(*P, nitems, smem, s);
  return launch_blk2<16, 512, 1>(*P, nitems, smem, s);
}
