// fcoo_engine.cu — the one-shot, flag-driven segmented-reduction engine (§IV-C/D)
// shared by SpMTTKRP (Eq.(6)) and SpTTM (Eq.(3)).
//
// Work decomposition: the nonzero stream is cut into tiles of T nonzeros
// (T = "threadlen", the sf granularity).  A lane-group of G lanes owns one tile; its
// lanes split the R columns (float4 per lane on the vector path), so a warp processes 32/G
// tiles side by side.  A group walks its tile in batches of 8 nonzeros: it loads 8 product
// indices per product mode and 8 values (128-bit loads, broadcast within the group), issues all
// factor-row gathers of the batch, then forms v * Hadamard(rows) and accumulates in registers.
// A set bf bit (segment head) closes the running segment: a segment that started inside the
// tile and ends inside it is STORED (no atomics, the common case); the at most two segments a
// tile shares with its neighbours (left-open when sf[t] == 0, right-open when sf[t+1] == 0) are
// combined with red.global.add.v4.f32 — "boundary-only atomics" (north_star).
// This replaces the paper's Titan-X adjacent-synchronisation carry chain.
#pragma once
#include <stdlib.h>

#include <type_traits>

#include "fcoo_engine.cuh"

namespace fcoo {

// Streaming loads of the read-once F-COO arrays: read-only path, no L1 allocation (L1 is kept
// for the gathered factor rows, "read-only data cache").
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream8(const void* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream4(const void* p) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// B consecutive 32-bit words starting at a B*4-byte aligned address.
template <int B>
__device__ __forceinline__ void ld_batch(const void* p, uint32_t (&w)[B]) {
  if constexpr (B == 8) {
    uint4 lo = ld_stream16(p), hi = ld_stream16(reinterpret_cast<const uint32_t*>(p) + 4);
    w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w; w[4] = hi.x; w[5] = hi.y; w[6] = hi.z; w[7] = hi.w;
  } else if constexpr (B == 4) {
    uint4 q = ld_stream16(p);
    w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
  } else if constexpr (B == 2) {
    uint2 q = ld_stream8(p);
    w[0] = q.x; w[1] = q.y;
  } else {
    w[0] = ld_stream4(p);
  }
}

// Nonzeros per batch: keep the batch's gathered rows within ~64 registers.
template <int NP, int VEC, int CPL>
constexpr int batch_size() {
  constexpr int regs = NP * VEC * CPL;
  return regs * 8 <= 64 ? 8 : regs * 4 <= 64 ? 4 : regs * 2 <= 64 ? 2 : 1;
}

__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Predicated segment flushes (no branch): store when the segment is owned by the tile, red.add when
// it is shared with a neighbour tile; a false predicate issues nothing to memory.
__device__ __forceinline__ void flush_if(bool st, bool rd, float* p, float4 v) {
  asm volatile(
      "{ .reg .pred ps, pr; setp.ne.b32 ps, %0, 0; setp.ne.b32 pr, %1, 0;\n"
      "  @ps st.global.v4.f32 [%2], {%3,%4,%5,%6};\n"
      "  @pr red.global.add.v4.f32 [%2], {%3,%4,%5,%6}; }" ::"r"((int)st),
      "r"((int)rd), "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}
__device__ __forceinline__ void flush_if(bool st, bool rd, float* p, float v) {
  asm volatile(
      "{ .reg .pred ps, pr; setp.ne.b32 ps, %0, 0; setp.ne.b32 pr, %1, 0;\n"
      "  @ps st.global.f32 [%2], %3;\n"
      "  @pr red.global.add.f32 [%2], %3; }" ::"r"((int)st),
      "r"((int)rd), "l"(p), "f"(v)
      : "memory");
}
// The same flushes through an NVLS multicast address (fused combine across ranks): a store
// reaches every rank's copy, a red.add is reduced in the NVSwitch and lands in every copy.
__device__ __forceinline__ void mc_flush_if(bool st, bool rd, float* p, float4 v) {
  asm volatile(
      "{ .reg .pred ps, pr; setp.ne.b32 ps, %0, 0; setp.ne.b32 pr, %1, 0;\n"
      "  @ps multimem.st.relaxed.sys.global.v4.f32 [%2], {%3,%4,%5,%6};\n"
      "  @pr multimem.red.relaxed.sys.global.add.v4.f32 [%2], {%3,%4,%5,%6}; }" ::"r"((int)st),
      "r"((int)rd), "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}
__device__ __forceinline__ float4 zero_if(bool z, float4 a) {
  return z ? make_float4(0.f, 0.f, 0.f, 0.f) : a;
}
__device__ __forceinline__ float zero_if(bool z, float a) { return z ? 0.f : a; }
// Deterministic handles: the shared-segment flush goes to the tile's partial slot (plain store)
__device__ __forceinline__ void store2_if(bool s0, float* p0, bool s1, float* p1, float4 v) {
  asm volatile(
      "{ .reg .pred ps, pr; setp.ne.b32 ps, %0, 0; setp.ne.b32 pr, %1, 0;\n"
      "  @ps st.global.v4.f32 [%2], {%4,%5,%6,%7};\n"
      "  @pr st.global.v4.f32 [%3], {%4,%5,%6,%7}; }" ::"r"((int)s0),
      "r"((int)s1), "l"(p0), "l"(p1), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}
__device__ __forceinline__ void store2_if(bool s0, float* p0, bool s1, float* p1, float v) {
  asm volatile(
      "{ .reg .pred ps, pr; setp.ne.b32 ps, %0, 0; setp.ne.b32 pr, %1, 0;\n"
      "  @ps st.global.f32 [%2], %4;\n"
      "  @pr st.global.f32 [%3], %4; }" ::"r"((int)s0),
      "r"((int)s1), "l"(p0), "l"(p1), "f"(v)
      : "memory");
}

// Accumulation-chain cap (DESIGN.md §2 Q16): a lane-group's fp32 partial of a segment is folded
// into a second register set every kChainChunks x 32 = 256 nonzeros (chain_fold), and the two are
// re-joined before any flush (chain_absorb), so no sequential fp32 chain inside a tile is longer
// than 256 + T/256 + 8 additions: per-element error <= (264 + T/256 + k) u * sum|contributions|
// for a segment split over k tiles (u = 2^-24).  fp64 accumulators (CP fit mode) need no cap.
constexpr int kChainChunks = 8;
__device__ __forceinline__ void chain_fold(float4& hi, float4& acc) {
  hi = make_float4(hi.x + acc.x, hi.y + acc.y, hi.z + acc.z, hi.w + acc.w);
  acc = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void chain_absorb(float4& acc, float4& hi) {
  acc = make_float4(acc.x + hi.x, acc.y + hi.y, acc.z + hi.z, acc.w + hi.w);
  hi = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void chain_fold(float& hi, float& acc) { hi += acc; acc = 0.f; }
__device__ __forceinline__ void chain_absorb(float& acc, float& hi) { acc += hi; hi = 0.f; }
template <class T>
__device__ __forceinline__ void chain_fold(T&, T&) {}
template <class T>
__device__ __forceinline__ void chain_absorb(T&, T&) {}

// Per-lane column slot: VEC consecutive fp32 factor entries (float4 on the vector path) and an
// accumulator of type ACC (fp32 for the product path; fp64 for the CP-ALS fit mode, where the
// identity-based fit needs the inner product <X, Xhat> to ~1e-12).
template <int VEC>
struct Ld;
template <>
struct Ld<4> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  static __device__ __forceinline__ T load(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
};
template <>
struct Ld<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.f; }
  static __device__ __forceinline__ T load(const float* p) { return __ldg(p); }
};

// fp64 accumulator (CP fit mode).  Products are formed in fp64 (exact for two fp32 factors)
// because the fit identity needs <X, Xhat> to ~1e-10 relative near fit = 1: an fp32 product
// rounding (2^-24 per term) left a ~1e-4 jitter in the fit of small converged problems.
struct d4 {
  double x, y, z, w;
};
struct d1 {
  double x;
};

template <int VEC, class ACC>
struct Acc;
template <>
struct Acc<4, float> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  template <int NP>
  static __device__ __forceinline__ void add(T& acc, float v, const float4 (&r)[NP]) {
    float4 h = r[0];
#pragma unroll
    for (int a = 1; a < NP; ++a) h = make_float4(h.x * r[a].x, h.y * r[a].y, h.z * r[a].z, h.w * r[a].w);
    acc = make_float4(fmaf(v, h.x, acc.x), fmaf(v, h.y, acc.y), fmaf(v, h.z, acc.z), fmaf(v, h.w, acc.w));
  }
  template <int NP>
  static __device__ __forceinline__ void add_inner(T& t, float v, const float4 (&r)[NP]) {  // t += v*prod_{a>=1} r[a]
    float4 h = r[1];
#pragma unroll
    for (int a = 2; a < NP; ++a) h = make_float4(h.x * r[a].x, h.y * r[a].y, h.z * r[a].z, h.w * r[a].w);
    t = make_float4(fmaf(v, h.x, t.x), fmaf(v, h.y, t.y), fmaf(v, h.z, t.z), fmaf(v, h.w, t.w));
  }
  static __device__ __forceinline__ void fold(T& acc, const T& t, float4 r0) {  // acc += t * r0
    acc = make_float4(fmaf(t.x, r0.x, acc.x), fmaf(t.y, r0.y, acc.y), fmaf(t.z, r0.z, acc.z), fmaf(t.w, r0.w, acc.w));
  }
  static __device__ __forceinline__ void store(float* p, T v) { *reinterpret_cast<float4*>(p) = v; }
  static __device__ __forceinline__ void red(float* p, T v) { red_add_v4(p, v); }
};
template <>
struct Acc<1, float> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.f; }
  template <int NP>
  static __device__ __forceinline__ void add(T& acc, float v, const float (&r)[NP]) {
    float h = r[0];
#pragma unroll
    for (int a = 1; a < NP; ++a) h *= r[a];
    acc = fmaf(v, h, acc);
  }
  template <int NP>
  static __device__ __forceinline__ void add_inner(T& t, float v, const float (&r)[NP]) {
    float h = r[1];
#pragma unroll
    for (int a = 2; a < NP; ++a) h *= r[a];
    t = fmaf(v, h, t);
  }
  static __device__ __forceinline__ void fold(T& acc, const T& t, float r0) { acc = fmaf(t, r0, acc); }
  static __device__ __forceinline__ void store(float* p, T v) { *p = v; }
  static __device__ __forceinline__ void red(float* p, T v) { atomicAdd(p, v); }
};
template <>
struct Acc<4, double> {
  using T = d4;
  static __device__ __forceinline__ T zero() { return d4{0.0, 0.0, 0.0, 0.0}; }
  template <int NP>
  static __device__ __forceinline__ void add(T& acc, float v, const float4 (&r)[NP]) {
    // products in fp64: r0*r1 of two fp32 values is exact, v*(r0*r1) rounds once at 2^-53
    double hx = r[0].x, hy = r[0].y, hz = r[0].z, hw = r[0].w;
#pragma unroll
    for (int a = 1; a < NP; ++a) { hx *= (double)r[a].x; hy *= (double)r[a].y; hz *= (double)r[a].z; hw *= (double)r[a].w; }
    const double dv = v;
    acc.x = fma(dv, hx, acc.x); acc.y = fma(dv, hy, acc.y); acc.z = fma(dv, hz, acc.z); acc.w = fma(dv, hw, acc.w);
  }
  template <int NP>
  static __device__ __forceinline__ void add_inner(T& t, float v, const float4 (&r)[NP]) {
    double hx = r[1].x, hy = r[1].y, hz = r[1].z, hw = r[1].w;
#pragma unroll
    for (int a = 2; a < NP; ++a) { hx *= (double)r[a].x; hy *= (double)r[a].y; hz *= (double)r[a].z; hw *= (double)r[a].w; }
    double dv = v;
    t.x = fma(dv, hx, t.x); t.y = fma(dv, hy, t.y); t.z = fma(dv, hz, t.z); t.w = fma(dv, hw, t.w);
  }
  static __device__ __forceinline__ void fold(T& acc, const T& t, float4 r0) {
    acc.x = fma(t.x, (double)r0.x, acc.x); acc.y = fma(t.y, (double)r0.y, acc.y);
    acc.z = fma(t.z, (double)r0.z, acc.z); acc.w = fma(t.w, (double)r0.w, acc.w);
  }
  static __device__ __forceinline__ void store(double* p, T v) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v.x, v.y);
    reinterpret_cast<double2*>(p)[1] = make_double2(v.z, v.w);
  }
  static __device__ __forceinline__ void red(double* p, T v) {
    atomicAdd(p, v.x); atomicAdd(p + 1, v.y); atomicAdd(p + 2, v.z); atomicAdd(p + 3, v.w);
  }
};
template <>
struct Acc<1, double> {
  using T = d1;
  static __device__ __forceinline__ T zero() { return d1{0.0}; }
  template <int NP>
  static __device__ __forceinline__ void add(T& acc, float v, const float (&r)[NP]) {
    double h = r[0];
#pragma unroll
    for (int a = 1; a < NP; ++a) h *= (double)r[a];
    acc.x = fma((double)v, h, acc.x);
  }
  template <int NP>
  static __device__ __forceinline__ void add_inner(T& t, float v, const float (&r)[NP]) {
    double h = r[1];
#pragma unroll
    for (int a = 2; a < NP; ++a) h *= (double)r[a];
    t.x = fma((double)v, h, t.x);
  }
  static __device__ __forceinline__ void fold(T& acc, const T& t, float r0) { acc.x = fma(t.x, (double)r0, acc.x); }
  static __device__ __forceinline__ void store(double* p, T v) {
    *p = v.x;
  }
  static __device__ __forceinline__ void red(double* p, T v) {
    atomicAdd(p, v.x);
  }
};

// NP product modes; G lanes per group (divides 32); VEC floats per lane per column slot;
// CPL column slots per lane (lane gl covers columns (gl + G*c)*VEC .. +VEC-1, c < CPL);
// FULL: every lane's every slot is a valid column (R == G*VEC*CPL), so no column guards.
//
// Per batch of B nonzeros the group (1) loads B indices per product mode and B values with
// 128-bit streaming loads, (2) issues all B*NP factor-row gathers of the batch back to back
// (LDG.128, one IMAD.WIDE each from a hoisted per-lane base pointer; a row whose index repeats
// the previous nonzero's — common under the Q5 product order — is an L1 hit or merges with the
// in-flight miss, so it costs no L2 bandwidth), then (3) accumulates v * Hadamard(rows).
// Segment heads are tested once per batch; only batches that contain a head take the
// per-nonzero path that closes and opens segments.
template <int NP, int G, int VEC, int CPL, class ACC, bool FULL>
__global__ void __launch_bounds__(256) k_segreduce(const EngineParams P) {
  using V = Ld<VEC>;
  using VT = typename V::T;
  using A = Acc<VEC, ACC>;
  using AT = typename A::T;
  constexpr int B = batch_size<NP, VEC, CPL>();  // nonzeros per batch (divides 32)
  const int gl = threadIdx.x % G;
  const int64_t t = P.tile_begin + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if (t >= P.tile_end || gated_off(P)) return;  // groups are lane-aligned: whole groups exit together

  const int R = P.R;
  const uint32_t rowb = (uint32_t)R * 4u;  // factor row stride in bytes
  int col[CPL];
  bool cok[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    col[c] = (gl + G * c) * VEC;
    cok[c] = FULL || col[c] < R;
  }
  // per-lane base pointers: factor a, column slot c
  const char* ub[NP][CPL];
#pragma unroll
  for (int a = 0; a < NP; ++a)
#pragma unroll
    for (int c = 0; c < CPL; ++c) ub[a][c] = reinterpret_cast<const char*>(P.U[a] + (cok[c] ? col[c] : 0));

  const int64_t p0 = t * (int64_t)P.T;
  const int64_t p1 = min(p0 + (int64_t)P.T, P.nnz);
  const int64_t pfull = p0 + ((p1 - p0) / B) * B;  // == p1 except in the tensor's last tile

  const bool left_open = !((P.sf[t >> 5] >> (t & 31)) & 1u);
  int64_t s = (int64_t)P.seg_base[t] - 1;  // current segment ordinal (incremented at each head)
  int64_t row = 0;
  if (left_open) row = P.seg_coord ? (int64_t)P.seg_coord[s] : s;
  bool own = false;  // did the current segment start inside this tile?

  AT acc[CPL], hi[CPL];  // hi: the chain-capped part of the running segment (chain_fold)
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = hi[c] = A::zero();
  auto flush = [&](bool store) {
    ACC* o = reinterpret_cast<ACC*>(P.out) + row * (int64_t)R;
    // deterministic handles: a shared segment goes to the tile's partial slot (0: left-open first
    // segment, 1: own right-open last segment), combined later in tile order
    ACC* dp = P.dpart ? reinterpret_cast<ACC*>(P.dpart) + ((size_t)t * 2 + (own ? 1 : 0)) * (uint32_t)R : nullptr;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (cok[c]) {
        if (store) A::store(o + col[c], acc[c]);
        else if (dp) A::store(dp + col[c], acc[c]);
        else A::red(o + col[c], acc[c]);
      }
  };
  auto open_segment = [&](int64_t p) {
    if (p != p0) flush(own);
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = A::zero();
    own = true;
    ++s;
    row = P.seg_coord ? (int64_t)P.seg_coord[s] : s;
  };

  uint32_t bfw = 0;
  for (int64_t pb = p0; pb < pfull; pb += B) {
    if (((pb - p0) & 31) == 0) bfw = ld_stream4(P.bf + (pb >> 5));
    uint32_t ix[NP][B];
    uint32_t vb[B];
#pragma unroll
    for (int a = 0; a < NP; ++a) ld_batch<B>(P.pidx[a] + pb, ix[a]);
    ld_batch<B>(P.val + pb, vb);
    const uint32_t heads = (bfw >> ((pb - p0) & 31)) & ((1u << B) - 1u);
    VT r[B][CPL][NP];
#pragma unroll
    for (int e = 0; e < B; ++e)
#pragma unroll
      for (int a = 0; a < NP; ++a)
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          r[e][c][a] = cok[c] ? V::load(reinterpret_cast<const float*>(ub[a][c] + (size_t)ix[a][e] * rowb)) : V::zero();
    if (heads == 0) {
#pragma unroll
      for (int e = 0; e < B; ++e)
#pragma unroll
        for (int c = 0; c < CPL; ++c) A::template add<NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) chain_absorb(acc[c], hi[c]);
#pragma unroll
      for (int e = 0; e < B; ++e) {
        if ((heads >> e) & 1u) open_segment(pb + e);
#pragma unroll
        for (int c = 0; c < CPL; ++c) A::template add<NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
      }
    }
    if (((pb - p0 + B) & (kChainChunks * 32 - 1)) == 0) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) chain_fold(hi[c], acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) chain_absorb(acc[c], hi[c]);
  // ragged tail of the tensor's last tile: one nonzero at a time
  for (int64_t p = pfull; p < p1; ++p) {
    if ((p & 31) == 0 || p == pfull) bfw = ld_stream4(P.bf + (p >> 5));
    if ((bfw >> (p & 31)) & 1u) open_segment(p);
    const float v = __uint_as_float(ld_stream4(P.val + p));
    VT r1[CPL][NP];
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      uint32_t i = ld_stream4(P.pidx[a] + p);
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        r1[c][a] = cok[c] ? V::load(reinterpret_cast<const float*>(ub[a][c] + (size_t)i * rowb)) : V::zero();
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) A::template add<NP>(acc[c], v, r1[c]);
  }
  const bool right_open = (t + 1 < P.ntiles) && !((P.sf[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u);
  flush(own && !right_open);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// B consecutive words from shared memory (broadcast within the group).
template <int B>
__device__ __forceinline__ void lds_batch(const uint32_t* p, uint32_t (&w)[B]) {
  static_assert(B == 1 || B == 2 || B == 4 || B % 4 == 0, "batch of 1, 2 or a multiple of 4 words");
  if constexpr (B > 8) {
#pragma unroll
    for (int k = 0; k < B / 4; ++k) {
      const uint4 q = reinterpret_cast<const uint4*>(p)[k];
      w[4 * k] = q.x; w[4 * k + 1] = q.y; w[4 * k + 2] = q.z; w[4 * k + 3] = q.w;
    }
  } else if constexpr (B == 8) {
    uint4 lo = reinterpret_cast<const uint4*>(p)[0], hi = reinterpret_cast<const uint4*>(p)[1];
    w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w; w[4] = hi.x; w[5] = hi.y; w[6] = hi.z; w[7] = hi.w;
  } else if constexpr (B == 4) {
    uint4 q = reinterpret_cast<const uint4*>(p)[0];
    w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
  } else if constexpr (B == 2) {
    uint2 q = reinterpret_cast<const uint2*>(p)[0];
    w[0] = q.x; w[1] = q.y;
  } else {
    w[0] = p[0];
  }
}

// Shared-memory staging geometry of k_segreduce_staged: per lane-group, NST stages of one
// 32-nonzero chunk each: NP index rows + the values + the bf word (16-byte padded); the
// per-group stride is padded to 4 (mod 32) words so the groups of a warp hit distinct banks.
template <int NP>
struct Stage {
  static constexpr int CH = 32;
  static constexpr int NST = 2;
  static constexpr int WORDS = (NP + 1) * CH + 4;
  static constexpr int STRIDE_RAW = NST * WORDS;
  static constexpr int STRIDE = STRIDE_RAW + ((4 - STRIDE_RAW % 32) + 32) % 32;
};

// Staged variant: the same segmented reduction, with the nonzero stream (indices, values, bf)
// double-buffered through shared memory by cp.async (LDGSTS) one 32-nonzero chunk ahead, so the
// HBM latency of the stream is off the critical path; only the L2-resident factor gathers remain
// exposed.  This is the "shared-memory staging of the nonzero stream" of the north star; the
// factor rows still go through L1 (most of the unified carveout stays L1).
template <int NP, int G, int VEC, int CPL, class ACC, bool FULL, bool DET>
__global__ void __launch_bounds__(256) k_segreduce_staged(const EngineParams P) {
  using V = Ld<VEC>;
  using VT = typename V::T;
  using A = Acc<VEC, ACC>;
  using AT = typename A::T;
  using S = Stage<NP>;
  constexpr int B = batch_size<NP, VEC, CPL>();
  constexpr int CH = S::CH;
  extern __shared__ uint4 smem_raw[];
  const int lane = threadIdx.x & 31;
  const int gl = threadIdx.x % G;
  const int64_t t = P.tile_begin + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  if (t >= P.tile_end || gated_off(P)) return;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  uint32_t* my = reinterpret_cast<uint32_t*>(smem_raw) + (threadIdx.x / G) * S::STRIDE;

  const int R = P.R;
  const uint32_t rowb = (uint32_t)R * 4u;
  int col[CPL];
  bool cok[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    col[c] = (gl + G * c) * VEC;
    cok[c] = FULL || col[c] < R;
  }
  const char* ub[NP][CPL];
#pragma unroll
  for (int a = 0; a < NP; ++a)
#pragma unroll
    for (int c = 0; c < CPL; ++c) ub[a][c] = reinterpret_cast<const char*>(P.U[a] + (cok[c] ? col[c] : 0));

  const int64_t p0 = t * (int64_t)P.T;
  const int64_t p1 = min(p0 + (int64_t)P.T, P.nnz);
  const int nchunk = (int)((p1 - p0) / CH);  // full chunks (all of them except in the last tile)

  const bool left_open = !((P.sf[t >> 5] >> (t & 31)) & 1u);
  // segment ordinal and output row in 32 bits (nsegs and every extent are < 2^32); s wraps to
  // 0xffffffff before the first head of tile 0 and is never used as a row there
  uint32_t s = P.seg_base[t] - 1u;
  uint32_t row = 0;
  if (left_open) row = P.seg_coord ? P.seg_coord[s] : s;
  bool own = false;
  ACC* const outp = reinterpret_cast<ACC*>(P.out);

  AT acc[CPL], hi[CPL];  // hi: the chain-capped part of the running segment (chain_fold)
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = hi[c] = A::zero();
  float* const mcp = NP >= 2 ? P.out_mc : nullptr;  // fused combine (float4 fp32, order >= 3; host checks)
  // deterministic handles, branch-free path: the only shared flush there is the left-open segment,
  // to slot 0 of this tile (address formed at the flush from the kernel parameter)
  auto dpt0 = [&]() { return reinterpret_cast<ACC*>(P.dpart) + (size_t)t * 2 * (uint32_t)R; };
  auto flush = [&](bool store) {
    ACC* o = outp + (size_t)row * (uint32_t)R;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (cok[c]) {
        if constexpr (DET) {  // deterministic handle: shared segment -> the tile's partial slot
          if (!store) {
            A::store(reinterpret_cast<ACC*>(P.dpart) + ((size_t)t * 2 + (own ? 1 : 0)) * (uint32_t)R + col[c], acc[c]);
            continue;
          }
        }
        if constexpr (std::is_same<AT, float4>::value && NP >= 2) {  // MTTKRP of order >= 3
          if (mcp) {
            mc_flush_if(store, !store, mcp + (size_t)row * (uint32_t)R + col[c], acc[c]);
            continue;
          }
        }
        if (store) A::store(o + col[c], acc[c]);
        else A::red(o + col[c], acc[c]);
      }
  };
  auto open_segment = [&](int64_t p) {
    if (p != p0) flush(own);
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = A::zero();
    own = true;
    ++s;
    row = P.seg_coord ? P.seg_coord[s] : s;
  };
  auto issue = [&](int64_t pc, int st) {  // group-cooperative copy of chunk [pc, pc+32) into stage st
    uint32_t* dst = my + st * S::WORDS;
#pragma unroll
    for (int a = 0; a <= NP; ++a) {
      const uint32_t* base = a < NP ? P.pidx[a] : reinterpret_cast<const uint32_t*>(P.val);
#pragma unroll
      for (int k = 0; k < (8 + G - 1) / G; ++k) {
        const int q = gl + k * G;
        if (q < 8) cp_async16(dst + a * CH + q * 4, base + pc + q * 4);
      }
    }
    if (gl == 0) cp_async4(dst + (NP + 1) * CH, P.bf + (pc >> 5));
  };

  if (nchunk > 0) issue(p0, 0);
  cp_async_commit();
  for (int ci = 0; ci < nchunk; ++ci) {
    if (ci + 1 < nchunk) issue(p0 + (int64_t)(ci + 1) * CH, (ci + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp(gmask);
    const uint32_t* stg = my + (ci & 1) * S::WORDS;
    const uint32_t bfw = stg[(NP + 1) * CH];
#pragma unroll
    for (int bi = 0; bi < CH / B; ++bi) {
      const int64_t pb = p0 + (int64_t)ci * CH + bi * B;
      uint32_t ix[NP][B];
      uint32_t vb[B];
#pragma unroll
      for (int a = 0; a < NP; ++a) lds_batch<B>(stg + a * CH + bi * B, ix[a]);
      lds_batch<B>(stg + NP * CH + bi * B, vb);
      const uint32_t heads = (bfw >> (bi * B)) & ((1u << B) - 1u);
      VT r[B][CPL][NP];
#pragma unroll
      for (int e = 0; e < B; ++e)
#pragma unroll
        for (int a = 0; a < NP; ++a)
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const float* gp = reinterpret_cast<const float*>(ub[a][c] + (size_t)ix[a][e] * rowb);
            r[e][c][a] = !cok[c] ? V::zero() : V::load(gp);
          }
      if (heads == 0) {
#pragma unroll
        for (int e = 0; e < B; ++e)
#pragma unroll
          for (int c = 0; c < CPL; ++c) A::template add<NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
      } else if constexpr (std::is_same<ACC, float>::value) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) chain_absorb(acc[c], hi[c]);
        // branch-free segment handling (short segments, e.g. SpTTM fibres): at a head the running
        // segment is flushed by a predicated store (owned) or red.add (shared with the left tile),
        // the accumulator is reset by select and the segment ordinal advances by the head bit
        const bool first = (ci == 0 && bi == 0);  // the tile's first nonzero opens, never closes
        // FM: 0 = store / red.add, 1 = store / tile partial (deterministic handle), 2 = multicast
        // (fused combine); chosen once per batch so the per-nonzero path carries no extra branch
        auto headed = [&](auto fm_tag) {
          constexpr int FM = decltype(fm_tag)::value;
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const bool hd = (heads >> e) & 1u;
            const bool cl = hd && (e != 0 || !first);
            ACC* o = outp + (size_t)row * (uint32_t)R;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
              if (cok[c]) {
                if constexpr (FM == 2) {
                  if constexpr (std::is_same<AT, float4>::value && NP >= 2)
                    mc_flush_if(cl && own, cl && !own, mcp + (size_t)row * (uint32_t)R + col[c], acc[c]);
                } else if constexpr (FM == 1) {
                  store2_if(cl && own, o + col[c], cl && !own, dpt0() + col[c], acc[c]);
                } else {
                  flush_if(cl && own, cl && !own, o + col[c], acc[c]);
                }
              }
              acc[c] = zero_if(hd, acc[c]);
            }
            own = own || hd;
            s += hd ? 1u : 0u;
            if (hd) row = P.seg_coord ? P.seg_coord[s] : s;
#pragma unroll
            for (int c = 0; c < CPL; ++c) A::template add<NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
          }
        };
        if constexpr (DET) {
          headed(std::integral_constant<int, 1>{});
        } else {
          if (mcp) headed(std::integral_constant<int, 2>{});
          else headed(std::integral_constant<int, 0>{});
        }
      } else {
#pragma unroll
        for (int e = 0; e < B; ++e) {
          if ((heads >> e) & 1u) open_segment(pb + e);
#pragma unroll
          for (int c = 0; c < CPL; ++c) A::template add<NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
        }
      }
    }
    if (ci % kChainChunks == kChainChunks - 1) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) chain_fold(hi[c], acc[c]);
    }
    __syncwarp(gmask);  // every lane is done with this stage before it is refilled
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) chain_absorb(acc[c], hi[c]);
  uint32_t bfw = 0;
  for (int64_t p = p0 + (int64_t)nchunk * CH; p < p1; ++p) {  // ragged tail of the last tile
    if ((p & 31) == 0 || p == p0 + (int64_t)nchunk * CH) bfw = ld_stream4(P.bf + (p >> 5));
    if ((bfw >> (p & 31)) & 1u) open_segment(p);
    const float v = __uint_as_float(ld_stream4(P.val + p));
    VT r1[CPL][NP];
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      uint32_t i = ld_stream4(P.pidx[a] + p);
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        r1[c][a] = cok[c] ? V::load(reinterpret_cast<const float*>(ub[a][c] + (size_t)i * rowb)) : V::zero();
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      A::template add<NP>(acc[c], v, r1[c]);
    }
  }
  const bool right_open = (t + 1 < P.ntiles) && !((P.sf[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u);
  flush(own && !right_open);
  if (mcp) __threadfence_system();  // multicast writes visible system-wide before the kernel ends
}

// CTAs per SM the staged kernel's shared-memory carveout is sized for: the register-limited count
// (64K registers / (regs x 256 threads), at most 4), so shared memory never lowers occupancy and
// the rest of the unified 228 KB stays L1 for the factor rows.  Measured: SpTTM (NP=1, 70 regs)
// 2 -> 3 CTAs is 10-15% faster on brainq; MTTKRP (>= 94 regs) stays at 2.
inline int staged_ctas_per_sm(const void* kern) {
  cudaFuncAttributes fa;
  int v = 2;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && fa.numRegs > 0) v = 65536 / (fa.numRegs * 256);
  return v < 1 ? 1 : v > 4 ? 4 : v;
}

// The staged kernel (stream through shared memory) when a lane-group has >= 4 lanes, else the
// plain one (tiny ranks: per-lane staging would not pay).
template <int NP, int G, int VEC, int CPL, class ACC>
cudaError_t launch_one(const EngineParams& P, cudaStream_t s) {
  const bool full = (P.R == G * VEC * CPL);
  const bool staged = G >= 4;
  const int TB = 256;
  void (*kern)(const EngineParams);
  size_t smem = 0;
  if (staged) {
    if (P.dpart)
      kern = full ? k_segreduce_staged<NP, G, VEC, CPL, ACC, true, true> : k_segreduce_staged<NP, G, VEC, CPL, ACC, false, true>;
    else
      kern = full ? k_segreduce_staged<NP, G, VEC, CPL, ACC, true, false> : k_segreduce_staged<NP, G, VEC, CPL, ACC, false, false>;
    smem = sizeof(uint32_t) * (size_t)(TB / G) * Stage<NP>::STRIDE;
  } else {
    kern = full ? k_segreduce<NP, G, VEC, CPL, ACC, true> : k_segreduce<NP, G, VEC, CPL, ACC, false>;
  }
  static bool configured[2][2][2] = {};  // [full][staged][deterministic]: one entry per kernel
  const int di = (staged && P.dpart) ? 1 : 0;
  if (!configured[full][staged][di]) {
    if (staged) {  // small staging buffers: ask for just enough carveout, keep the rest as L1
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int ctas = staged_ctas_per_sm(reinterpret_cast<const void*>(kern));
      int pct = (int)((ctas * smem * 100 + 228 * 1024 - 1) / (228 * 1024)) + 1;
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
    } else {  // no shared memory: give the whole unified carveout to L1 (factor rows)
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    }
    configured[full][staged][di] = true;
  }
  int64_t groups = P.tile_end - P.tile_begin;
  int64_t threads = groups * G;
  unsigned blocks = (unsigned)((threads + TB - 1) / TB);
  if (blocks == 0) return cudaSuccess;
  kern<<<blocks, TB, smem, s>>>(P);
  count_launch();
  return cudaGetLastError();
}

template <int NP, int VEC, int CPL, class ACC>
cudaError_t launch_g(const EngineParams& P, int G, cudaStream_t s) {
  switch (G) {
    case 1: return launch_one<NP, 1, VEC, CPL, ACC>(P, s);
    case 2: return launch_one<NP, 2, VEC, CPL, ACC>(P, s);
    case 4: return launch_one<NP, 4, VEC, CPL, ACC>(P, s);
    case 8: return launch_one<NP, 8, VEC, CPL, ACC>(P, s);
    case 16: return launch_one<NP, 16, VEC, CPL, ACC>(P, s);
    default: return launch_one<NP, 32, VEC, CPL, ACC>(P, s);
  }
}

template <int NP, class ACC>
cudaError_t launch_np(const EngineParams& P, bool vec_ok, cudaStream_t s) {
  const int R = P.R;
  if (vec_ok) {  // float4 per lane: G = next pow2 of R/4 (<= 32)
    int q = R / 4, G = 1;
    while (G < q) G <<= 1;
    return launch_g<NP, 4, 1, ACC>(P, G, s);
  }
  if (R <= 32) {
    int G = 1;
    while (G < R) G <<= 1;
    return launch_g<NP, 1, 1, ACC>(P, G, s);
  }
  int cpl = (R + 31) / 32;
  if (cpl <= 2) return launch_one<NP, 32, 1, 2, ACC>(P, s);
  if (cpl <= 4) return launch_one<NP, 32, 1, 4, ACC>(P, s);
  return launch_one<NP, 32, 1, 8, ACC>(P, s);
}

}  // namespace fcoo
