// fcoo_blocked_kernels.cuh — SpMTTKRP on a BLOCKED F-COO handle (FCOO_BUILD_BLOCKED).
//
// The stream is the concatenation over b of the F-COO of X_b = {nonzeros with floor(i_outer/BR)
// == b} (outer = first product mode of reading Q5), each block padded to a multiple of T.  By
// linearity of Eq.(6), M = sum_b MTTKRP(X_b); so a CTA works on tiles of ONE block
// and keeps that block's BR outer factor rows in shared memory, loaded once by a TMA bulk copy
// (cp.async.bulk + mbarrier).  Per nonzero the lane-group then reads the outer row from shared
// memory (LDS.128) and gathers only the other product modes' rows from L2 (ld.global.cg: L2
// only, no L1 allocation — measured 3-5% faster than the read-only path for these random
// rows).  On B200 the L1TEX data pipe (~128 B/clk/SM, shared by LDG hits, LDS and shuffles) is
// the binding resource of this kernel (profiles/round2); an outer row from shared memory costs
// one wavefront and no L2 traffic, against ~1.7 data-pipe cycles for an L2-resident LDG row
// (tools/gather_ceiling.py): measured 1.29-1.34x over the unblocked kernel at R=32.
//
// The segmented reduction is the paper's flag-driven one: bf marks segment heads,
// sf[t] = bf[t*T] tells a tile whether it starts inside a segment; a row recurs once per block,
// so EVERY segment flush is a red.global.add (the output is zeroed first).  The nonzero stream
// (packed words, values, bf) is double-buffered through shared memory with cp.async, one
// 32-nonzero chunk ahead, as in the unblocked engine.
#pragma once
#include "fcoo_blocked.cuh"
#include "fcoo_engine_kernels.cuh"

namespace fcoo {

__device__ __forceinline__ bool blocked_gated_off(const BlockedParams& P) {
  return P.gate && ((__ldg(P.gate) != 0) != (P.gate_on != 0));
}

// ---- TMA bulk copy global -> shared with an mbarrier (SASS: UBLKCP + SYNCS) ----
__device__ __forceinline__ void mbar_init(uint64_t* m, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(n)
               : "memory");
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
      "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(mb),
      "r"(parity)
      : "memory");
}

// Random factor-row gathers: L2 only (.cg), no L1 allocation.
template <int VEC>
__device__ __forceinline__ typename Ld<VEC>::T ld_cg(const float* p);
template <>
__device__ __forceinline__ float4 ld_cg<4>(const float* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ float ld_cg<1>(const float* p) {
  float r;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
template <int VEC>
__device__ __forceinline__ typename Ld<VEC>::T lds_row(uint32_t a);
template <>
__device__ __forceinline__ float4 lds_row<4>(uint32_t a) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
  return r;
}
template <>
__device__ __forceinline__ float lds_row<1>(uint32_t a) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
  return r;
}

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}

// acc += v * Hadamard(r[0..NP)) for fp32 float4 lanes with packed FMUL2 / FFMA2 (sm_100).
template <int NP>
__device__ __forceinline__ void had_acc_f4(float4& acc, float v, const float4 (&r)[NP]) {
  unsigned long long h0 = pack2(r[0].x, r[0].y), h1 = pack2(r[0].z, r[0].w);
#pragma unroll
  for (int a = 1; a < NP; ++a) {
    asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(h0) : "l"(pack2(r[a].x, r[a].y)));
    asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(h1) : "l"(pack2(r[a].z, r[a].w)));
  }
  unsigned long long a0 = pack2(acc.x, acc.y), a1 = pack2(acc.z, acc.w), vv = pack2(v, v);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(vv), "l"(h0));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a1) : "l"(vv), "l"(h1));
  unpack2(a0, acc.x, acc.y);
  unpack2(a1, acc.z, acc.w);
}

template <int VEC, class ACC, int NP>
__device__ __forceinline__ void acc_add(typename Acc<VEC, ACC>::T& acc, float v, const typename Ld<VEC>::T (&r)[NP]) {
  if constexpr (VEC == 4 && std::is_same<ACC, float>::value) had_acc_f4<NP>(acc, v, r);
  else Acc<VEC, ACC>::template add<NP>(acc, v, r);
}

// NP product modes (outer + NP-1 gathered), G lanes per group, VEC floats per column slot, CPL
// column slots per lane; SMEM: outer rows from the shared-memory block (else LDG, for a block
// too large for shared memory); TB threads per CTA.
// NCP copies of the block (NCP > 1 only for rows narrower than 128 B: copy k starts k row-widths
// past a 128-B boundary, and group g reads row r from copy (g - r) mod NCP, so the NCP groups that
// share a 128-B bank line in one LDS.128 always hit disjoint banks; measured).
template <int NP, int G, int VEC, int CPL, class ACC, bool FULL, int NCP, int TB, int MINB>
__global__ void __launch_bounds__(TB, MINB) k_mttkrp_blocked(const BlockedParams P) {
  constexpr bool SMEM = NCP > 0;
  using V = Ld<VEC>;
  using VT = typename V::T;
  using A = Acc<VEC, ACC>;
  using AT = typename A::T;
  constexpr int NW = NP >= 2 ? NP - 1 : 1;
  constexpr int NST = blocked_nst<NP>();
  using S = BStage<NW, G, NST>;
  constexpr int B = batch_size<NP, VEC, CPL>();
  constexpr int CH = S::CH;
  extern __shared__ uint4 smem_raw[];
  __shared__ uint64_t mbar;
  if (blocked_gated_off(P)) return;  // before any TMA is in flight
  const int2 item = P.items[P.item0 + blockIdx.x];
  const int b = item.x;
  const int R = P.R;
  float* blk = reinterpret_cast<float*>(smem_raw);
  // floats from one copy of the block to the next (a multiple of 128 B plus one row)
  const uint32_t cstride = NCP > 1 ? ((uint32_t)P.BR * R + 31u) / 32u * 32u + (uint32_t)R : 0u;
  uint32_t* stage_base =
      reinterpret_cast<uint32_t*>(smem_raw) + (SMEM ? (NCP > 1 ? NCP * cstride : (size_t)P.BR * R) : 0);  // R % 4 == 0
  if constexpr (SMEM) {
    if (threadIdx.x == 0) {
      mbar_init(&mbar, NCP);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int r0 = b * P.BR;
      const int nr = min(P.BR, P.Io - r0);
#pragma unroll
      for (int k = 0; k < NCP; ++k)
        bulk_g2s(blk + k * cstride, P.U[0] + (size_t)r0 * R, (uint32_t)nr * (uint32_t)R * 4u, &mbar);
    }
  }
  const int g = threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int64_t t = (int64_t)item.y + g;
  const bool live = t < P.blk_start[b + 1] / P.T && t >= P.tile_begin && t < P.tile_end;
  uint32_t* my = stage_base + g * S::STRIDE;

  const uint32_t rowb = (uint32_t)R * 4u;
  int col[CPL];
  bool cok[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    col[c] = (gl + G * c) * VEC;
    cok[c] = FULL || col[c] < R;
  }
  uint32_t sb[CPL];           // shared-memory address of column slot c of local outer row 0
  const char* ub[NP][CPL];    // global base of column slot c of each factor (outer: block row 0)
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int cc = cok[c] ? col[c] : 0;
    sb[c] = (uint32_t)__cvta_generic_to_shared(blk) + (uint32_t)cc * 4u;
    ub[0][c] = reinterpret_cast<const char*>(P.U[0] + (size_t)b * P.BR * R + cc);
#pragma unroll
    for (int a = 1; a < NP; ++a) ub[a][c] = reinterpret_cast<const char*>(P.U[a] + cc);
  }
  const int shift = P.shift;
  const uint32_t lmask = NP >= 2 ? ((shift >= 32) ? 0xffffffffu : ((1u << shift) - 1u)) : 0u;

  const int64_t p0 = t * (int64_t)P.T;
  const int64_t pend = live ? min(p0 + (int64_t)P.T, P.blk_end[b]) : p0;
  const int nchunk = (int)((pend - p0) / CH);
  const bool left_open = live && !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = live ? P.seg_base[t] - 1u : 0u;
  uint32_t row = left_open ? P.seg_coord[s] : 0u;
  ACC* const outp = reinterpret_cast<ACC*>(P.out);
  float* const mcp = P.out_mc;

  AT acc[CPL], hi[CPL];  // hi: the chain-capped part of the running segment (chain_fold)
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = hi[c] = A::zero();
  auto flush = [&]() {
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (cok[c]) {
        if constexpr (std::is_same<AT, float4>::value) {
          if (mcp) {
            mc_flush_if(false, true, mcp + (size_t)row * (uint32_t)R + col[c], acc[c]);
            continue;
          }
        }
        A::red(outp + (size_t)row * (uint32_t)R + col[c], acc[c]);
      }
  };
  // rows of nonzero e: r[0] outer (shared memory or global), r[1..NP-2] middles, r[NP-1] last
  auto gather = [&](const uint32_t* w, int wstride, VT (&r)[CPL][NP]) {
    const uint32_t w0 = w[0];
    const uint32_t local = NP >= 2 ? (shift >= 32 ? 0u : (w0 >> shift)) : w0;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      if (!cok[c]) {
#pragma unroll
        for (int a = 0; a < NP; ++a) r[c][a] = V::zero();
        continue;
      }
      if constexpr (NCP > 1)
        r[c][0] = lds_row<VEC>(sb[c] + (((uint32_t)g - local) & (NCP - 1)) * (cstride * 4u) + local * rowb);
      else if constexpr (SMEM) r[c][0] = lds_row<VEC>(sb[c] + local * rowb);
      else r[c][0] = V::load(reinterpret_cast<const float*>(ub[0][c] + (size_t)local * rowb));
      if constexpr (NP >= 2) {
#pragma unroll
        for (int a = 1; a + 1 < NP; ++a)
          r[c][a] = ld_cg<VEC>(reinterpret_cast<const float*>(ub[a][c] + (size_t)w[a * wstride] * rowb));
        r[c][NP - 1] = ld_cg<VEC>(reinterpret_cast<const float*>(ub[NP - 1][c] + (size_t)(w0 & lmask) * rowb));
      }
    }
  };

  auto issue = [&](int64_t pc, int st) {  // group-cooperative cp.async of chunk [pc, pc+32)
    uint32_t* dst = my + st * S::WORDS;
#pragma unroll
    for (int a = 0; a <= NW; ++a) {
      const uint32_t* base = a < NW ? P.pk + (int64_t)a * P.nstream : reinterpret_cast<const uint32_t*>(P.val);
#pragma unroll
      for (int k = 0; k < (8 + G - 1) / G; ++k) {
        const int q = gl + k * G;
        if (q < 8) cp_async16(dst + a * CH + q * 4, base + pc + q * 4);
      }
    }
    if (gl == 0) cp_async4(dst + (NW + 1) * CH, P.bf + (pc >> 5));
  };
#pragma unroll
  for (int j = 0; j + 1 < NST; ++j) {  // NST - 1 chunks in flight
    if (j < nchunk) issue(p0 + (int64_t)j * CH, j);
    cp_async_commit();
  }
  if constexpr (SMEM) mbar_wait(&mbar, 0);  // every thread: the block rows are resident

  for (int ci = 0; ci < nchunk; ++ci) {
    if (ci + NST - 1 < nchunk) issue(p0 + (int64_t)(ci + NST - 1) * CH, (ci + NST - 1) % NST);
    cp_async_commit();
    cp_async_wait<NST - 1>();
    __syncwarp(gmask);
    const uint32_t* stg = my + (ci % NST) * S::WORDS;
    const uint32_t bfw = stg[(NW + 1) * CH];
#pragma unroll
    for (int bi = 0; bi < CH / B; ++bi) {
      uint32_t w[NW][B];
      uint32_t vb[B];
#pragma unroll
      for (int a = 0; a < NW; ++a) lds_batch<B>(stg + a * CH + bi * B, w[a]);
      lds_batch<B>(stg + NW * CH + bi * B, vb);
      const uint32_t heads = (bfw >> (bi * B)) & ((1u << B) - 1u);
      VT r[B][CPL][NP];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        uint32_t we[NW];
#pragma unroll
        for (int a = 0; a < NW; ++a) we[a] = w[a][e];
        gather(we, 1, r[e]);
      }
      if (heads == 0) {
#pragma unroll
        for (int e = 0; e < B; ++e)
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc_add<VEC, ACC, NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
      } else {
        const bool first = (ci == 0 && bi == 0);
#pragma unroll
        for (int c = 0; c < CPL; ++c) chain_absorb(acc[c], hi[c]);
#pragma unroll
        for (int e = 0; e < B; ++e) {
          if ((heads >> e) & 1u) {
            if (e != 0 || !first) flush();
#pragma unroll
            for (int c = 0; c < CPL; ++c) acc[c] = A::zero();
            ++s;
            row = P.seg_coord[s];
          }
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc_add<VEC, ACC, NP>(acc[c], __uint_as_float(vb[e]), r[e][c]);
        }
      }
    }
    if (ci % kChainChunks == kChainChunks - 1) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) chain_fold(hi[c], acc[c]);
    }
    __syncwarp(gmask);  // every lane is done with this stage before it is refilled
  }
  if (!live) return;
#pragma unroll
  for (int c = 0; c < CPL; ++c) chain_absorb(acc[c], hi[c]);
  // ragged end of a block's last tile: one nonzero at a time
  for (int64_t p = p0 + (int64_t)nchunk * CH; p < pend; ++p) {
    if ((P.bf[p >> 5] >> (p & 31)) & 1u) {
      if (p != p0) flush();
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = A::zero();
      ++s;
      row = P.seg_coord[s];
    }
    uint32_t we[NW];
#pragma unroll
    for (int a = 0; a < NW; ++a) we[a] = P.pk[(int64_t)a * P.nstream + p];
    VT r1[CPL][NP];
    gather(we, 1, r1);
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc_add<VEC, ACC, NP>(acc[c], P.val[p], r1[c]);
  }
  flush();
  if (mcp) __threadfence_system();
}

}  // namespace fcoo


namespace fcoo {

template <int NP, int G, int VEC, int CPL, class ACC, int NCP, int TB>
cudaError_t launch_blocked_one(const BlockedParams& P, int nitems, cudaStream_t s) {
  constexpr bool SMEM = NCP > 0;
  constexpr int NW = NP >= 2 ? NP - 1 : 1;
  // one product mode (SpTTM, order-2 MTTKRP): 77 registers, so 3 CTAs of 256 threads fit per SM
  constexpr int MINB = TB == 256 ? (NP == 1 ? 3 : 2) : 1;
  constexpr bool FULL = VEC == 4;  // float4 shapes are chosen only when R == 4 * G
  void (*kern)(const BlockedParams) = k_mttkrp_blocked<NP, G, VEC, CPL, ACC, FULL, NCP, TB, MINB>;
  const size_t smem = blocked_block_bytes(P.BR, P.R, NCP) +
                      sizeof(uint32_t) * (size_t)(TB / G) * BStage<NW, G, blocked_nst<NP>()>::STRIDE;
  // attributes are set when the dynamic shared memory grows (not per call: cheap host path, and
  // nothing but launches happens while cp_als captures an iteration into a CUDA graph)
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // carveout: shared memory for the CTAs that fit by registers/threads, the rest stays L1
    const int ctas = std::max(1, std::min(MINB, (int)((228 * 1024) / (smem + 1024))));
    int pct = (int)((ctas * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)) + 1;
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
    configured = smem;
  }
  if (nitems <= 0) return cudaSuccess;
  kern<<<(unsigned)nitems, TB, smem, s>>>(P);
  count_launch();
  return cudaGetLastError();
}

template <int NP, int G, class ACC>
cudaError_t launch_blocked_g4(const BlockedParams& P, int nitems, const BlockedShape& sh, cudaStream_t s) {
  constexpr int C = blocked_copies(4 * G);
  if (!sh.smem) return launch_blocked_one<NP, G, 4, 1, ACC, 0, 256>(P, nitems, s);
  if (sh.TB == 512) return launch_blocked_one<NP, G, 4, 1, ACC, 1, 512>(P, nitems, s);
  if constexpr (C > 1)
    if (sh.ncp == C) return launch_blocked_one<NP, G, 4, 1, ACC, C, 256>(P, nitems, s);
  return launch_blocked_one<NP, G, 4, 1, ACC, 1, 256>(P, nitems, s);
}

template <int NP, class ACC>
cudaError_t launch_blocked_np(const BlockedParams& P, int nitems, bool vec_ok, cudaStream_t s) {
  const BlockedShape sh = blocked_shape(NP, P.R, P.BR, vec_ok);
  if (sh.VEC == 4) {
    switch (sh.G) {
      case 2: return launch_blocked_g4<NP, 2, ACC>(P, nitems, sh, s);
      case 4: return launch_blocked_g4<NP, 4, ACC>(P, nitems, sh, s);
      case 8: return launch_blocked_g4<NP, 8, ACC>(P, nitems, sh, s);
      case 16: return launch_blocked_g4<NP, 16, ACC>(P, nitems, sh, s);
      default: return launch_blocked_g4<NP, 32, ACC>(P, nitems, sh, s);
    }
  }
  switch (sh.CPL) {
    case 1: return launch_blocked_one<NP, 32, 1, 1, ACC, 0, 256>(P, nitems, s);
    case 2: return launch_blocked_one<NP, 32, 1, 2, ACC, 0, 256>(P, nitems, s);
    case 4: return launch_blocked_one<NP, 32, 1, 4, ACC, 0, 256>(P, nitems, s);
    default: return launch_blocked_one<NP, 32, 1, 8, ACC, 0, 256>(P, nitems, s);
  }
}

}  // namespace fcoo
