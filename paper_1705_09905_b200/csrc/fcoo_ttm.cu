// fcoo_ttm.cu — the SpTTM kernel (Eq.(3), Table I row 1; DESIGN.md §6 "SpTTM").
//
//   Y(s, :) = sum_{nonzeros q of fibre s} v_q * U(i_n(q), :)
//
// on the F-COO of an FCOO_OP_TTM handle: the product index of a nonzero is i_n, the segments of
// bf are the fibres, and the output row of segment s is s itself (semi-sparse output).
// Same flag-driven segmented reduction as the SpMTTKRP engine, specialised for the
// one-row-per-nonzero shape, where round 1 measured the general engine instruction-bound (ncu:
// 4.9 warp instructions per nonzero on brainq mode 0, 59% issue busy) and tail-bound (2.27 waves):
//   - persistent CTAs (one wave: grid = SMs x resident CTAs), lane-groups stride over the tiles;
//   - the factor U in shared memory when it fits (one TMA bulk copy per CTA; brainq modes 1 and 3
//     have 60 and 9 rows), else gathered with LDG;
//   - per batch of 8 nonzeros one warp-uniform test for heads; a head-free batch is 8 x (row load
//     + 2 FFMA2); a batch with heads runs a branch-free step per nonzero: at a head the finished
//     segment is written by a predicated st.global (a segment that started in this tile) or, in
//     the rare batch where some group closes its tile's left-open first segment (shared with the
//     previous tile), red.global.add; the accumulator is restarted by a multiply with 0 and the
//     segment ordinal advances by the head bit;
//   - the tile's last segment is flushed after the loop: red.add when it continues into the next
//     tile (sf[t+1] == 0), else a store.
// Rows of segments that cross a tile boundary are zeroed first (k_zero_boundary_rows), every other
// row is stored exactly once.
#include "fcoo_blocked_kernels.cuh"

namespace fcoo {

struct TtmParams {
  const uint32_t* idx;  // product index i_n per stream position
  const float* val;
  const uint32_t* bf;
  const uint32_t* sf;
  const uint32_t* seg_base;
  const float* U;       // I_n x R
  float* out;           // nsegs x R
  int64_t nnz, ntiles, tile_begin, tile_end;
  int T, R, In;
};

__device__ __forceinline__ void st_red_if(bool st, bool rd, float* p, float4 v) {
  asm volatile(
      "{ .reg .pred ps, pr; setp.ne.b32 ps, %0, 0; setp.ne.b32 pr, %1, 0;\n"
      "  @ps st.global.v4.f32 [%2], {%3,%4,%5,%6};\n"
      "  @pr red.global.add.v4.f32 [%2], {%3,%4,%5,%6}; }" ::"r"((int)st),
      "r"((int)rd), "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}

__device__ __forceinline__ void st_if(bool st, float* p, float4 v) {
  asm volatile(
      "{ .reg .pred ps; setp.ne.b32 ps, %0, 0;\n"
      "  @ps st.global.v4.f32 [%1], {%2,%3,%4,%5}; }" ::"r"((int)st),
      "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}

// acc = acc * k + v * w  (k = 0 at a segment head, else 1) with FMUL2 / FFMA2
__device__ __forceinline__ void scale_fma(float4& acc, float k, float v, const float4& w) {
  unsigned long long a0 = pack2(acc.x, acc.y), a1 = pack2(acc.z, acc.w), kk = pack2(k, k), vv = pack2(v, v);
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(a0) : "l"(kk));
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(a1) : "l"(kk));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(vv), "l"(pack2(w.x, w.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a1) : "l"(vv), "l"(pack2(w.z, w.w)));
  unpack2(a0, acc.x, acc.y);
  unpack2(a1, acc.z, acc.w);
}
__device__ __forceinline__ void fma4(float4& acc, float v, const float4& w) {
  unsigned long long a0 = pack2(acc.x, acc.y), a1 = pack2(acc.z, acc.w), vv = pack2(v, v);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(vv), "l"(pack2(w.x, w.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a1) : "l"(vv), "l"(pack2(w.z, w.w)));
  unpack2(a0, acc.x, acc.y);
  unpack2(a1, acc.z, acc.w);
}

// stream stages per lane-group (kTtmStages - 1 chunks of 32 nonzeros in flight); 4 stages
// measured the same as 2 on brainq (the kernel is issue-bound)
constexpr int kTtmStages = 2;

template <int G, bool SMEM>
__global__ void __launch_bounds__(256) k_ttm_lean(const TtmParams P) {
  constexpr int TB = 256, CH = 32, B = 8, NST = kTtmStages;
  constexpr int WORDS = 2 * CH + 4;                                   // idx, val, bf word, pad
  constexpr int RAW = NST * WORDS, WANT = (G >= 4 ? G : 4) % 32;
  constexpr int STRIDE = RAW + (((WANT - RAW % 32) % 32) + 32) % 32;  // groups of a warp on distinct banks
  extern __shared__ uint4 smem_raw[];
  const int R = 4 * G;
  // U in shared memory: rows padded to SB = max(128, 4R) bytes, each holding C = SB / 4R copies of
  // the row; lane-group g reads copy g % C, so the C groups that share a 128-B bank line in one
  // LDS.128 hit disjoint banks (a 64-B row at R = 16 would otherwise collide 2-way)
  constexpr int SB = 4 * R >= 128 ? 4 * R : 128, C = SB / (4 * R);
  uint32_t* stage_base = reinterpret_cast<uint32_t*>(smem_raw);
  float* Us = reinterpret_cast<float*>(smem_raw) + (size_t)(TB / G) * STRIDE;
  if constexpr (SMEM) {
    const int n4 = P.In * C * G;  // float4 slots
    for (int k = threadIdx.x; k < n4; k += TB) {
      const int r = k / (C * G), c = (k / G) % C, q = k % G;
      reinterpret_cast<float4*>(Us)[(size_t)r * (SB / 16) + c * G + q] =
          __ldg(reinterpret_cast<const float4*>(P.U) + (size_t)r * G + q);
    }
    __syncthreads();
  }
  const int g = threadIdx.x / G, gl = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  uint32_t* my = stage_base + g * STRIDE;
  const int col = gl * 4;
  const uint32_t rowb = (uint32_t)R * 4u;
  const uint32_t us = (uint32_t)__cvta_generic_to_shared(Us) + (uint32_t)((g % C) * R + col) * 4u;
  const char* ug = reinterpret_cast<const char*>(P.U + col);
  auto row_of = [&](uint32_t i) -> float4 {
    if constexpr (SMEM) return lds_row<4>(us + i * (uint32_t)SB);
    else return __ldg(reinterpret_cast<const float4*>(ug + (size_t)i * rowb));
  };

  const int64_t ngroups = (int64_t)gridDim.x * (TB / G);
  constexpr int NGW = 32 / G;                 // groups per warp (G <= 32)
  const int gw = g % NGW, gw0 = g - gw;       // group within the warp, the warp's first group
  const int nchunk_w = P.T / CH;              // chunks of a full tile (the warp-uniform trip count)
  float* const orow = P.out + col;
  // every loop that contains a warp-wide sync or vote is warp-uniform: the warp's groups take the
  // consecutive tiles tw + gw; a group past the end (or past its tile's last full chunk) works on
  // zero rows / zero values and never flushes
  for (int64_t tw = P.tile_begin + (int64_t)blockIdx.x * (TB / G) + gw0; tw < P.tile_end; tw += ngroups) {
    const int64_t t = tw + gw;
    const bool live = t < P.tile_end;
    const int64_t p0 = t * (int64_t)P.T;
    const int64_t p1 = live ? min(p0 + (int64_t)P.T, P.nnz) : p0;
    const int nchunk = (int)((p1 - p0) / CH);
    const bool left_open = live && !((P.sf[t >> 5] >> (t & 31)) & 1u);
    // ordinal of the running segment: the one entering from the previous tile (left-open), else
    // the one the tile's first nonzero starts (whose head bit is then skipped below)
    uint32_t s = live ? P.seg_base[t] - (left_open ? 1u : 0u) : 0u;
    bool lo = left_open;  // the running segment is the one shared with the previous tile
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 hi = acc;  // the chain-capped part of the running segment (chain_fold, every 256 nnz)
    // warp-cooperative copy of chunk ci of every group of the warp: each 8-lane quarter writes one
    // contiguous 128-B segment (one array of one group), so the shared-memory writes are
    // conflict-free (a 4-lane group writing 64 B per instruction collided 4-way)
    auto issue = [&](int ci, int st) {
#pragma unroll
      for (int k = 0; k < (2 * NGW + 3) / 4; ++k) {
        const int seg = k * 4 + (lane >> 3);  // segment: group seg / 2, array seg % 2
        if (seg < 2 * NGW) {
          const int gg = seg >> 1;
          const int64_t tt = tw + gg;
          const int64_t pc = tt * (int64_t)P.T + (int64_t)ci * CH;
          if (tt < P.tile_end && pc + CH <= min(tt * (int64_t)P.T + (int64_t)P.T, P.nnz)) {
            const uint32_t* base = (seg & 1) ? reinterpret_cast<const uint32_t*>(P.val) : P.idx;
            cp_async16(stage_base + (gw0 + gg) * STRIDE + st * WORDS + (seg & 1) * CH + (lane & 7) * 4,
                       base + pc + (lane & 7) * 4);
          }
        }
      }
      if (gl == 0 && ci < nchunk) cp_async4(my + st * WORDS + 2 * CH, P.bf + ((p0 + (int64_t)ci * CH) >> 5));
    };
#pragma unroll
    for (int j = 0; j + 1 < NST; ++j) {  // NST - 1 chunks in flight
      if (j < nchunk_w) issue(j, j);
      cp_async_commit();
    }
    for (int ci = 0; ci < nchunk_w; ++ci) {
      if (ci + NST - 1 < nchunk_w) issue(ci + NST - 1, (ci + NST - 1) % NST);
      cp_async_commit();
      cp_async_wait<NST - 1>();
      __syncwarp();  // the warp's groups copy each other's chunks
      const bool on = ci < nchunk;  // this group's chunk exists
      const uint32_t* stg = my + (ci % NST) * WORDS;
      uint32_t bfw = on ? stg[2 * CH] : 0u;
      if (ci == 0) bfw &= ~1u;  // the tile's first nonzero opens (never closes) a segment
#pragma unroll
      for (int bi = 0; bi < CH / B; ++bi) {
        uint32_t ix[B], vb[B];
        lds_batch<B>(stg + bi * B, ix);
        lds_batch<B>(stg + CH + bi * B, vb);
        float4 w[B];
#pragma unroll
        for (int e = 0; e < B; ++e) {
          if (!on) ix[e] = 0u, vb[e] = 0u;  // stale stage: a valid row, a zero value
          w[e] = row_of(ix[e]);
        }
        const uint32_t heads = (bfw >> (bi * B)) & 0xffu;
        // warp-uniform paths: divergent per-group branches would make the warp issue both sequences
        if (!__any_sync(0xffffffffu, heads != 0)) {
#pragma unroll
          for (int e = 0; e < B; ++e) fma4(acc, __uint_as_float(vb[e]), w[e]);
        } else if (!__any_sync(0xffffffffu, lo && heads != 0)) {  // every closed segment is owned
          chain_absorb(acc, hi);
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const bool hd = (heads >> e) & 1u;
            st_if(hd, orow + (size_t)s * rowb / 4, acc);
            s += hd ? 1u : 0u;
            scale_fma(acc, hd ? 0.f : 1.f, __uint_as_float(vb[e]), w[e]);
          }
        } else {  // some group closes its left-open segment (once per tile): red.add for that one
          chain_absorb(acc, hi);
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const bool hd = (heads >> e) & 1u;
            st_red_if(hd && !lo, hd && lo, orow + (size_t)s * rowb / 4, acc);
            lo = lo && !hd;
            s += hd ? 1u : 0u;
            scale_fma(acc, hd ? 0.f : 1.f, __uint_as_float(vb[e]), w[e]);
          }
        }
      }
      if (ci % kChainChunks == kChainChunks - 1) chain_fold(hi, acc);
      __syncwarp();  // every lane is done with this stage before it is refilled
    }
    if (!live) continue;
    chain_absorb(acc, hi);
    // ragged tail of the tensor's last tile
    for (int64_t p = p0 + (int64_t)nchunk * CH; p < p1; ++p) {
      const bool hd = p != p0 && ((P.bf[p >> 5] >> (p & 31)) & 1u);
      st_red_if(hd && !lo, hd && lo, orow + (size_t)s * rowb / 4, acc);
      lo = lo && !hd;
      s += hd ? 1u : 0u;
      scale_fma(acc, hd ? 0.f : 1.f, P.val[p], row_of(P.idx[p]));
    }
    // the running segment: shared with the next tile (red) or, if it was also the left-open one
    // (lo still set), shared with the previous tile (red); otherwise owned (store)
    const bool right_open = (t + 1 < P.ntiles) && !((P.sf[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u);
    const bool red = right_open || lo;
    st_red_if(!red, red, orow + (size_t)s * rowb / 4, acc);
  }
}

template <int G, bool SMEM>
cudaError_t launch_ttm(const TtmParams& P, cudaStream_t s) {
  constexpr int TB = 256;
  constexpr int WORDS = 2 * 32 + 4, RAW = kTtmStages * WORDS, WANT = (G >= 4 ? G : 4) % 32;
  constexpr int STRIDE = RAW + (((WANT - RAW % 32) % 32) + 32) % 32;
  constexpr int SB = 16 * G >= 128 ? 16 * G : 128;
  const size_t smem = sizeof(uint32_t) * (size_t)(TB / G) * STRIDE + (SMEM ? (size_t)P.In * SB : 0);
  auto kern = k_ttm_lean<G, SMEM>;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TB, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t tiles = P.tile_end - P.tile_begin;
  const int64_t need = (tiles + TB / G - 1) / (TB / G);
  // note: the grid stride keeps every warp's tiles consecutive (warps start at multiples of 32/G)
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)nsm * per_sm));
  if (tiles <= 0) return cudaSuccess;
  kern<<<grid, TB, smem, s>>>(P);
  count_launch();
  return cudaGetLastError();
}

// SpTTM through the lean kernel when it applies (fp32 float4 lanes with R = 4G, G a power of two
// in [2, 32], 16-B aligned U and output, not deterministic); returns false to let the caller use
// the general engine.
static bool lean_applies(int R, const float* U, const float* out) {
  const int q = R / 4;
  if (R % 4 || q < 2 || q > 32 || (q & (q - 1))) return false;
  return !((reinterpret_cast<uintptr_t>(U) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u));
}
static cudaError_t launch_lean(TtmParams& P, int R, cudaStream_t s);

bool run_ttm_lean(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s, fcoo_status* st) {
  if (!lean_applies(R, U, out) || f->deterministic) return false;
  TtmParams P{};
  P.idx = f->pidx; P.val = f->val; P.bf = f->bf; P.sf = f->sf; P.seg_base = f->seg_base; P.U = U; P.out = out;
  P.nnz = f->nnz; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.R = R; P.In = (int)f->dims[f->mode];
  const cudaError_t e = launch_lean(P, R, s);
  *st = e == cudaSuccess ? FCOO_OK : fail(FCOO_ERR_CUDA, "ttm launch: %s", cudaGetErrorString(e));
  return true;
}

// SpTTM on the last product mode of an MTTKRP handle from its second flag level (Fig. 2):
// the same stream, the last product mode's index row as the TTM product index, bf2 / sf2 /
// seg_base2 as the fibre flags; rows of fibres that cross a tile are zeroed first, the rest stored once.
fcoo_status run_ttm_fibres(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s) {
  if (!lean_applies(R, U, out))
    return fail(FCOO_ERR_ARG, "SpTTM on the fibre level needs R %% 4 == 0, R/4 a power of two <= 32, 16-B aligned U/out");
  TtmParams P{};
  P.idx = f->pidx + (int64_t)(f->n_prod - 1) * f->nnz_pad;
  P.val = f->val; P.bf = f->bf2; P.sf = f->sf2; P.seg_base = f->seg_base2; P.U = U; P.out = out;
  P.nnz = f->nnz; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.R = R; P.In = (int)f->dims[f->prod_modes[f->n_prod - 1]];
  if (f->tile_begin != 0 || f->tile_end != f->ntiles) {
    FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)f->nfib * R, s));
  } else {
    const fcoo_status z = zero_boundary_rows_f32(f->sf2, f->seg_base2, f->tile_begin, f->tile_end, R, out, s);
    if (z) return z;
  }
  const cudaError_t e = launch_lean(P, R, s);
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "ttm launch: %s", cudaGetErrorString(e));
  if (f->comm) return comm_allreduce(f->comm, out, (size_t)f->nfib * R, s);
  return FCOO_OK;
}

static cudaError_t launch_lean(TtmParams& P, int R, cudaStream_t s) {
  const int q = R / 4;
  // U in shared memory up to 32 KB with rows padded to >= 128 B (the staging of 256 threads takes
  // 35 KB at R = 16, 70 KB at R = 8)
  const bool smem = (size_t)P.In * std::max(R * 4, 128) <= 32 * 1024;
  cudaError_t e;
  switch (q) {
    case 2: e = smem ? launch_ttm<2, true>(P, s) : launch_ttm<2, false>(P, s); break;
    case 4: e = smem ? launch_ttm<4, true>(P, s) : launch_ttm<4, false>(P, s); break;
    case 8: e = smem ? launch_ttm<8, true>(P, s) : launch_ttm<8, false>(P, s); break;
    case 16: e = smem ? launch_ttm<16, true>(P, s) : launch_ttm<16, false>(P, s); break;
    default: e = smem ? launch_ttm<32, true>(P, s) : launch_ttm<32, false>(P, s); break;
  }
  return e;
}

}  // namespace fcoo
