// fcoo_blocked.cuh — host-side declarations of the blocked SpMTTKRP (FCOO_BUILD_BLOCKED): the
// kernel parameters, the launch shape, and the per-(NP, accumulator) launchers instantiated in
// fcoo_blocked_np<NP>_<acc>.cu (kernels: fcoo_blocked_kernels.cuh).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "fcoo_engine.cuh"

namespace fcoo {

struct BlockedParams {
  const uint32_t* pk;          // n_words x nstream: word 0 = (local outer << shift) | last, then middles
  const float* val;
  const uint32_t* bf;
  const uint32_t* sf;
  const uint32_t* seg_base;
  const uint32_t* seg_coord;   // row of segment s
  const int64_t* blk_start;    // [nblocks + 1]
  const int64_t* blk_end;      // [nblocks]
  const int2* items;           // (block, first tile), this launch: items[item0 + blockIdx.x]
  const float* U[kMaxProd];    // U[0] = outer factor, U[1..NP-2] middle, U[NP-1] last
  int64_t nstream, ntiles, tile_begin, tile_end, item0;
  int T, R, BR, Io, shift;
  void* out;                   // ACC* I_n x R, zeroed by the caller
  float* out_mc;               // multicast view of the output (fused combine) or nullptr
  const int* gate;
  int gate_on;
};

// Shared-memory staging of the stream: per lane-group, 2 stages of one 32-nonzero chunk:
// NW packed-word rows + the values + the bf word (+3 pad words, 16-B aligned).  The per-group
// stride is padded to G (mod 32) words so the 32/G groups of a warp read distinct banks.
template <int NW, int G>
struct BStage {
  static constexpr int CH = 32;
  static constexpr int WORDS = (NW + 1) * CH + 4;
  static constexpr int RAW = 2 * WORDS;
  static constexpr int WANT = (G >= 4 ? G : 4) % 32;
  static constexpr int STRIDE = RAW + (((WANT - RAW % 32) % 32) + 32) % 32;
};

// Host side: shared-memory bytes and launch shape of the blocked kernel for (R, BR).
struct BlockedShape {
  int G, VEC, CPL, TB;
  bool smem;
  size_t block_bytes;
};
// Staging bytes of a CTA of TB threads (lane-groups of G lanes, NW packed-word rows).
inline size_t blocked_stage_bytes(int NW, int G, int TB) {
  const int words = (NW + 1) * 32 + 4, raw = 2 * words, want = (G >= 4 ? G : 4) % 32;
  const int stride = raw + (((want - raw % 32) % 32) + 32) % 32;
  return sizeof(uint32_t) * (size_t)(TB / G) * stride;
}

inline BlockedShape blocked_shape(int NP, int R, int BR, bool vec_ok) {
  BlockedShape sh{};
  // float4 lanes when R/4 is a power of two in [2, 32] (every lane full: the paper's ranks
  // 8..64 and 128); otherwise one warp per tile with CPL scalar column slots per lane
  const int q = R / 4;
  if (vec_ok && q >= 2 && q <= 32 && (q & (q - 1)) == 0) {
    sh.G = q; sh.VEC = 4; sh.CPL = 1;
  } else {
    vec_ok = false;
    sh.G = 32; sh.VEC = 1;
    const int cpl = (R + 31) / 32;
    sh.CPL = cpl <= 1 ? 1 : cpl <= 2 ? 2 : cpl <= 4 ? 4 : 8;
  }
  sh.block_bytes = (size_t)BR * R * 4;
  // the outer block in shared memory with two 256-thread CTAs per SM when block + staging fit
  // ~110 KB each, else one 512-thread CTA up to ~220 KB, else the outer rows are gathered from
  // global memory like the others (always for scalar lanes: the TMA bulk copy moves whole 16-B
  // units of 16-B aligned rows)
  const int NW = NP >= 2 ? NP - 1 : 1;
  sh.smem = false;
  sh.TB = 256;
  if (vec_ok) {
    if (sh.block_bytes + blocked_stage_bytes(NW, sh.G, 256) <= 110 * 1024) {
      sh.smem = true;
    } else if (sh.block_bytes + blocked_stage_bytes(NW, sh.G, 512) <= 220 * 1024) {
      sh.smem = true;
      sh.TB = 512;
    }
  }
  return sh;
}

template <int NP, class ACC>
cudaError_t launch_blocked_np(const BlockedParams& P, int nitems, bool vec_ok, cudaStream_t s);

}  // namespace fcoo
