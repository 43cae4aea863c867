// fcoo_blocked.cuh — host-side declarations of the blocked SpMTTKRP (FCOO_BUILD_BLOCKED): the
// kernel parameters, the launch shape, and the per-(NP, accumulator) launchers instantiated in
// fcoo_blocked_np<NP>_<acc>.cu (kernels: fcoo_blocked_kernels.cuh).
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
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

// Shared-memory staging of the stream: per lane-group, NST stages of one 32-nonzero chunk each
// (NST - 1 chunks in flight): NW packed-word rows + the values + the bf word (+3 pad words, 16-B
// aligned).  The per-group stride is padded to G (mod 32) words so the 32/G groups of a warp read
// distinct banks.  NST = 2 (SpTTM with 4 stages measured the same: not stream-latency bound).
template <int NP>
constexpr int blocked_nst() { return 2; }
template <int NW, int G, int NST = 2>
struct BStage {
  static constexpr int CH = 32;
  static constexpr int WORDS = (NW + 1) * CH + 4;
  static constexpr int RAW = NST * WORDS;
  static constexpr int WANT = (G >= 4 ? G : 4) % 32;
  static constexpr int STRIDE = RAW + (((WANT - RAW % 32) % 32) + 32) % 32;
};

// Host side: shared-memory bytes and launch shape of the blocked kernel for (R, BR).
struct BlockedShape {
  int G, VEC, CPL, TB;
  bool smem;
  int ncp;  // copies of the block in shared memory (0: outer rows from global memory)
  size_t block_bytes;
};
// Copies of the block that make the float4 row reads of a warp bank-conflict-free: rows of 4R
// bytes < 128 B share a bank line 128 / 4R at a time (R = 16: 2 copies, R = 8: 4).
constexpr int blocked_copies(int R) { return 4 * R < 128 ? 128 / (4 * R) : 1; }
// Shared-memory bytes of the block with ncp copies (copy k starts k rows past a 128-B boundary).
inline size_t blocked_block_bytes(int BR, int R, int ncp) {
  if (ncp <= 0) return 0;
  if (ncp == 1) return (size_t)BR * R * 4;
  return (size_t)ncp * (((size_t)BR * R + 31) / 32 * 32 + R) * 4;
}
// Staging bytes of a CTA of TB threads (lane-groups of G lanes, NW packed-word rows, NST stages).
inline size_t blocked_stage_bytes(int NW, int G, int TB, int NST) {
  const int words = (NW + 1) * 32 + 4, raw = NST * words, want = (G >= 4 ? G : 4) % 32;
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
  const int NW = NP >= 2 ? NP - 1 : 1, NST = 2;
  sh.smem = false;
  sh.ncp = 0;
  sh.TB = 256;
  if (vec_ok) {
    // copies of a narrow-row block only for one product mode (SpTTM, where each row read is the
    // only gather: 55.4 -> 52.7 us on brainq mode 1 at equal occupancy) and only where they keep
    // the CTAs per SM (occupancy outweighs the conflicts); SpMTTKRP at R = 16 measured 13% SLOWER
    // with copies (0.58 -> 0.67 ms, 2 CTAs/SM either way: the L1 left beside 2 x 108 KB of shared
    // memory), so its block stays single
    const int C = NP == 1 ? blocked_copies(R) : 1, want = NP == 1 ? 3 : 2;
    const size_t st256 = blocked_stage_bytes(NW, sh.G, 256, NST);
    auto ctas = [&](size_t bytes) { return std::min<int>(want, (int)((228 * 1024) / (bytes + st256 + 1024))); };
    if (C > 1 && ctas(blocked_block_bytes(BR, R, C)) >= ctas(sh.block_bytes) &&
        blocked_block_bytes(BR, R, C) + st256 <= 110 * 1024) {
      sh.smem = true;
      sh.ncp = C;
    } else if (sh.block_bytes + st256 <= 110 * 1024) {
      sh.smem = true;
      sh.ncp = 1;
    } else if (sh.block_bytes + blocked_stage_bytes(NW, sh.G, 512, NST) <= 220 * 1024) {
      sh.smem = true;
      sh.ncp = 1;
      sh.TB = 512;
    }
  }
  return sh;
}

template <int NP, class ACC>
cudaError_t launch_blocked_np(const BlockedParams& P, int nitems, bool vec_ok, cudaStream_t s);

}  // namespace fcoo
