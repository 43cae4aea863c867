// fcoo_engine.cuh — declarations shared by the engine translation units.
#pragma once
#include "fcoo_internal.cuh"

namespace fcoo {

constexpr int kMaxProd = kMaxOrder - 1;

struct EngineParams {
  const uint32_t* pidx[kMaxProd];  // product index arrays, row stride nnz_pad
  const float* U[kMaxProd];        // factor matrix for product position a (I x R, row-major)
  const float* val;
  const uint32_t* bf;
  const uint32_t* sf;
  const uint32_t* seg_base;
  const uint32_t* seg_coord;       // row of segment s = seg_coord[s]; nullptr -> row = s
  int64_t nnz, ntiles, tile_begin, tile_end;
  int T, R;
  void* out;  // float* (fp32 accumulation) or double* (fp64 accumulation)
  // fused combine (fcoo_mttkrp_mc): multicast address of the output; segment
  // flushes go to every rank's copy with multimem.st / multimem.red.add (fp32 float4 path only)
  float* out_mc;
  // deterministic handles: per-tile partials of the shared segments, ACC[ntiles][2][R] (slot 0:
  // the tile's left-open first segment, slot 1: its own right-open last segment); nullptr = red.add
  void* dpart;
  // device-side gate (CP-ALS fit mode): when non-null the launch does its work only if
  // (*gate != 0) == gate_on, so the fp32/fp64 choice needs no host synchronisation
  const int* gate;
  int gate_on;
};

__device__ __forceinline__ bool gated_off(const EngineParams& P) {
  return P.gate && ((__ldg(P.gate) != 0) != (P.gate_on != 0));
}

// Launch the segmented-reduction kernel for NP product modes, accumulator type ACC (instantiated
// in fcoo_engine_np<NP>.cu so the template instances compile in parallel).
template <int NP, class ACC>
cudaError_t launch_np(const EngineParams& P, bool vec_ok, cudaStream_t s);

}  // namespace fcoo
