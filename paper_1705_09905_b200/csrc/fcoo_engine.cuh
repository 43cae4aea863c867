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
  // hot rows: a product index kHotTag | r reads row r of Uh[a] (the r-th most frequent row of
  // U[a], gathered per call); nullptr when the position has no tags
  const float* Uh[kMaxProd];
};

// Row address of product index w: tagged hot rows come from the contiguous hot copy.
__device__ __forceinline__ const char* row_ptr(const char* cold, const char* hot, uint32_t w, uint32_t rowb) {
  return (w & kHotTag) ? hot + (size_t)(w & ~kHotTag) * rowb : cold + (size_t)w * rowb;
}

// Per call: gather the hot rows of every tagged product position into f->uhot (fcoo_engine.cu).
fcoo_status prepare_hot(fcoo_s* f, const float* const* U, const int* R, const float** Uh, cudaStream_t s);

// Launch the segmented-reduction kernel for NP product modes, accumulator type ACC (instantiated
// in fcoo_engine_np<NP>.cu so the template instances compile in parallel).
template <int NP, class ACC>
cudaError_t launch_np(const EngineParams& P, bool vec_ok, cudaStream_t s);

}  // namespace fcoo
