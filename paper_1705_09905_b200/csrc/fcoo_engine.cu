// fcoo_engine.cu — host side of the segmented-reduction engine (see fcoo_engine_kernels.cuh):
// output preparation, kernel dispatch by (product-mode count, rank, accumulator type), and the
// SpMTTKRP / SpTTM entry points behind the C ABI.
#include <stdlib.h>

#include "fcoo_blocked.cuh"
#include "fcoo_engine.cuh"

namespace fcoo {

// Zero the output rows of segments that cross a tile boundary (they are combined by atomics);
// every other row is written exactly once by a plain store.  One thread per tile t: the segment
// seg_base[t]-1 crosses into t iff sf[t] == 0; it is zeroed only by the first tile it crosses
// into, i.e. when its head lies in tile t-1 (seg_base[t-1] != seg_base[t]).
template <class ACC>
__global__ void k_zero_boundary_rows(const uint32_t* __restrict__ sf, const uint32_t* __restrict__ seg_base,
                                     int64_t tile_begin, int64_t tile_end, int R, ACC* __restrict__ out) {
  int64_t t = tile_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tile_end || t == 0) return;
  const bool left_open = !((sf[t >> 5] >> (t & 31)) & 1u);
  if (!left_open || seg_base[t - 1] == seg_base[t]) return;
  ACC* o = out + ((int64_t)seg_base[t] - 1) * R;
  for (int c = 0; c < R; ++c) o[c] = ACC(0);
}

// Deterministic handles (FCOO_BUILD_DETERMINISTIC): one warp per tile t of the shard starts the
// ordered sum of every tile-crossing segment that begins in t (slot 1: t's own right-open last
// segment) or enters the shard at t = tile_begin (slot 0), adds slot 0 of each following tile the
// segment covers, in tile order, and stores the row; lanes stride over the R columns.
template <class ACC>
__global__ void k_combine_boundaries(const uint32_t* __restrict__ sf, const uint32_t* __restrict__ seg_base,
                                     const uint32_t* __restrict__ seg_coord, int64_t ntiles, int64_t tile_begin,
                                     int64_t tile_end, int R, const ACC* __restrict__ dpart, ACC* __restrict__ out,
                                     const int* gate, int gate_on) {
  const int64_t t = tile_begin + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (t >= tile_end) return;
  if (gate && ((__ldg(gate) != 0) != (gate_on != 0))) return;  // the gated-off MTTKRP wrote no partials
  auto sfbit = [&](int64_t u) { return (sf[u >> 5] >> (u & 31)) & 1u; };
  auto right_open = [&](int64_t u) { return u + 1 < ntiles && !sfbit(u + 1); };
  const uint32_t h0 = seg_base[t], h1 = seg_base[t + 1];  // heads before tile t / before t + 1
  for (int which = 0; which < 2; ++which) {
    uint32_t ord;
    bool cont;
    if (which == 0) {  // the shard's first tile, entered by a segment that began in an earlier shard
      if (!(t == tile_begin && t > 0 && !sfbit(t))) continue;
      ord = h0 - 1u;
      cont = (h1 == h0) && right_open(t);
    } else {  // a segment that starts in t and continues into t + 1
      if (!(h1 > h0 && right_open(t))) continue;
      ord = h1 - 1u;
      cont = true;
    }
    const int64_t row = seg_coord ? (int64_t)seg_coord[ord] : (int64_t)ord;
    for (int c = lane; c < R; c += 32) {
      ACC sum = dpart[((size_t)t * 2 + (which == 0 ? 0 : 1)) * (uint32_t)R + c];
      bool more = cont;
      for (int64_t u = t + 1; more && u < tile_end; ++u) {
        sum += dpart[(size_t)u * 2 * (uint32_t)R + c];
        more = (seg_base[u + 1] == seg_base[u]) && right_open(u);
      }
      out[row * R + c] = sum;
    }
  }
}

// rows of segments crossing a tile boundary (flag level sf / seg_base) set to 0 (see above)
fcoo_status zero_boundary_rows_f32(const uint32_t* sf, const uint32_t* seg_base, int64_t tile_begin, int64_t tile_end,
                                   int R, float* out, cudaStream_t s) {
  const int64_t nt = tile_end - tile_begin;
  if (nt <= 0) return FCOO_OK;
  k_zero_boundary_rows<float><<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(sf, seg_base, tile_begin, tile_end, R, out);
  FCOO_LAUNCH_CHECK();
  return FCOO_OK;
}

namespace {

template <class ACC>
fcoo_status combine_boundaries(fcoo_s* f, int R, const ACC* dpart, ACC* out, cudaStream_t s, const int* gate = nullptr,
                               int gate_on = 0) {
  const int64_t nt = f->tile_end - f->tile_begin;
  if (nt <= 0) return FCOO_OK;
  k_combine_boundaries<ACC><<<(unsigned)((nt * 32 + 255) / 256), 256, 0, s>>>(
      f->sf, f->seg_base, (f->op == FCOO_OP_MTTKRP && !f->dense_rows) ? f->seg_coord : nullptr, f->ntiles,
      f->tile_begin, f->tile_end, R, dpart, out, gate, gate_on);
  FCOO_LAUNCH_CHECK();
  return FCOO_OK;
}

template <class ACC>
cudaError_t launch_engine(const EngineParams& P, int NP, bool vec_ok, cudaStream_t s) {
  switch (NP) {
    case 1: return launch_np<1, ACC>(P, vec_ok, s);
    case 2: return launch_np<2, ACC>(P, vec_ok, s);
    case 3: return launch_np<3, ACC>(P, vec_ok, s);
    case 4: return launch_np<4, ACC>(P, vec_ok, s);
    case 5: return launch_np<5, ACC>(P, vec_ok, s);
    case 6: return launch_np<6, ACC>(P, vec_ok, s);
    default: return launch_np<7, ACC>(P, vec_ok, s);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }


template <class ACC>
fcoo_status prepare_output(fcoo_s* f, int R, ACC* out, int64_t rows, bool all_rows_are_segments, cudaStream_t s) {
  bool whole = (f->tile_begin == 0 && f->tile_end == f->ntiles);
  if (!all_rows_are_segments || !whole) {
    // empty rows (or rows owned by other shards) must read 0
    FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(ACC) * (size_t)(rows * R), s));
    return FCOO_OK;
  }
  int64_t nt = f->tile_end - f->tile_begin;
  if (nt > 0) {  // rows are segment ordinals here (TTM, or MTTKRP with every slice non-empty)
    k_zero_boundary_rows<ACC><<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(f->sf, f->seg_base, f->tile_begin,
                                                                         f->tile_end, R, out);
    FCOO_LAUNCH_CHECK();
  }
  return FCOO_OK;
}

}  // namespace

template <class ACC>
cudaError_t launch_blocked(const BlockedParams& P, int NP, int nitems, bool vec_ok, cudaStream_t s) {
  switch (NP) {
    case 1: return launch_blocked_np<1, ACC>(P, nitems, vec_ok, s);
    case 2: return launch_blocked_np<2, ACC>(P, nitems, vec_ok, s);
    case 3: return launch_blocked_np<3, ACC>(P, nitems, vec_ok, s);
    default: return launch_blocked_np<4, ACC>(P, nitems, vec_ok, s);
  }
}

// SpMTTKRP on a blocked handle (fcoo_blocked.cuh): zero the output (a row recurs once per block,
// every flush is a red.add), pick the work table for the launch shape, restrict it to the shard.
template <class ACC>
fcoo_status mttkrp_blocked(fcoo_s* f, const float* const* factors, int R, ACC* out, cudaStream_t s, const int* gate,
                           int gate_on, float* out_mc) {
  BlockedParams P{};
  bool vec_ok = (R % 4 == 0) && R <= 128 && aligned16(out);
  for (int a = 0; a < f->n_prod; ++a) {
    const int m = f->prod_modes[a];
    if (!factors[m]) return fail(FCOO_ERR_ARG, "factors[%d] is NULL", m);
    P.U[a] = factors[m];
    vec_ok = vec_ok && aligned16(factors[m]);
  }
  if (out_mc && (!vec_ok || !std::is_same<ACC, float>::value))
    return fail(FCOO_ERR_ARG, "fused combine needs the float4 path (R %% 4 == 0, R <= 128, aligned)");
  P.pk = f->pidx; P.val = f->val; P.bf = f->bf; P.sf = f->sf; P.seg_base = f->seg_base; P.seg_coord = f->seg_coord;
  P.blk_start = f->blk_start; P.blk_end = f->blk_end;
  P.nstream = f->nnz_pad; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.R = R; P.BR = f->block_rows; P.Io = (int)f->dims[f->prod_modes[0]]; P.shift = f->pk_shift;
  P.out = out; P.out_mc = out_mc; P.gate = gate; P.gate_on = gate_on;
  if (!out_mc) FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(ACC) * (size_t)f->dims[f->mode] * R, s));
  const BlockedShape sh = blocked_shape(f->n_prod, R, f->block_rows, vec_ok);
  int k = 0;
  while ((1 << k) < sh.TB / sh.G) ++k;
  const std::vector<int2>& items = f->h_items[k];
  // items whose tiles [t0, t0 + gpc) meet the shard's [tile_begin, tile_end) (sorted by t0)
  const int gpc = 1 << k;
  int64_t i0 = 0, i1 = (int64_t)items.size();
  while (i0 < i1 && (int64_t)items[i0].y + gpc <= f->tile_begin) ++i0;
  while (i1 > i0 && (int64_t)items[i1 - 1].y >= f->tile_end) --i1;
  P.items = f->items[k];
  P.item0 = i0;
  cudaError_t e = launch_blocked<ACC>(P, f->n_prod, (int)(i1 - i0), vec_ok, s);
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "blocked mttkrp launch: %s", cudaGetErrorString(e));
  return FCOO_OK;
}

template <class ACC>
fcoo_status mttkrp_t(fcoo_s* f, const float* const* factors, int R, ACC* out, cudaStream_t s,
                     const int* gate = nullptr, int gate_on = 0, float* out_mc = nullptr) {
  if (f->blocked) return mttkrp_blocked<ACC>(f, factors, R, out, s, gate, gate_on, out_mc);
  EngineParams P{};
  P.out_mc = out_mc;
  P.gate = gate;
  P.gate_on = gate_on;
  bool vec_ok = (R % 4 == 0) && R <= 128 && aligned16(out);
  for (int a = 0; a < f->n_prod; ++a) {
    int m = f->prod_modes[a];
    if (!factors[m]) return fail(FCOO_ERR_ARG, "factors[%d] is NULL", m);
    P.U[a] = factors[m];
    P.pidx[a] = f->pidx + (int64_t)a * f->nnz_pad;
    vec_ok = vec_ok && aligned16(factors[m]);
  }
  P.val = f->val; P.bf = f->bf; P.sf = f->sf; P.seg_base = f->seg_base;
  P.seg_coord = f->dense_rows ? nullptr : f->seg_coord;
  P.nnz = f->nnz; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.R = R; P.out = out;
  // all rows are segments (dense_rows): only tile-crossing rows need zeroing; the fused-combine
  // caller zeroes its (multicast-bound) buffer itself
  if (!out_mc) {
    fcoo_status st = prepare_output<ACC>(f, R, out, f->dims[f->mode], f->dense_rows != 0, s);
    if (st) return st;
  } else if (!vec_ok || R < 16 || f->n_prod < 2) {  // the staged float4 kernel (G = R/4 >= 4 lanes)
    return fail(FCOO_ERR_ARG, "fused combine needs the staged float4 engine (order >= 3, R %% 4 == 0, 16 <= R <= 128, aligned)");
  }
  if (f->deterministic) {
    fcoo_status st = ensure_dpart(f, sizeof(ACC) * (size_t)f->ntiles * 2 * (size_t)R, s);
    if (st) return st;
  }
  P.dpart = f->deterministic ? f->dpart : nullptr;
  cudaError_t e = launch_engine<ACC>(P, f->n_prod, vec_ok, s);
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "mttkrp launch: %s", cudaGetErrorString(e));
  if (f->deterministic) return combine_boundaries<ACC>(f, R, reinterpret_cast<const ACC*>(f->dpart), out, s, gate, gate_on);
  return FCOO_OK;
}

fcoo_status ensure_dpart(fcoo_s* f, size_t bytes, cudaStream_t s) {
  if (f->bytes_dpart >= bytes) return FCOO_OK;
  if (f->dpart) f->alloc.put(f->dpart, f->bytes_dpart, s);
  f->dpart = f->alloc.get(bytes, s);
  f->bytes_dpart = f->dpart ? bytes : 0;
  if (!f->dpart) return fail(FCOO_ERR_OOM, "deterministic partials (%zu bytes)", bytes);
  return FCOO_OK;
}

fcoo_status run_mttkrp(fcoo_s* f, const float* const* factors, int R, float* out, cudaStream_t s, const int* gate,
                       int gate_on) {
  Nvtx range("fcoo_mttkrp");
  fcoo_status st = FCOO_OK;
  if (f->nnz == 0)  // a row shard that received no nonzeros (distributed build)
    FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)f->dims[f->mode] * R, s));
  else
    st = mttkrp_t<float>(f, factors, R, out, s, gate, gate_on);
  if (st) return st;
  if (f->comm) return comm_allreduce(f->comm, out, (size_t)f->dims[f->mode] * R, s);
  if (f->row_comm) return comm_gather_rows(f->row_comm, out, f->row_bounds, R, s);
  return FCOO_OK;
}

// SpMTTKRP with the cross-rank combine fused into the epilogue: zero the local
// copy, barrier, kernel writing through the multicast address, barrier.
fcoo_status run_mttkrp_mc(fcoo_s* f, const float* const* factors, int R, fcoo_mc_t mc, cudaStream_t s) {
  float *uc = nullptr, *mcp = nullptr;
  size_t bytes = 0;
  fcoo_comm_t comm = nullptr;
  mc_views(mc, &uc, &mcp, &bytes, &comm);
  if (f->row_sharded || f->nnz == 0) return fail(FCOO_ERR_ARG, "fused combine: row-sharded handle (use fcoo_mttkrp)");
  const size_t need = sizeof(float) * (size_t)f->dims[f->mode] * (size_t)R;
  if (bytes < need) return fail(FCOO_ERR_ARG, "multicast buffer holds %zu bytes, output needs %zu", bytes, need);
  if (f->comm && f->comm != comm) return fail(FCOO_ERR_ARG, "handle sharded over a different comm");
  {  // every rank must process exactly its own shard, or shared rows would be added nranks times
    int rank = 0, nranks = 1;
    comm_rank_size(comm, &rank, &nranks);
    if (f->nshards != nranks || f->shard != rank)
      return fail(FCOO_ERR_ARG, "fused combine: handle shard %d/%d does not match comm rank %d/%d", f->shard,
                  f->nshards, rank, nranks);
  }
  if (f->deterministic) return fail(FCOO_ERR_ARG, "fused combine: the multicast reduction order is not fixed (deterministic handle)");
  FCOO_CUDA_TRY(cudaMemsetAsync(uc, 0, need, s));
  fcoo_status st = comm_barrier(comm, s);
  if (st) return st;
  st = mttkrp_t<float>(f, factors, R, uc, s, nullptr, 0, mcp);
  if (st) return st;
  return comm_barrier(comm, s);
}

// fp64-accumulating MTTKRP (CP-ALS fit mode); sharded handles return the LOCAL partial.
fcoo_status run_mttkrp_f64(fcoo_s* f, const float* const* factors, int R, double* out, cudaStream_t s,
                           const int* gate, int gate_on) {
  Nvtx range("fcoo_mttkrp_f64");
  if (f->nnz == 0) {
    FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)f->dims[f->mode] * R, s));
    return FCOO_OK;
  }
  return mttkrp_t<double>(f, factors, R, out, s, gate, gate_on);
}

// SpTTM on a blocked handle (FCOO_BUILD_BLOCKED, op TTM): the blocked kernel with one product
// mode (the outer = last = mode n, U's block of BR rows in shared memory); segment s flushes into
// its fibre's row seg_row[s] with red.add, so the nfib x R output is zeroed first.
fcoo_status ttm_blocked(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s) {
  BlockedParams P{};
  const bool vec_ok = (R % 4 == 0) && R <= 128 && aligned16(out) && aligned16(U);
  P.U[0] = U;
  P.pk = f->pidx; P.val = f->val; P.bf = f->bf; P.sf = f->sf; P.seg_base = f->seg_base; P.seg_coord = f->seg_row;
  P.blk_start = f->blk_start; P.blk_end = f->blk_end;
  P.nstream = f->nnz_pad; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.R = R; P.BR = f->block_rows; P.Io = (int)f->dims[f->mode]; P.shift = 0;
  P.out = out;
  FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)f->nfib * R, s));
  const BlockedShape sh = blocked_shape(1, R, f->block_rows, vec_ok);
  int k = 0;
  while ((1 << k) < sh.TB / sh.G) ++k;
  const std::vector<int2>& items = f->h_items[k];
  const int gpc = 1 << k;
  int64_t i0 = 0, i1 = (int64_t)items.size();
  while (i0 < i1 && (int64_t)items[i0].y + gpc <= f->tile_begin) ++i0;
  while (i1 > i0 && (int64_t)items[i1 - 1].y >= f->tile_end) --i1;
  P.items = f->items[k];
  P.item0 = i0;
  cudaError_t e = launch_blocked<float>(P, 1, (int)(i1 - i0), vec_ok, s);
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "blocked ttm launch: %s", cudaGetErrorString(e));
  if (f->comm) return comm_allreduce(f->comm, out, (size_t)f->nfib * R, s);
  return FCOO_OK;
}

fcoo_status run_ttm(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s) {
  Nvtx range("fcoo_ttm");
  if (f->blocked) return ttm_blocked(f, U, R, out, s);
  EngineParams P{};
  bool vec_ok = (R % 4 == 0) && R <= 128 && aligned16(out) && aligned16(U);
  P.U[0] = U;
  P.pidx[0] = f->pidx;
  P.val = f->val; P.bf = f->bf; P.sf = f->sf; P.seg_base = f->seg_base;
  P.seg_coord = nullptr;  // output row = fibre (segment) ordinal
  P.nnz = f->nnz; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.R = R; P.out = out;
  fcoo_status st = prepare_output<float>(f, R, out, f->nsegs, true, s);
  if (st) return st;
  if (run_ttm_lean(f, U, R, out, s, &st)) {  // fcoo_ttm.cu: the specialised SpTTM kernel
    if (st) return st;
    if (f->comm) return comm_allreduce(f->comm, out, (size_t)f->nsegs * R, s);
    return FCOO_OK;
  }
  if (f->deterministic) {
    st = ensure_dpart(f, sizeof(float) * (size_t)f->ntiles * 2 * (size_t)R, s);
    if (st) return st;
  }
  P.dpart = f->deterministic ? f->dpart : nullptr;
  cudaError_t e = launch_engine<float>(P, 1, vec_ok, s);
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "ttm launch: %s", cudaGetErrorString(e));
  if (f->deterministic) {
    st = combine_boundaries<float>(f, R, reinterpret_cast<const float*>(f->dpart), out, s);
    if (st) return st;
  }
  if (f->comm) return comm_allreduce(f->comm, out, (size_t)f->nsegs * R, s);
  return FCOO_OK;
}

}  // namespace fcoo
