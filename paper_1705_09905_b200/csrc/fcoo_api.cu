// fcoo_api.cu — the C ABI surface of libfcoo (include/fcoo.h): argument validation, status
// strings, allocator plumbing, handle metadata/export, sharding.
#include <stdarg.h>
#include <string.h>

#include <algorithm>

#include "fcoo_internal.cuh"

namespace fcoo {

std::atomic<uint64_t> g_launches{0};
static thread_local char t_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}

fcoo_status fail(fcoo_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return s;
}

void* Alloc::get(size_t bytes, cudaStream_t s) const {
  if (bytes == 0) return nullptr;
  if (custom) return a.alloc(bytes, (void*)s, a.ctx);
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void Alloc::put(void* p, size_t bytes, cudaStream_t s) const {
  if (!p) return;
  if (custom) a.free(p, bytes, (void*)s, a.ctx);
  else cudaFreeAsync(p, s);
}

fcoo_status build_impl(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, const fcoo_allocator* alloc,
                       cudaStream_t s, fcoo_t* out);
void destroy_impl(fcoo_s* f);

// fcoo_export of a blocked handle: decode the packed words into global product indices
// (outer = local + b*BR, last = low bits, middles as stored); padding positions give 0.
__global__ void k_unpack_blocked(const uint32_t* __restrict__ pk, const int64_t* __restrict__ blk_start,
                                 const int64_t* __restrict__ blk_end, int64_t nblocks, int64_t ns, int n_prod,
                                 int shift, int BR, uint32_t* __restrict__ pidx) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ns) return;
  int64_t lo = 0, hi = nblocks;  // blk_start[lo] <= q < blk_start[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (blk_start[mid] <= q) lo = mid; else hi = mid;
  }
  const bool live = q < blk_end[lo];
  const uint32_t w0 = pk[q];
  const uint32_t local = n_prod >= 2 ? (w0 >> shift) : w0;
  pidx[q] = live ? local + (uint32_t)(lo * BR) : 0u;
  if (n_prod >= 2) {
    for (int a = 1; a + 1 < n_prod; ++a) pidx[(int64_t)a * ns + q] = live ? pk[(int64_t)a * ns + q] : 0u;
    pidx[(int64_t)(n_prod - 1) * ns + q] = live ? (w0 & ((1u << shift) - 1u)) : 0u;
  }
}

}  // namespace fcoo

extern "C" {

const char* fcoo_status_str(fcoo_status s) {
  switch (s) {
    case FCOO_OK: return "FCOO_OK";
    case FCOO_ERR_ARG: return "FCOO_ERR_ARG";
    case FCOO_ERR_ORDER: return "FCOO_ERR_ORDER";
    case FCOO_ERR_MODE: return "FCOO_ERR_MODE";
    case FCOO_ERR_INDEX_RANGE: return "FCOO_ERR_INDEX_RANGE";
    case FCOO_ERR_DUPLICATE: return "FCOO_ERR_DUPLICATE";
    case FCOO_ERR_EMPTY: return "FCOO_ERR_EMPTY";
    case FCOO_ERR_KEY_BITS: return "FCOO_ERR_KEY_BITS";
    case FCOO_ERR_RANK: return "FCOO_ERR_RANK";
    case FCOO_ERR_SHAPE: return "FCOO_ERR_SHAPE";
    case FCOO_ERR_ALIGN: return "FCOO_ERR_ALIGN";
    case FCOO_ERR_OOM: return "FCOO_ERR_OOM";
    case FCOO_ERR_CUDA: return "FCOO_ERR_CUDA";
    case FCOO_ERR_NCCL: return "FCOO_ERR_NCCL";
    case FCOO_ERR_NOT_FINITE: return "FCOO_ERR_NOT_FINITE";
    case FCOO_ERR_IO: return "FCOO_ERR_IO";
  }
  return "FCOO_ERR_UNKNOWN";
}

const char* fcoo_last_error(void) { return fcoo::t_err; }

uint64_t fcoo_launch_count(void) { return fcoo::g_launches.load(); }

fcoo_status fcoo_build(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, const fcoo_allocator* alloc,
                       void* stream, fcoo_t* out) {
  return fcoo::build_impl(coo, mode, opts, alloc, (cudaStream_t)stream, out);
}

fcoo_status fcoo_build_sharded(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, fcoo_comm_t comm,
                               const fcoo_allocator* alloc, void* stream, fcoo_t* out) {
  if (!comm) return fcoo::fail(FCOO_ERR_ARG, "NULL comm");
  if (!out) return fcoo::fail(FCOO_ERR_ARG, "NULL out");
  int rank = 0, nranks = 1;
  fcoo::comm_rank_size(comm, &rank, &nranks);
  fcoo_t f = nullptr;
  fcoo_status st = fcoo::build_impl(coo, mode, opts, alloc, (cudaStream_t)stream, &f);
  if (st) return st;
  st = fcoo_set_shard(f, rank, nranks, comm);
  if (st) {
    fcoo_destroy(f);
    return st;
  }
  *out = f;
  return FCOO_OK;
}

fcoo_status fcoo_mttkrp(fcoo_t f, const float* const* factors, int R, float* out, void* stream) {
  if (!f || !factors || !out) return fcoo::fail(FCOO_ERR_ARG, "NULL handle/factors/out");
  if (f->op != FCOO_OP_MTTKRP) return fcoo::fail(FCOO_ERR_SHAPE, "handle was built for SpTTM");
  if (R < 1 || R > 256) return fcoo::fail(FCOO_ERR_RANK, "R=%d outside [1,256]", R);
  return fcoo::run_mttkrp(f, factors, R, out, (cudaStream_t)stream);
}

fcoo_status fcoo_mttkrp_mc(fcoo_t f, const float* const* factors, int R, fcoo_mc_t out, void* stream) {
  if (!f || !factors || !out) return fcoo::fail(FCOO_ERR_ARG, "NULL handle/factors/out");
  if (f->op != FCOO_OP_MTTKRP) return fcoo::fail(FCOO_ERR_SHAPE, "handle was built for SpTTM");
  if (R < 1 || R > 256) return fcoo::fail(FCOO_ERR_RANK, "R=%d outside [1,256]", R);
  return fcoo::run_mttkrp_mc(f, factors, R, out, (cudaStream_t)stream);
}

fcoo_status fcoo_ttm(fcoo_t f, const float* U, int R, float* out, void* stream) {
  if (!f || !U || !out) return fcoo::fail(FCOO_ERR_ARG, "NULL handle/U/out");
  if (R < 1 || R > 256) return fcoo::fail(FCOO_ERR_RANK, "R=%d outside [1,256]", R);
  if (f->op != FCOO_OP_TTM) {
    if (!f->fibre_flags) return fcoo::fail(FCOO_ERR_SHAPE, "handle was built for SpMTTKRP (without FCOO_BUILD_FIBRE_FLAGS)");
    return fcoo::run_ttm_fibres(f, U, R, out, (cudaStream_t)stream);
  }
  return fcoo::run_ttm(f, U, R, out, (cudaStream_t)stream);
}

fcoo_status fcoo_ttmc(fcoo_t f, const float* const* factors, const int* ranks, float* out, void* stream) {
  if (!f || !factors || !ranks || !out) return fcoo::fail(FCOO_ERR_ARG, "NULL handle/factors/ranks/out");
  if (f->op != FCOO_OP_MTTKRP) return fcoo::fail(FCOO_ERR_SHAPE, "SpTTMc needs a handle built for FCOO_OP_MTTKRP");
  if (f->blocked) return fcoo::fail(FCOO_ERR_SHAPE, "SpTTMc needs an unblocked handle (built without FCOO_BUILD_BLOCKED)");
  return fcoo::run_ttmc(f, factors, ranks, out, (cudaStream_t)stream);
}

fcoo_status fcoo_info(fcoo_t f, fcoo_info_t* info) {
  if (!f || !info) return fcoo::fail(FCOO_ERR_ARG, "NULL handle/info");
  memset(info, 0, sizeof(*info));
  info->order = f->order; info->op = f->op; info->mode = f->mode;
  info->n_idx = f->n_idx; info->n_prod = f->n_prod;
  for (int m = 0; m < fcoo::kMaxOrder; ++m) {
    info->idx_modes[m] = f->idx_modes[m];
    info->prod_modes[m] = f->prod_modes[m];
    info->dims[m] = f->dims[m];
  }
  info->nnz = f->nnz; info->nsegs = f->nsegs; info->ntiles = f->ntiles; info->tile_nnz = f->T;
  info->dense_rows = f->dense_rows;
  info->storage_bytes = (4 * (int64_t)f->n_prod + 4) * f->nnz + (f->nnz + 7) / 8 + 4 * ((f->ntiles + 31) / 32);
  info->seg_table_bytes = 4 * (f->ntiles + 1) + 4 * f->nsegs * f->n_idx;
  info->device_bytes = (int64_t)(f->bytes_pidx + f->bytes_val + f->bytes_bf + f->bytes_sf + f->bytes_seg_base +
                                 f->bytes_seg_coord + f->bytes_perm);
  info->shard = f->shard; info->nshards = f->nshards;
  info->tile_begin = f->tile_begin; info->tile_end = f->tile_end;
  info->blocked = f->blocked;
  info->block_rows = f->blocked ? f->block_rows : 0;
  info->nblocks = f->blocked ? f->nblocks : 0;
  info->nstream = f->blocked ? f->nnz_pad : f->nnz;
  info->pk_shift = f->pk_shift;
  info->n_words = f->n_words;
  if (f->blocked)  // packed words + values + bf over the padded stream, block tables
    info->device_bytes += (int64_t)(f->bytes_blk + f->bytes_seg_row + f->bytes_fib);
  info->nfib = f->op != FCOO_OP_TTM ? (f->fibre_flags ? f->nfib : 0) : f->blocked ? f->nfib : f->nsegs;
  info->fibre_flags = f->fibre_flags;
  if (f->fibre_flags) info->device_bytes += (int64_t)(f->bytes_l2 + f->bytes_fib);
  info->row_sharded = f->row_sharded;
  info->row_rank = f->row_rank;
  info->row_nranks = f->row_nranks;
  info->row_begin = f->row_sharded ? f->row_bounds[f->row_rank] : 0;
  info->row_end = f->row_sharded ? f->row_bounds[f->row_rank + 1] : f->dims[f->mode];
  return FCOO_OK;
}

fcoo_status fcoo_export(fcoo_t f, fcoo_host_view* v, void* stream) {
  if (!f || !v) return fcoo::fail(FCOO_ERR_ARG, "NULL handle/view");
  cudaStream_t s = (cudaStream_t)stream;
  if (f->blocked) {
    const int64_t ns = f->nnz_pad;
    if (v->perm) {
      if (!f->perm) return fcoo::fail(FCOO_ERR_ARG, "perm requested but the handle was built without KEEP_PERM");
      FCOO_CUDA_TRY(cudaMemcpyAsync(v->perm, f->perm, 4 * ns, cudaMemcpyDeviceToHost, s));
    }
    if (v->bf) FCOO_CUDA_TRY(cudaMemcpyAsync(v->bf, f->bf, (ns + 7) / 8, cudaMemcpyDeviceToHost, s));
    if (v->sf) FCOO_CUDA_TRY(cudaMemcpyAsync(v->sf, f->sf, 4 * ((f->ntiles + 31) / 32), cudaMemcpyDeviceToHost, s));
    if (v->seg_base) FCOO_CUDA_TRY(cudaMemcpyAsync(v->seg_base, f->seg_base, 4 * f->ntiles, cudaMemcpyDeviceToHost, s));
    if (v->seg_coord && f->nsegs > 0)
      FCOO_CUDA_TRY(cudaMemcpyAsync(v->seg_coord, f->seg_coord, 4 * f->nsegs * f->n_idx, cudaMemcpyDeviceToHost, s));
    if (v->val) FCOO_CUDA_TRY(cudaMemcpyAsync(v->val, f->val, 4 * ns, cudaMemcpyDeviceToHost, s));
    if (v->pk) FCOO_CUDA_TRY(cudaMemcpyAsync(v->pk, f->pidx, 4 * ns * f->n_words, cudaMemcpyDeviceToHost, s));
    if (v->blk_start) memcpy(v->blk_start, f->h_blk_start.data(), sizeof(int64_t) * (f->nblocks + 1));
    if (v->blk_end) memcpy(v->blk_end, f->h_blk_end.data(), sizeof(int64_t) * f->nblocks);
    if (f->op == FCOO_OP_TTM) {
      if (v->seg_row && f->nsegs > 0)
        FCOO_CUDA_TRY(cudaMemcpyAsync(v->seg_row, f->seg_row, 4 * f->nsegs, cudaMemcpyDeviceToHost, s));
      if (v->fib_coord && f->nfib > 0)
        FCOO_CUDA_TRY(cudaMemcpyAsync(v->fib_coord, f->fib_coord, 4 * f->nfib * f->n_idx, cudaMemcpyDeviceToHost, s));
    }
    if (v->pidx) {
      fcoo::Buf tmp(&f->alloc, sizeof(uint32_t) * (size_t)(ns * f->n_prod), s);
      if (!tmp.ok()) return fcoo::fail(FCOO_ERR_OOM, "export scratch");
      fcoo::k_unpack_blocked<<<(unsigned)((ns + 255) / 256), 256, 0, s>>>(
          f->pidx, f->blk_start, f->blk_end, f->nblocks, ns, f->n_prod, f->pk_shift, f->block_rows, tmp.as<uint32_t>());
      FCOO_LAUNCH_CHECK();
      FCOO_CUDA_TRY(cudaMemcpyAsync(v->pidx, tmp.p, 4 * ns * f->n_prod, cudaMemcpyDeviceToHost, s));
      FCOO_CUDA_TRY(cudaStreamSynchronize(s));
    }
    FCOO_CUDA_TRY(cudaStreamSynchronize(s));
    return FCOO_OK;
  }
  const int64_t nnz = f->nnz;
  if (v->perm) {
    if (!f->perm) return fcoo::fail(FCOO_ERR_ARG, "perm requested but the handle was built without KEEP_PERM");
    FCOO_CUDA_TRY(cudaMemcpyAsync(v->perm, f->perm, 4 * nnz, cudaMemcpyDeviceToHost, s));
  }
  if (v->bf) FCOO_CUDA_TRY(cudaMemcpyAsync(v->bf, f->bf, (nnz + 7) / 8, cudaMemcpyDeviceToHost, s));
  if (v->sf) FCOO_CUDA_TRY(cudaMemcpyAsync(v->sf, f->sf, 4 * ((f->ntiles + 31) / 32), cudaMemcpyDeviceToHost, s));
  if (v->seg_base) FCOO_CUDA_TRY(cudaMemcpyAsync(v->seg_base, f->seg_base, 4 * f->ntiles, cudaMemcpyDeviceToHost, s));
  if (v->seg_coord && f->nsegs > 0)
    FCOO_CUDA_TRY(cudaMemcpyAsync(v->seg_coord, f->seg_coord, 4 * f->nsegs * f->n_idx, cudaMemcpyDeviceToHost, s));
  if (v->pidx)
    for (int a = 0; a < f->n_prod; ++a)
      FCOO_CUDA_TRY(cudaMemcpyAsync(v->pidx + a * nnz, f->pidx + a * f->nnz_pad, 4 * nnz, cudaMemcpyDeviceToHost, s));
  if (v->val) FCOO_CUDA_TRY(cudaMemcpyAsync(v->val, f->val, 4 * nnz, cudaMemcpyDeviceToHost, s));
  if (f->op == FCOO_OP_TTM && v->fib_coord && f->nsegs > 0)  // plain SpTTM: the fibres are the segments
    FCOO_CUDA_TRY(cudaMemcpyAsync(v->fib_coord, f->seg_coord, 4 * f->nsegs * f->n_idx, cudaMemcpyDeviceToHost, s));
  if (f->fibre_flags) {  // second flag level of an MTTKRP handle
    if (v->bf2) FCOO_CUDA_TRY(cudaMemcpyAsync(v->bf2, f->bf2, (nnz + 7) / 8, cudaMemcpyDeviceToHost, s));
    if (v->fib_coord && f->nfib > 0)
      FCOO_CUDA_TRY(cudaMemcpyAsync(v->fib_coord, f->fib_coord, 4 * f->nfib * (f->order - 1), cudaMemcpyDeviceToHost, s));
  }
  FCOO_CUDA_TRY(cudaStreamSynchronize(s));
  return FCOO_OK;
}

fcoo_status fcoo_debug_flip_bit(fcoo_t f, int which, int64_t bit) {
  if (!f) return fcoo::fail(FCOO_ERR_ARG, "NULL handle");
  const int64_t n = which == 0 ? f->nnz_pad : which == 1 ? f->ntiles : -1;
  if (n < 0) return fcoo::fail(FCOO_ERR_ARG, "which must be 0 (bf) or 1 (sf)");
  if (bit < 0 || bit >= n) return fcoo::fail(FCOO_ERR_ARG, "bit %lld outside [0, %lld)", (long long)bit, (long long)n);
  uint32_t* word = (which == 0 ? f->bf : f->sf) + (bit >> 5);
  uint32_t w = 0;
  FCOO_CUDA_TRY(cudaMemcpy(&w, word, 4, cudaMemcpyDeviceToHost));
  if (which == 0 && !((w >> (bit & 31)) & 1u)) {  // setting: only to restore a head this call cleared
    auto it = std::find(f->debug_cleared.begin(), f->debug_cleared.end(), bit);
    if (it == f->debug_cleared.end())
      return fcoo::fail(FCOO_ERR_ARG, "setting a bf bit is not memory-safe (only cleared heads can be restored)");
    f->debug_cleared.erase(it);
  } else if (which == 0) {
    f->debug_cleared.push_back(bit);
  }
  if (which == 1 && f->op != FCOO_OP_MTTKRP)
    return fcoo::fail(FCOO_ERR_ARG, "sf flips are supported on MTTKRP handles only");
  w ^= 1u << (bit & 31);
  FCOO_CUDA_TRY(cudaMemcpy(word, &w, 4, cudaMemcpyHostToDevice));
  return FCOO_OK;
}

fcoo_status fcoo_destroy(fcoo_t f) {
  fcoo::destroy_impl(f);
  return FCOO_OK;
}

fcoo_status fcoo_shard_range(int64_t ntiles, int shard, int nshards, int64_t* begin, int64_t* end) {
  if (!begin || !end || ntiles < 0 || nshards < 1 || shard < 0 || shard >= nshards)
    return fcoo::fail(FCOO_ERR_ARG, "bad shard %d/%d of %lld tiles", shard, nshards, (long long)ntiles);
  *begin = ntiles * shard / nshards;
  *end = ntiles * (shard + 1) / nshards;
  return FCOO_OK;
}

fcoo_status fcoo_set_shard(fcoo_t f, int shard, int nshards, fcoo_comm_t comm) {
  if (!f) return fcoo::fail(FCOO_ERR_ARG, "NULL handle");
  int64_t b = 0, e = 0;
  fcoo_status st = fcoo_shard_range(f->ntiles, shard, nshards, &b, &e);
  if (st) return st;
  f->shard = shard;
  f->nshards = nshards;
  f->tile_begin = b;
  f->tile_end = e;
  if (f->row_sharded && nshards > 1) return fcoo::fail(FCOO_ERR_ARG, "handle is row-sharded (fcoo_set_row_shard)");
  f->comm = nshards > 1 ? comm : nullptr;
  return FCOO_OK;
}

}  // extern "C"
