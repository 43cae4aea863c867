// fcoo_internal.cuh — private declarations shared by the libfcoo translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler is attached

#include "fcoo.h"

namespace fcoo {

constexpr int kMaxOrder = 8;

// Thread-local detail message for fcoo_last_error().
void set_error(const char* fmt, ...);
fcoo_status fail(fcoo_status s, const char* fmt, ...);

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Device memory through the caller's allocator (or stream-ordered cudaMallocAsync).
struct Alloc {
  fcoo_allocator a{};
  bool custom = false;
  void* get(size_t bytes, cudaStream_t s) const;
  void put(void* p, size_t bytes, cudaStream_t s) const;
};

// NVTX phase range (SURVEY §5 tracing: build / kernel / collective / solve phases show up by name
// on an nsys or ncu --nvtx timeline); host-side, around the enqueue of the phase's work.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

struct Buf {  // RAII temp buffer
  const Alloc* al = nullptr;
  void* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  Buf() = default;
  Buf(const Alloc* a, size_t bytes, cudaStream_t st) : al(a), n(bytes), s(st) { p = bytes ? a->get(bytes, st) : nullptr; }
  ~Buf() { if (p) al->put(p, n, s); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  bool ok() const { return n == 0 || p != nullptr; }
};

}  // namespace fcoo

// The F-COO handle (layout in DESIGN.md "Data layout in HBM").
struct fcoo_s {
  int order = 0, op = 0, mode = 0, n_idx = 0, n_prod = 0;
  int idx_modes[fcoo::kMaxOrder] = {0}, prod_modes[fcoo::kMaxOrder] = {0};
  int64_t dims[fcoo::kMaxOrder] = {0};
  int64_t nnz = 0, nnz_pad = 0, ntiles = 0, nsegs = 0, T = 256;
  int dense_rows = 0;
  int deterministic = 0;  // FCOO_BUILD_DETERMINISTIC: tile partials + ordered combine, no red.add
  // device arrays
  uint32_t* pidx = nullptr;      // n_prod x nnz_pad (row a = product mode prod_modes[a])
  float* val = nullptr;          // nnz_pad
  uint32_t* bf = nullptr;        // nnz_pad / 32 words, LSB-first
  uint32_t* sf = nullptr;        // ceil(ntiles/32) words (+1)
  uint32_t* seg_base = nullptr;  // ntiles + 1 (last = nsegs)
  uint32_t* seg_coord = nullptr; // nsegs x n_idx
  uint32_t* perm = nullptr;      // nnz (KEEP_PERM only)
  size_t bytes_pidx = 0, bytes_val = 0, bytes_bf = 0, bytes_sf = 0, bytes_seg_base = 0, bytes_seg_coord = 0,
         bytes_perm = 0;
  // blocked layout (FCOO_BUILD_BLOCKED): pidx holds n_words packed words per
  // position (word 0: (i_outer - b*BR) << pk_shift | i_last; words 1..: middle product modes)
  int blocked = 0, block_rows = 0, pk_shift = 0, n_words = 0;
  int64_t nblocks = 0;
  int64_t* blk_start = nullptr;  // device [nblocks + 1]: first stream position of block b
  int64_t* blk_end = nullptr;    // device [nblocks]: end of block b's nonzeros
  size_t bytes_blk = 0;
  // blocked SpTTM handles (op TTM): the output rows are the fibres (distinct index tuples in
  // lexicographic order); seg_row[s] = fibre of blocked segment s, fib_coord = the tuples
  uint32_t* seg_row = nullptr;    // device [nsegs]
  uint32_t* fib_coord = nullptr;  // device [nfib x n_idx] (fibre-flag MTTKRP handles: [nfib x (order-1)])
  // second flag level (FCOO_BUILD_FIBRE_FLAGS, plain MTTKRP handles; Fig. 2): bf2 marks
  // the heads of fibres = (index tuple, every product coordinate but the last) on the same stream,
  // with its own tile flags and fibre ordinals, so fcoo_ttm runs SpTTM on the last product mode
  int fibre_flags = 0;
  uint32_t* bf2 = nullptr;        // nnz_pad / 32 words
  uint32_t* sf2 = nullptr;        // ceil(ntiles/32) words (+1)
  uint32_t* seg_base2 = nullptr;  // ntiles + 1
  size_t bytes_l2 = 0;
  int64_t nfib = 0;
  size_t bytes_seg_row = 0, bytes_fib = 0;
  std::vector<int64_t> h_blk_start, h_blk_end;  // host copies (work tables, export)
  // work items of the blocked SpMTTKRP, one table per groups-per-CTA value gpc = 1 << k (k < 10):
  // item = (block b, first tile t0), t0 = first tile of b + j*gpc; device int2 + host copy
  int2* items[10] = {nullptr};
  std::vector<int2> h_items[10];
  // deterministic handles: the per-tile boundary partials (2 x R x sizeof(ACC) per tile), kept
  // by the handle and grown on demand (fcoo::ensure_dpart) so no call allocates inside a CUDA
  // graph capture (cp_als reserves the largest size it needs before capturing)
  void* dpart = nullptr;
  size_t bytes_dpart = 0;
  std::vector<int64_t> debug_cleared;  // bf heads cleared by fcoo_debug_flip_bit (restorable)
  // shard
  int shard = 0, nshards = 1;
  int64_t tile_begin = 0, tile_end = 0;
  fcoo_comm_t comm = nullptr;
  // row shard (fcoo_set_row_shard / fcoo_build_distributed, SURVEY §8(e) owned-rows combine): the
  // handle holds only the nonzeros of index-mode rows [row_bounds[row_rank], row_bounds[row_rank+1]),
  // so its MTTKRP rows there are complete and the ranks' owned row ranges are all-gathered
  int row_sharded = 0, row_rank = 0, row_nranks = 1;
  std::vector<int64_t> row_bounds;
  fcoo_comm_t row_comm = nullptr;
  fcoo::Alloc alloc;
  cudaStream_t build_stream = nullptr;
  int device = 0;
};

namespace fcoo {
// engine entry points (fcoo_engine.cu)
// gate (device int, may be null): the launch works only if (*gate != 0) == gate_on
fcoo_status run_mttkrp(fcoo_s* f, const float* const* factors, int R, float* out, cudaStream_t s,
                       const int* gate = nullptr, int gate_on = 0);
fcoo_status run_mttkrp_f64(fcoo_s* f, const float* const* factors, int R, double* out, cudaStream_t s,
                           const int* gate = nullptr, int gate_on = 0);
// comm (fcoo_comm.cu)
fcoo_status comm_allreduce(fcoo_comm_t comm, float* buf, size_t count, cudaStream_t s);
fcoo_status comm_allreduce_f64(fcoo_comm_t comm, double* buf, size_t count, cudaStream_t s);
void comm_rank_size(fcoo_comm_t comm, int* rank, int* nranks);
fcoo_status comm_barrier(fcoo_comm_t comm, cudaStream_t s);
void mc_views(fcoo_mc_t m, float** uc, float** mc, size_t* bytes, fcoo_comm_t* comm);
fcoo_status run_mttkrp_mc(fcoo_s* f, const float* const* factors, int R, fcoo_mc_t out, cudaStream_t s);
fcoo_status run_ttm(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s);
// owned-rows combine of a row-sharded handle: rank k broadcasts rows [bounds[k], bounds[k+1]) of
// `out` (R columns) in one NCCL group, so every rank ends with the full output (fcoo_comm.cu)
fcoo_status comm_gather_rows(fcoo_comm_t comm, float* out, const std::vector<int64_t>& bounds, int R, cudaStream_t s);
fcoo_status comm_gather_rows_f64(fcoo_comm_t comm, double* out, const std::vector<int64_t>& bounds, int R,
                                 cudaStream_t s);
// distributed build helpers (fcoo_comm.cu): in-place sum of u32 counts; all-gather of nranks u64
// per rank; grouped send/recv of `elem` bytes per item (send[j]/recv[j] items to/from rank j)
fcoo_status comm_allreduce_u32(fcoo_comm_t comm, uint32_t* buf, size_t count, cudaStream_t s);
// every rank's status -> the largest (collective; a local failure stops all ranks together)
fcoo_status comm_agree(fcoo_comm_t comm, fcoo_status local, cudaStream_t s);
fcoo_status comm_allgather_u64(fcoo_comm_t comm, const uint64_t* send, uint64_t* recv, size_t count, cudaStream_t s);
fcoo_status comm_exchange(fcoo_comm_t comm, const void* sendbuf, const int64_t* send_counts, void* recvbuf,
                          const int64_t* recv_counts, size_t elem, cudaStream_t s);
// a handle for (op, mode) of a tensor with no nonzeros on this rank (distributed build); its
// SpMTTKRP output is all zero (fcoo_build.cu)
fcoo_status build_empty(int order, const int64_t* dims, int op, int mode, const fcoo_allocator* alloc, cudaStream_t s,
                        fcoo_t* out);
// SpTTM through the specialised kernel (fcoo_ttm.cu) when it applies; false = use the engine
bool run_ttm_lean(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s, fcoo_status* st);
// SpTTM on the last product mode of a fibre-flag MTTKRP handle (second flag level; fcoo_ttm.cu)
fcoo_status run_ttm_fibres(fcoo_s* f, const float* U, int R, float* out, cudaStream_t s);
fcoo_status zero_boundary_rows_f32(const uint32_t* sf, const uint32_t* seg_base, int64_t tile_begin, int64_t tile_end,
                                   int R, float* out, cudaStream_t s);
// deterministic handles: make f->dpart hold at least `bytes` (stream-ordered on s)
fcoo_status ensure_dpart(fcoo_s* f, size_t bytes, cudaStream_t s);
fcoo_status run_ttmc(fcoo_s* f, const float* const* factors, const int* ranks, float* out, cudaStream_t s);
}  // namespace fcoo

#define FCOO_CUDA_TRY(expr)                                                                         \
  do {                                                                                              \
    cudaError_t _e = (expr);                                                                        \
    if (_e != cudaSuccess)                                                                          \
      return fcoo::fail(FCOO_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
  } while (0)

#define FCOO_LAUNCH_CHECK()                                                                         \
  do {                                                                                              \
    fcoo::count_launch();                                                                           \
    cudaError_t _e = cudaGetLastError();                                                            \
    if (_e != cudaSuccess)                                                                          \
      return fcoo::fail(FCOO_ERR_CUDA, "%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
  } while (0)
