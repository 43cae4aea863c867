/*
 * fcoo.h — C ABI of libfcoo, a B200-native (sm_100a) implementation of the F-COO hot path of
 * Liu, Wen, Sarwate, Dehnavi, "A Unified Optimization Approach for Sparse Tensor Operations on
 * GPUs" (arXiv 1705.09905).  Citations: P:Lnnn = /root/reference/PAPER.md line (section / eq.).
 *
 * Conventions
 *   - Modes are 0-based (the paper is 1-based).  Rank R is the number of factor columns.
 *   - "device" = a CUDA device pointer on the current device; "host" = host memory.
 *   - Every call that launches work enqueues it on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream) and returns without synchronising, except where stated.
 *   - Outputs are overwritten, never accumulated.  Rows of an MTTKRP output with no nonzeros
 *     are exactly 0.
 *   - Errors are returned as fcoo_status; nothing is thrown across the ABI and nothing exits.
 *     Host-checkable errors return before any launch.  fcoo_last_error() gives a
 *     thread-local detail string for the last failure.
 *   - Floating point: fp32 storage and fp32 accumulation (the paper's single precision,
 *     P:L272 Table II caption); the CP-ALS R x R algebra is done in fp64.
 */
#ifndef FCOO_H
#define FCOO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The numeric values 0..6 coincide with the oracle's own enum (oracle/). */
typedef enum {
  FCOO_OK = 0,
  FCOO_ERR_ARG = 1,         /* NULL pointer, bad size, bad option */
  FCOO_ERR_ORDER = 2,       /* order outside [2, 8] */
  FCOO_ERR_MODE = 3,        /* mode >= order */
  FCOO_ERR_INDEX_RANGE = 4, /* some idx[m][q] >= dims[m] (detected on device) */
  FCOO_ERR_DUPLICATE = 5,   /* two nonzeros share all coordinates (detected on device) */
  FCOO_ERR_EMPTY = 6,       /* nnz == 0 */
  FCOO_ERR_KEY_BITS = 7,    /* sum_m ceil(log2 dims[m]) > 128: sort key does not fit (<= 64: u64 keys, else u128) */
  FCOO_ERR_RANK = 8,        /* R outside [1, 256] */
  FCOO_ERR_SHAPE = 9,       /* op/handle mismatch (e.g. fcoo_ttm on an MTTKRP handle) */
  FCOO_ERR_ALIGN = 10,      /* reserved */
  FCOO_ERR_OOM = 11,        /* device allocation failed */
  FCOO_ERR_CUDA = 12,       /* CUDA launch / runtime error */
  FCOO_ERR_NCCL = 13,       /* NCCL error */
  FCOO_ERR_NOT_FINITE = 14, /* reserved */
  FCOO_ERR_IO = 15          /* .tns file: cannot open/read/write, or a malformed line */
} fcoo_status;

/* Operation a handle is built for: Table I.
 *   FCOO_OP_MTTKRP on mode n: index mode {n}; product modes = all others (Eq.(6)).
 *   FCOO_OP_TTM    on mode n: product mode {n}; index modes = all others (Eq.(3)). */
typedef enum { FCOO_OP_MTTKRP = 0, FCOO_OP_TTM = 1 } fcoo_op;

/* COO input.  Borrowed: must stay valid until the stream work of the call
 * that reads it completes.  Coordinates are 0-based; duplicates are an error (reading Q6). */
typedef struct {
  int order;                   /* N, 2..8 */
  const int64_t* dims;         /* host [order]; 1 <= dims[m] < 2^32 */
  int64_t nnz;                 /* >= 1, < 2^32 */
  const uint32_t* const* idx;  /* host array of `order` DEVICE pointers, idx[m][q] (SoA) */
  const float* val;            /* device [nnz] */
} fcoo_coo;

/* Optional device allocator (the Python binding passes torch's caching allocator).
 * NULL -> cudaMallocAsync / cudaFreeAsync on the call's stream. */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* ctx);
  void (*free)(void* ptr, size_t bytes, void* stream, void* ctx);
  void* ctx;
} fcoo_allocator;

#define FCOO_BUILD_KEEP_PERM 1u /* keep the sorted->input permutation for fcoo_export */
/* Order the product modes of an MTTKRP handle by DESCENDING extent (ties by mode id) instead of
 * the default ascending order of reading Q5: the last (per-nonzero random) product mode is then
 * the smallest factor.  Same segments, same sum, another canonical permutation. */
#define FCOO_BUILD_PRODUCT_DESC 2u
/* Bitwise-reproducible SpMTTKRP / SpTTM on this handle (SURVEY §8(b) DETERMINISTIC): instead of
 * red.global.add, a tile writes the partial sums of the (at most two) segments it shares with its
 * neighbours to a per-call scratch array (2 x R per tile, through the handle's allocator), and a
 * second kernel adds the partials of each tile-crossing segment in tile order and stores the row.
 * Same sum, a fixed association: repeated calls give identical bits (also the CP-ALS fit-mode
 * fp64 pass on such handles).  SpTTMc keeps red.add. */
#define FCOO_BUILD_DETERMINISTIC 4u
/* Blocked F-COO (reading Q22): the stream is the concatenation,
 * over b = 0, 1, ..., of the F-COO of the sub-tensor X_b = {nonzeros with floor(i_outer / BR) == b},
 * "outer" = the first product mode of reading Q5 (smallest extent), BR = block_rows; each block is
 * padded with empty positions to a multiple of T, so every tile belongs to one block.  Eq.(6) is
 * linear in X, so MTTKRP(X) = sum_b MTTKRP(X_b): the SpMTTKRP kernel keeps block b's BR outer
 * factor rows in shared memory (one TMA bulk copy per CTA) and gathers only the other product
 * modes from L2; every segment flush is a red.global.add (a row recurs once per block).
 * Per nonzero the stream holds ONE packed word (i_outer - b*BR) << IB | i_last (IB =
 * ceil(log2 I_last), "last" = last product mode of Q5; order 2: the local outer index alone),
 * plus, for order >= 4, the global index of each middle product mode: 8 B/nnz + flags for a
 * 3-order tensor instead of Table II's 12.  FCOO_OP_TTM: the one product mode n is blocked (the
 * word is i_n - b*BR); segments are (block, fibre) pairs, mapped to the fibre table (output rows)
 * by a sort of the segments' tuples.  Requires 2 <= order <= 5 and ceil(log2 BR) + IB <= 32 (else
 * FCOO_ERR_ARG); incompatible with DETERMINISTIC and PRODUCT_DESC (ARG); fcoo_ttmc rejects blocked
 * handles (SHAPE).  The build synchronises the host twice (block sizes, then errors), a TTM build
 * three times (then the fibre count). */
#define FCOO_BUILD_BLOCKED 8u
/* Second flag level (FCOO_OP_MTTKRP, plain layout, order >= 3; Fig. 2: "one F-COO
 * serves TTM-3 and MTTKRP-1"): besides bf (slice heads), the build marks in bf2 the heads of the
 * FIBRES of the same sorted stream -- (index tuple, every product coordinate but the last) -- with
 * their own tile flags sf2, ordinals and fibre table, so that fcoo_ttm on this MTTKRP handle runs
 * SpTTM (Eq.(3)) on the handle's LAST product mode (prod_modes[n_prod-1]) without a second build.
 * Excludes BLOCKED and DETERMINISTIC (ARG). */
#define FCOO_BUILD_FIBRE_FLAGS 16u

/* Build options.  NULL -> {FCOO_OP_MTTKRP, 0 (automatic), 0}.
 * tile_nnz = T, the partition length ("threadlen", P:L272 / P:L426): a multiple of 32 in
 * [32, 8192], or 0 = automatic (enough tiles to fill the GPU ~4x at R=32: about nnz/37888,
 * rounded to the nearest power of two in [32, 2048]; fcoo_info reports the value used).
 * sf has one bit per tile; one GPU lane-group processes one tile. */
typedef struct {
  int op;          /* fcoo_op */
  int tile_nnz;    /* T */
  unsigned flags;  /* FCOO_BUILD_* */
  int block_rows;  /* BR for FCOO_BUILD_BLOCKED: 0 = 512; otherwise in [32, 65536] (ignored without the flag) */
} fcoo_build_opts;

typedef struct fcoo_s* fcoo_t;
typedef struct fcoo_comm_s* fcoo_comm_t;
typedef struct fcoo_mc_s* fcoo_mc_t;

/*
 * fcoo_build — F-COO format for (op, mode) (§IV-B, Fig. 2; Table II).
 * Sorts the nonzeros on the device with the index modes as major key (ascending mode order)
 * and the product modes as minor keys in ascending extent order (reading Q5), then writes:
 *   product-mode index arrays and values in sorted order ("only keeps the indices on the
 *   product mode"), bf (1 bit per nonzero, 1 = first nonzero of a new index tuple, i.e. a new
 *   slice/fibre; reading Q1), sf (1 bit per tile: sf[t] = bf[t*T]; reading Q3), and
 *   the segment tables seg_base[t] (heads before tile t) and seg_coord[s] (index tuple of
 *   segment s) which the paper leaves implicit (reading Q4).
 * Inputs are device arrays (see fcoo_coo).  Performs ONE host synchronisation on `stream` to
 * report data errors (INDEX_RANGE, DUPLICATE) and to size the segment table; on success *out
 * owns all its device memory (allocated through `alloc`) until fcoo_destroy.  The result is a
 * pure function of the input (bit-exact against the oracle build).
 */
fcoo_status fcoo_build(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, const fcoo_allocator* alloc,
                       void* stream, fcoo_t* out);

/*
 * fcoo_mttkrp — SpMTTKRP on the handle's mode n, one-shot (§IV-C, Eq.(6)):
 *   out(i_n, :) = sum_{nonzeros q of slice i_n} v_q * Hadamard_{m != n} factors[m](i_m(q), :)
 * as a flag-driven segmented reduction: each lane-group walks one tile of T
 * nonzeros, gathers the product-mode factor rows (fp32 row-major I_m x R, 16-B aligned rows on
 * the vector path when R % 4 == 0), accumulates in registers, stores segments it owns and uses
 * red.global.add only for the (at most two) segments it shares with a neighbouring tile.
 *   factors: host array of `order` DEVICE pointers; factors[n] is ignored (may be NULL).
 *   R: 1..256.  out: device, I_n x R fp32 row-major, overwritten.
 * On a sharded handle (fcoo_set_shard) only the shard's tiles are processed; with a comm the
 * partial outputs are summed by an NCCL all-reduce so every rank holds the full result.
 * Errors: SHAPE (handle built for TTM), RANK, ARG, CUDA, NCCL.  Asynchronous.
 */
fcoo_status fcoo_mttkrp(fcoo_t f, const float* const* factors, int R, float* out, void* stream);

/*
 * fcoo_ttm — SpTTM on the handle's mode n (Eq.(3); Table I row 1):
 *   out(s, :) = sum_{nonzeros q of fibre s} v_q * U(i_n(q), :)
 * on the same segmented-reduction engine.  Output is semi-sparse: one dense R-row
 * per non-empty fibre s (in lexicographic order of the index tuple); the fibre coordinates are
 * the fib_coord table (fcoo_export; = seg_coord on a plain handle).  On a blocked handle
 * (FCOO_BUILD_BLOCKED) the kernel keeps block b of U (BR rows) in shared memory and every
 * (block, fibre) segment is added into its fibre's row with red.global.add.
 *   U: device, I_n x R fp32 row-major.  out: device, nfib x R fp32 (fcoo_info), overwritten.
 * On an MTTKRP handle built with FCOO_BUILD_FIBRE_FLAGS the same call runs SpTTM on the handle's
 * last product mode m = prod_modes[n_prod-1] from the second flag level: U is I_m x R, out is
 * nfib x R with one row per fibre in the stream's key order (fib_coord: index mode, then the other
 * product modes in prod_modes order); it needs R % 4 == 0, R/4 a power of two <= 32, and 16-byte
 * aligned U and out (else ARG).
 * Errors: SHAPE (MTTKRP handle without the second flag level), RANK, ARG, CUDA, NCCL.  Asynchronous.
 */
fcoo_status fcoo_ttm(fcoo_t f, const float* U, int R, float* out, void* stream);

/*
 * fcoo_ttmc — SpTTMc (tensor times matrix chain, the Tucker/HOOI kernel) on the handle's mode n,
 * Eq.(4) (Table I row 3): same index-mode segments as SpMTTKRP, Kronecker
 * instead of Hadamard product of the product-mode rows:
 *   out(i_n, :) = sum_{nonzeros q of slice i_n} v_q * (U_a(i_a(q), :) (x) U_b(i_b(q), :)),
 * a < b the two other modes in ascending mode order (Eq.(1) Kronecker layout: column p*R_b + q).
 *   f: a handle built with FCOO_OP_MTTKRP on an order-3 tensor (else SHAPE / ORDER).
 *   factors: host array of `order` DEVICE pointers, factors[m] is I_m x ranks[m] fp32 row-major
 *   (factors[n] ignored).  ranks: host [order]; R_a * R_b <= 1024 (else RANK).
 *   out: device, I_n x (R_a*R_b) fp32 row-major, overwritten.  Asynchronous.
 */
fcoo_status fcoo_ttmc(fcoo_t f, const float* const* factors, const int* ranks, float* out, void* stream);

typedef struct {
  int order, op, mode;
  int n_idx, n_prod;
  int idx_modes[8], prod_modes[8]; /* prod_modes in stored (ascending extent) order */
  int64_t dims[8];
  int64_t nnz, nsegs, ntiles, tile_nnz;
  int dense_rows;          /* MTTKRP with every slice non-empty: seg_coord is the identity */
  int64_t storage_bytes;   /* Table II core bytes: (4*n_prod+4)*nnz + ceil(nnz/8) + 4*ceil(ntiles/32) */
  int64_t seg_table_bytes; /* seg_base + seg_coord bytes (reading Q4) */
  int64_t device_bytes;    /* everything the handle holds on the device (with padding) */
  int shard, nshards;      /* tile range in use: [tile_begin, tile_end) */
  int64_t tile_begin, tile_end;
  int blocked;             /* built with FCOO_BUILD_BLOCKED */
  int block_rows;          /* BR (blocked handles; 0 otherwise) */
  int64_t nblocks;         /* ceil(I_outer / BR) (blocked handles; 0 otherwise) */
  int64_t nstream;         /* stream positions (blocked: nnz + padding = ntiles * tile_nnz; else nnz) */
  int pk_shift;            /* IB of the packed word (blocked handles) */
  int n_words;             /* packed words per nonzero (blocked handles: 1 + max(0, n_prod - 2)) */
  int64_t nfib;            /* SpTTM handles: output rows = fibres (non-empty index tuples); = nsegs for a
                              plain handle, <= nsegs for a blocked one (a fibre recurs once per block); MTTKRP
                              handles: the fibres of the second flag level (FCOO_BUILD_FIBRE_FLAGS), else 0 */
  int row_sharded;         /* fcoo_set_row_shard / fcoo_build_distributed with nranks > 1 */
  int row_rank, row_nranks;
  int64_t row_begin, row_end; /* index-mode rows this handle holds ([0, I_n) when not row-sharded) */
  int fibre_flags;         /* built with FCOO_BUILD_FIBRE_FLAGS (second flag level) */
} fcoo_info_t;

/* fcoo_info — host-side metadata; no device work. */
fcoo_status fcoo_info(fcoo_t f, fcoo_info_t* info);

/* Host view for fcoo_export: each non-NULL pointer receives a copy (host memory, caller-owned).
 * Sizes (S = fcoo_info nstream: nnz, or nnz + padding for a blocked handle):
 * perm u32[S] (only with FCOO_BUILD_KEEP_PERM; 0xFFFFFFFF at padding), bf u8[ceil(S/8)]
 * (LSB-first, pad 0), sf u32[ceil(ntiles/32)], seg_base u32[ntiles], seg_coord u32[nsegs*n_idx],
 * pidx u32[n_prod*S] (product modes in prod_modes order, GLOBAL indices; a blocked handle's packed
 * words are decoded on the device; 0 at padding), val f32[S] (0 at padding);
 * blocked handles only: pk u32[n_words*S] (the packed words as stored), blk_start i64[nblocks+1]
 * (first stream position of each block; last = S), blk_end i64[nblocks] (end of its nonzeros). */
typedef struct {
  uint32_t* perm;
  uint8_t* bf;
  uint32_t* sf;
  uint32_t* seg_base;
  uint32_t* seg_coord;
  uint32_t* pidx;
  float* val;
  uint32_t* pk;
  int64_t* blk_start;
  int64_t* blk_end;
  uint32_t* seg_row;   /* blocked SpTTM handles: u32[nsegs], the fibre (output row) of each segment */
  uint32_t* fib_coord; /* SpTTM handles: u32[nfib*n_idx], the index tuple of each output row (plain: = seg_coord);
                          fibre-flag MTTKRP handles: u32[nfib*(order-1)] (index mode, then prod_modes but the last) */
  uint8_t* bf2;        /* fibre-flag MTTKRP handles: the second flag level, u8[ceil(S/8)] (LSB-first) */
} fcoo_host_view;

/* fcoo_export — copy the handle's arrays to host buffers; synchronises `stream`. */
fcoo_status fcoo_export(fcoo_t f, fcoo_host_view* view, void* stream);

/* fcoo_debug_flip_bit — TEST SUPPORT: flip bit `bit` of the handle's device
 * bf array (which = 0; bit < stream length) or sf array (which = 1; bit < ntiles), synchronously, so
 * a test can show that the parity checks detect a corrupted flag.  The handle's results are wrong
 * afterwards (flip the same bit again to restore it).  Only flips that keep every kernel
 * memory-safe are allowed: clearing a bf head (a segment ordinal can only lag) and restoring a head
 * cleared this way, and flipping an sf bit of an MTTKRP handle; setting any other bf bit or touching
 * sf of an SpTTM handle could index past the segment table and is rejected (ARG).  Errors: ARG (NULL, bit out of range, which not 0/1, a
 * rejected flip), CUDA. */
fcoo_status fcoo_debug_flip_bit(fcoo_t f, int which, int64_t bit);

/* fcoo_destroy — free the handle (stream-ordered frees on the build stream). NULL is OK. */
fcoo_status fcoo_destroy(fcoo_t f);

/* ---- multi-GPU ("multiple-GPUs can be used") ----
 * One process per GPU.  Rank 0 calls fcoo_comm_unique_id and broadcasts the 128 bytes (the
 * Python binding uses torch.distributed); every rank calls fcoo_comm_init with its device current
 * (collective: NCCL communicator init, also for nranks == 1, so the NCCL path can be exercised on
 * one GPU; handles never attach a 1-rank comm).  Errors: ARG, OOM, NCCL.  fcoo_comm_destroy frees
 * it (NULL is OK); no handle or multicast buffer may still use it. */
fcoo_status fcoo_comm_unique_id(void* out128);
fcoo_status fcoo_comm_init(int rank, int nranks, const void* uid128, fcoo_comm_t* out);
fcoo_status fcoo_comm_destroy(fcoo_comm_t comm);
/* In-place sum all-reduce of `count` fp32 values on `stream` (NCCL over NVLink/NVSwitch). */
fcoo_status fcoo_allreduce_sum(fcoo_comm_t comm, float* buf, size_t count, void* stream);

/* ---- collective fused into the SpMTTKRP epilogue (P:L369 multi-GPU) ----
 * fcoo_mc_alloc — COLLECTIVE over `comm` (every rank calls it with the same `bytes`): each rank
 * allocates `bytes` (rounded up to the multicast granularity) of its own device memory and binds
 * it to one NVLink-SHARP multicast object shared by all ranks (created on rank 0, exported as a
 * fabric handle and broadcast over the comm's NCCL communicator).  A 1-rank comm gives a
 * one-device multicast object.  Errors: ARG (NULL/zero, comm without NCCL, device without
 * multicast support), OOM, CUDA, NCCL.  Synchronises the host (setup, not the timed path).
 * fcoo_mc_ptr — this rank's local (unicast) device view of the buffer and its requested size.
 * fcoo_mc_free — unmap and release (synchronises the device; collective only in the sense that
 *   no rank may still be writing through the multicast range). */
fcoo_status fcoo_mc_alloc(fcoo_comm_t comm, size_t bytes, fcoo_mc_t* out);
fcoo_status fcoo_mc_ptr(fcoo_mc_t mc, void** local, size_t* bytes);
fcoo_status fcoo_mc_free(fcoo_mc_t mc);
/* fcoo_mttkrp_mc — SpMTTKRP (as fcoo_mttkrp) on a sharded handle whose combine across ranks is
 * fused into the kernel's epilogue: segments owned by one tile are written with multimem.st
 * (every rank's copy), segments shared with neighbouring tiles — the only rows partial on more
 * than one rank — with multimem.red.add, reduced in the NVSwitch.  No separate all-reduce: each
 * rank's copy holds the full I_n x R output (row-major fp32, via fcoo_mc_ptr) when the call's
 * work completes on `stream`.  Sequence on `stream`: zero the local copy, comm barrier (no rank
 * writes into a copy before it is zeroed), kernel, comm barrier (every rank's writes landed).
 * Requires the staged float4 engine: order >= 3, R % 4 == 0, 16 <= R <= 128, 16-byte aligned factors;
 * buffer >= I_n*R*4 bytes; every rank calls it (collective).  Errors: ARG, RANK, SHAPE, CUDA, NCCL. */
fcoo_status fcoo_mttkrp_mc(fcoo_t f, const float* const* factors, int R, fcoo_mc_t out, void* stream);

/* fcoo_set_shard — restrict the handle to the tiles of shard `shard` of `nshards`: the
 * tile-aligned nnz range [floor(shard*ntiles/nshards), floor((shard+1)*ntiles/nshards)).
 * comm (may be NULL) is used by fcoo_mttkrp / fcoo_ttm to all-reduce the partial outputs.
 * nshards == 1 restores the whole handle. */
fcoo_status fcoo_set_shard(fcoo_t f, int shard, int nshards, fcoo_comm_t comm);

/* fcoo_build_sharded — fcoo_build followed by fcoo_set_shard(rank, nranks, comm) with the rank
 * and size of `comm` (every rank sorts the whole tensor redundantly —
 * no distributed sort — and then works only on its tile-aligned, nnz-balanced slice; the
 * handle keeps the full stream, the kernels read only the slice).  fcoo_mttkrp / fcoo_ttm on the
 * result all-reduce the partial outputs over `comm`, so every rank receives the full output.
 * Same inputs, ownership, host synchronisation and errors as fcoo_build, plus ARG for a NULL
 * comm.  `comm` must outlive the handle. */
fcoo_status fcoo_build_sharded(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, fcoo_comm_t comm,
                               const fcoo_allocator* alloc, void* stream, fcoo_t* out);

/* fcoo_shard_range — the tile range fcoo_set_shard uses (pure host arithmetic, no device):
 * [*begin, *end) = [floor(shard*ntiles/nshards), floor((shard+1)*ntiles/nshards)). */
fcoo_status fcoo_shard_range(int64_t ntiles, int shard, int nshards, int64_t* begin, int64_t* end);

/* ---- distributed build and owned-rows combine (SURVEY §8(e) alternative, §8(f)-4) ----
 * The tile shards above split one redundantly-built stream and sum partial outputs.  The row-
 * partitioned path instead gives rank k the nonzeros of the index-mode rows [b_k, b_{k+1}) only:
 * slices (the SpMTTKRP segments, Eq.(6)) never cross ranks, so each rank's output rows
 * there are complete and the combine is an all-gather of owned row ranges (one NCCL group of
 * in-place broadcasts: about half the bytes of the all-reduce), and no rank sorts more than its
 * own nonzeros.  The steps are exported separately so each can be tested on one GPU. */

/* fcoo_slice_histogram — hist[i] = number of nonzeros of `coo` with coordinate i in `mode`
 * (hist: device u32[dims[mode]], overwritten).  nnz may be 0.  Errors: ARG, ORDER, MODE,
 * INDEX_RANGE (synchronises `stream` to report it), CUDA. */
fcoo_status fcoo_slice_histogram(const fcoo_coo* coo, int mode, uint32_t* hist, void* stream);

/* fcoo_row_partition — host arithmetic, no device.  From a (global) slice histogram hist[0..I)
 * (host), the row bounds of nranks contiguous ranges balanced by nonzero count:
 *   bounds[0] = 0, bounds[nranks] = I, and for 0 < k < nranks bounds[k] = the smallest r with
 *   sum(hist[0..r)) >= ceil(k * nnz / nranks), nnz = sum(hist).
 * A slice heavier than nnz / nranks can leave a rank with no rows (bounds[k] == bounds[k+1]).
 * bounds: host int64[nranks + 1].  Errors: ARG. */
fcoo_status fcoo_row_partition(const uint32_t* hist, int64_t I, int nranks, int64_t* bounds);

/* fcoo_bucket_rows — stable partition of the nonzeros of `coo` by destination rank (the k with
 * bounds[k] <= i_mode < bounds[k+1]): idx_out (host array of `order` DEVICE pointers, nnz u32
 * each) and val_out (device, nnz f32) receive the nonzeros grouped by destination in rank order,
 * input order kept inside a group; counts (host int64[nranks]) the group sizes.  Synchronises.
 * Errors: ARG, ORDER, MODE, INDEX_RANGE (a coordinate >= bounds[nranks]), OOM, CUDA. */
fcoo_status fcoo_bucket_rows(const fcoo_coo* coo, int mode, const int64_t* bounds, int nranks,
                             uint32_t* const* idx_out, float* val_out, int64_t* counts, const fcoo_allocator* alloc,
                             void* stream);

/* fcoo_set_row_shard — declare that MTTKRP handle f holds exactly the nonzeros of rows
 * [bounds[rank], bounds[rank+1]) of the whole tensor (bounds: host int64[nranks+1], from 0 to I_n,
 * non-decreasing).  fcoo_mttkrp then writes those complete rows and, with a comm of nranks ranks
 * whose rank is `rank`, all-gathers every rank's owned rows so each holds the full output; with
 * comm == NULL the output holds this rank's rows only (the others 0).  Checks on the device that
 * the handle's rows lie in its range (one host sync).  Excludes fcoo_set_shard tile shards and the
 * fused multicast combine.  Errors: ARG, SHAPE (SpTTM handle), OOM, CUDA. */
fcoo_status fcoo_set_row_shard(fcoo_t f, int rank, int nranks, const int64_t* bounds, fcoo_comm_t comm);

/* fcoo_build_distributed — COLLECTIVE over comm: each rank passes its own chunk `local` of the
 * tensor (any split of the nonzeros; nnz may be 0 on some ranks; same order and dims everywhere)
 * and receives the F-COO handle (FCOO_OP_MTTKRP only) of its rows of `mode`:
 *   fcoo_slice_histogram -> NCCL all-reduce -> fcoo_row_partition -> fcoo_bucket_rows ->
 *   NCCL all-gather of the per-destination counts -> grouped ncclSend/ncclRecv of the buckets
 *   (own bucket: device copy) -> fcoo_build (opts: tile, flags, block rows as usual) -> fcoo_set_row_shard.
 * A rank whose range received no nonzeros gets an empty handle (its rows read 0).  A local failure
 * (bad coordinate, allocation) is agreed across the ranks before each collective step, so every rank
 * returns an error instead of waiting in a collective.  Synchronises the host several times (setup path).  Errors: as fcoo_build, plus SHAPE (opts->op != MTTKRP), ARG
 * (FCOO_BUILD_KEEP_PERM: a permutation would index the rank's received nonzeros), NCCL. */
fcoo_status fcoo_build_distributed(const fcoo_coo* local, int mode, const fcoo_build_opts* opts, fcoo_comm_t comm,
                                   const fcoo_allocator* alloc, void* stream, fcoo_t* out);

/* ---- CP-ALS (Algorithm 1, generalised to order N) ----
 * Per iteration, for n = 0..N-1: M = MTTKRP_n (fcoo_mttkrp, one F-COO handle per mode built up
 * front); V = Hadamard_{m != n} U_m^T U_m (fp64); U_n = M V^{-1} (fp64 Cholesky, with a
 * Jacobi pseudo-inverse fallback when V is not positive definite, reading Q14); lambda =
 * column 2-norms of U_n; U_n normalised (reading Q13).  After the last mode:
 *   fit = 1 - sqrt(max(0, |X|^2 + |Xhat|^2 - 2 <X, Xhat>)) / |X|,
 *   <X, Xhat> = sum_r lambda_r sum_i M(i,r) U_N(i,r),  |Xhat|^2 = lambda^T (Hadamard_m G_m) lambda.
 * Stops early when tol > 0 and |fit - fit_prev| < tol ("no improvement").
 * With comm != NULL every rank builds all modes, processes its shard of every mode, and
 * all-reduces M; the R x R work is replicated, so the factors stay identical on all ranks. */
typedef struct {
  int R;            /* 1..256 */
  int iters;        /* >= 1 */
  double tol;       /* 0 = run all iterations */
  int tile_nnz;     /* 0 -> automatic (see fcoo_build_opts) */
  fcoo_comm_t comm; /* NULL = single GPU */
  int rank, nranks; /* shard of this process (ignored when comm == NULL) */
  uint64_t seed;    /* != 0: the library seeds the factors itself (below); 0: caller's init */
  int deterministic; /* != 0: build every mode with FCOO_BUILD_DETERMINISTIC, so repeated runs
                        give bitwise-identical factors, lambda and fit trace */
  int layout;        /* 0 = automatic: every mode's handle uses the blocked F-COO (FCOO_BUILD_BLOCKED)
                        when the build allows it (not deterministic, order <= 5, packed word fits),
                        else the plain F-COO; 1 = always the plain F-COO */
  int dist;          /* != 0 (needs comm): `tensor` is THIS RANK'S CHUNK of the nonzeros (any split; same
                        order and dims on every rank) and every mode's handle is built by
                        fcoo_build_distributed: each rank's MTTKRP covers its nnz-balanced rows and the
                        owned-rows all-gather replaces the all-reduce (the last mode in fp64, gathered
                        in fp64); |X|^2 is summed over the ranks.  Excludes deterministic. */
} fcoo_cp_opts;

/*
 * cp_als — factors: host array of `order` DEVICE pointers to I_m x R fp32 buffers holding the
 * initial factors on entry (opts->seed == 0: caller-seeded) and the unit-column factors on exit.
 * opts->seed != 0 overwrites them first, on the device, with entry e of mode m =
 * (h(seed, 1000 + m, e) >> 40) * 2^-24 in [0, 1), h the counter-based splitmix64 hash of
 * DESIGN.md §4 (the same values as the test generator's factors(dims, R, seed)), so every rank of
 * a sharded run starts from identical factors without a host round trip.
 * lambda: device [R] fp32 (out).  fit_trace: host [iters] (out).  iters_done: host (out).
 * Synchronises `stream` once per iteration when tol > 0 (to read the fit for the stopping rule),
 * otherwise once at the end (the fit trace stays on the device until then).
 */
fcoo_status cp_als(const fcoo_coo* tensor, const fcoo_cp_opts* opts, float* const* factors, float* lambda,
                   double* fit_trace, int* iters_done, const fcoo_allocator* alloc, void* stream);

/*
 * FROSTT .tns text I/O (host only; no device work).  Table IV's datasets
 * are distributed as FROSTT text: one nonzero per line, "i_1 ... i_N v", 1-based coordinates,
 * whitespace-separated; lines whose first non-blank character is '#' and blank lines are
 * skipped.  Every data line must have the arity of the first (N + 1 fields, 2 <= N <= 8);
 * coordinates are integers in [1, 2^32 - 1]; v is a decimal float, rounded once to fp32.
 *
 * fcoo_tns_read — parse `path` with `nthreads` host threads (0 = all cores) into a
 *   library-owned host tensor (0-based SoA).  dims_override: host [N] or NULL; NULL gives
 *   dims[m] = max coordinate of mode m, otherwise every coordinate must be <= dims_override[m].
 *   Errors: FCOO_ERR_IO (cannot open/read; malformed line: wrong arity, non-numeric, index < 1 or
 *   > 2^32 - 1 -- fcoo_last_error() names the line), FCOO_ERR_ORDER, FCOO_ERR_EMPTY (no data
 *   line), FCOO_ERR_INDEX_RANGE (coordinate above dims_override), FCOO_ERR_ARG.
 * fcoo_tns_info — order, dims (host [8]; the first `order` entries written) and nnz.
 * fcoo_tns_copy — copy into caller-owned HOST buffers: idx = host array of `order` host
 *   pointers to nnz uint32 each, val = nnz floats.  File order is kept (not sorted).
 * fcoo_tns_destroy — free the host tensor (NULL is a no-op).
 * fcoo_tns_write — write a tensor held in HOST buffers as 1-based FROSTT text, file order =
 *   row order, values as "%.9g" (exact fp32 round trip).  nnz == 0 writes an empty file.
 */
typedef struct fcoo_tns_s* fcoo_tns_t;
fcoo_status fcoo_tns_read(const char* path, int nthreads, const int64_t* dims_override, fcoo_tns_t* out);
fcoo_status fcoo_tns_info(fcoo_tns_t t, int* order, int64_t* dims, int64_t* nnz);
fcoo_status fcoo_tns_copy(fcoo_tns_t t, uint32_t* const* idx, float* val);
fcoo_status fcoo_tns_destroy(fcoo_tns_t t);
fcoo_status fcoo_tns_write(const char* path, int order, int64_t nnz, const uint32_t* const* idx, const float* val);

const char* fcoo_status_str(fcoo_status s);
const char* fcoo_last_error(void);
/* Number of kernel launches this library enqueued so far in this process (for bench.py). */
uint64_t fcoo_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FCOO_H */
