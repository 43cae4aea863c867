// fcoo_build.cu — F-COO construction on the device (§IV-B, Fig. 2, Table II).
//
// Pipeline:
//   k_pack_keys   validate coordinates, pack one u64 sort key per nonzero:
//                 index modes (ascending mode id) most significant, then the product modes in
//                 ascending-extent order (reading Q5); ord = input ordinal
//   CUB onesweep radix sort of (key, payload) over the key bits actually used (stable); the
//                 payload is the value's bits, or the input ordinal when KEEP_PERM asks for perm
//   k_flags       bf word per 32 nonzeros by warp ballot (head = index bits differ from the
//                 previous key; reading Q1), duplicate detection (Q6), unpack product
//                 indices from the key, gather values by ord, per-word head counts
//   CUB exclusive scan of the word counts -> word_base (heads before word w)
//   k_tiles       sf[t] = bf[t*T] by ballot (Q3), seg_base[t] = word_base[t*T/32]
//   one host sync: error flags + nsegs
//   k_seg_coord   seg_coord[s] = index tuple of the s-th head (reading Q4)
#include <cub/cub.cuh>
#include <stdarg.h>

#include "fcoo_internal.cuh"

namespace fcoo {

namespace {

enum : uint32_t { ERRF_INDEX_RANGE = 1u, ERRF_DUPLICATE = 2u };

struct KeyLayout {
  int order;
  int key_modes[kMaxOrder];   // key position a -> tensor mode
  int shift[kMaxOrder];       // bit offset of key position a
  uint32_t dims[kMaxOrder];   // extent of key position a (for validation), 0 = 2^32
  uint64_t mask[kMaxOrder];
  int n_idx;
  int prod_bits;              // bits below the index part
  // blocked layout (BR > 0): block id floor(i_outer / BR) above every coordinate, at blk_shift;
  // the outer mode is key position n_idx (the first product mode of reading Q5)
  uint32_t BR;
  int blk_shift;
};

struct IdxPtrs {
  const uint32_t* p[kMaxOrder];
};

// payload: the input ordinal (KEEP_PERM builds) or the value's bits (val_in != nullptr), so the
// radix sort carries the values along and the flags kernel needs no random gather
template <class K>
__global__ void k_pack_keys(IdxPtrs idx, KeyLayout L, int64_t nnz, const float* __restrict__ val_in,
                            K* __restrict__ keys, uint32_t* __restrict__ ord, uint32_t* __restrict__ err) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  K key = 0;
  bool bad = false;
#pragma unroll
  for (int a = 0; a < kMaxOrder; ++a) {
    if (a < L.order) {
      uint32_t c = idx.p[a][q];
      bad |= (L.dims[a] != 0u && c >= L.dims[a]);
      key |= (K)((uint64_t)c & L.mask[a]) << L.shift[a];
    }
  }
  if (bad) atomicOr(err, ERRF_INDEX_RANGE);
  if (L.BR) key |= (K)(idx.p[L.n_idx][q] / L.BR) << L.blk_shift;
  keys[q] = key;
  ord[q] = val_in ? __float_as_uint(val_in[q]) : (uint32_t)q;
}

template <class K>
__device__ __forceinline__ K index_part(K key, int prod_bits) {
  return prod_bits >= (int)(8 * sizeof(K)) ? (K)0 : (key >> prod_bits);
}

// One thread per (padded) position p; nnz_pad is a multiple of 32 so warps are whole words.
template <class K>
__global__ void k_flags(const K* __restrict__ keys, const uint32_t* __restrict__ ord,
                        const float* __restrict__ val_in, KeyLayout L, int n_prod, int64_t nnz, int64_t nnz_pad,
                        uint32_t* __restrict__ pidx, float* __restrict__ val, uint32_t* __restrict__ bf,
                        uint32_t* __restrict__ wcount, uint32_t* __restrict__ perm, uint32_t* __restrict__ err) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz_pad) return;  // nnz_pad % 32 == 0 and blockDim % 32 == 0: whole warps exit together
  bool live = p < nnz;
  bool head = false;
  if (live) {
    K key = keys[p];
    if (p == 0) {
      head = true;
    } else {
      K prev = keys[p - 1];
      head = index_part(key, L.prod_bits) != index_part(prev, L.prod_bits);
      if (key == prev) atomicOr(err, ERRF_DUPLICATE);
    }
    for (int a = 0; a < n_prod; ++a) {
      int ka = L.n_idx + a;
      pidx[(int64_t)a * nnz_pad + p] = (uint32_t)((key >> L.shift[ka]) & L.mask[ka]);
    }
    uint32_t o = ord[p];  // input ordinal (perm != nullptr) or the sorted value's bits
    if (perm) {
      val[p] = val_in[o];
      perm[p] = o;
    } else {
      val[p] = __uint_as_float(o);
    }
  } else {
    for (int a = 0; a < n_prod; ++a) pidx[(int64_t)a * nnz_pad + p] = 0u;
    val[p] = 0.0f;
  }
  uint32_t word = __ballot_sync(0xffffffffu, head);
  if ((threadIdx.x & 31) == 0) {
    bf[p >> 5] = word;
    wcount[p >> 5] = __popc(word);
  }
}

// One thread per tile: sf bit (ballot over 32 tiles) and seg_base.
__global__ void k_tiles(const uint32_t* __restrict__ bf, const uint32_t* __restrict__ wbase, int64_t ntiles,
                        int64_t words_per_tile, int64_t nwords, uint32_t* __restrict__ sf,
                        uint32_t* __restrict__ seg_base) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bit = false;
  if (t < ntiles) {
    int64_t w = t * words_per_tile;
    bit = bf[w] & 1u;
    seg_base[t] = wbase[w];
  }
  if (t == ntiles) seg_base[t] = wbase[nwords];
  uint32_t word = __ballot_sync(0xffffffffu, bit);
  if ((threadIdx.x & 31) == 0 && (t >> 5) <= (ntiles - 1) >> 5) sf[t >> 5] = word;
}

template <class K>
__global__ void k_seg_coord(const K* __restrict__ keys, const uint32_t* __restrict__ bf,
                            const uint32_t* __restrict__ wbase, KeyLayout L, int64_t nnz,
                            uint32_t* __restrict__ seg_coord) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  uint32_t word = bf[p >> 5];
  int b = (int)(p & 31);
  if (!((word >> b) & 1u)) return;
  uint32_t s = wbase[p >> 5] + __popc(word & ((1u << b) - 1u));
  K key = keys[p];
  for (int a = 0; a < L.n_idx; ++a) seg_coord[(int64_t)s * L.n_idx + a] = (uint32_t)((key >> L.shift[a]) & L.mask[a]);
}

// ---- second flag level (FCOO_BUILD_FIBRE_FLAGS; Fig. 2) ----
// bf2: heads of fibres = positions whose key differs from the previous one above the last product
// mode's bits (fib_shift = the bit offset of the second-to-last key position)
template <class K>
__global__ void k_fibre_flags(const K* __restrict__ keys, int fib_shift, int64_t nnz, int64_t nnz_pad,
                              uint32_t* __restrict__ bf2, uint32_t* __restrict__ wcount) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz_pad) return;  // whole warps
  bool head = false;
  if (p < nnz) head = p == 0 || (keys[p] >> fib_shift) != (keys[p - 1] >> fib_shift);
  const uint32_t word = __ballot_sync(0xffffffffu, head);
  if ((threadIdx.x & 31) == 0) {
    bf2[p >> 5] = word;
    wcount[p >> 5] = __popc(word);
  }
}

// fibre table: the key's fields above the last product mode (index modes, then product modes in
// Q5 order but the last) of every bf2 head
template <class K>
__global__ void k_fib_coord_l2(const K* __restrict__ keys, const uint32_t* __restrict__ bf2,
                               const uint32_t* __restrict__ wbase, KeyLayout L, int64_t nnz,
                               uint32_t* __restrict__ fib) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const uint32_t word = bf2[p >> 5];
  const int b = (int)(p & 31);
  if (!((word >> b) & 1u)) return;
  const uint32_t r = wbase[p >> 5] + __popc(word & ((1u << b) - 1u));
  const K key = keys[p];
  const int nf = L.order - 1;
  for (int a = 0; a < nf; ++a) fib[(int64_t)r * nf + a] = (uint32_t)((key >> L.shift[a]) & L.mask[a]);
}

// ---- blocked layout (FCOO_BUILD_BLOCKED) ----
// start[b] = first sorted position whose block id is >= b (start[nblocks] = nnz): thread p writes
// start[b] for every b in (block(p-1), block(p)], so each entry is written exactly once.
template <class K>
__global__ void k_blk_bounds(const K* __restrict__ keys, int64_t nnz, int blk_shift, int64_t nblocks,
                             int64_t* __restrict__ start) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > nnz) return;
  const int64_t bp = p < nnz ? (int64_t)(keys[p] >> blk_shift) : nblocks;
  const int64_t bq = p > 0 ? (int64_t)(keys[p - 1] >> blk_shift) : -1;
  for (int64_t b = bq + 1; b <= bp; ++b) start[b] = p;
}

// qmap[q] = sorted position of stream position q, or 0xffffffff for padding (binary search of the
// block of q in pstart[0..nblocks]).
__global__ void k_blk_qmap(const int64_t* __restrict__ pstart, const int64_t* __restrict__ start, int64_t nblocks,
                           int64_t nstream, uint32_t* __restrict__ qmap) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nstream) return;
  int64_t lo = 0, hi = nblocks;  // pstart[lo] <= q < pstart[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (pstart[mid] <= q) lo = mid; else hi = mid;
  }
  const int64_t r = q - pstart[lo];
  qmap[q] = r < start[lo + 1] - start[lo] ? (uint32_t)(start[lo] + r) : 0xffffffffu;
}

// One thread per stream position q (nstream % 32 == 0: whole warps): packed words, values, bf,
// per-word head counts, perm; a head is a real position whose (block, index tuple) differs from
// the previous sorted key (the block id sits above the index part of the key).
template <class K>
__global__ void k_flags_blocked(const K* __restrict__ keys, const uint32_t* __restrict__ ord,
                                const float* __restrict__ val_in, KeyLayout L, int n_prod, int pk_shift,
                                const uint32_t* __restrict__ qmap, int64_t nstream, uint32_t* __restrict__ pk,
                                float* __restrict__ val, uint32_t* __restrict__ bf, uint32_t* __restrict__ wcount,
                                uint32_t* __restrict__ perm, uint32_t* __restrict__ err) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nstream) return;
  const uint32_t p = qmap[q];
  const bool live = p != 0xffffffffu;
  const int n_words = n_prod >= 2 ? n_prod - 1 : 1;
  bool head = false;
  if (live) {
    const K key = keys[p];
    if (p == 0) {
      head = true;
    } else {
      const K prev = keys[p - 1];
      head = index_part(key, L.prod_bits) != index_part(prev, L.prod_bits);
      if (key == prev) atomicOr(err, ERRF_DUPLICATE);
    }
    const int ko = L.n_idx, kl = L.n_idx + n_prod - 1;
    const uint32_t b = (uint32_t)(key >> L.blk_shift);
    const uint32_t local = (uint32_t)((key >> L.shift[ko]) & L.mask[ko]) - b * L.BR;
    const uint32_t last = (uint32_t)((key >> L.shift[kl]) & L.mask[kl]);
    pk[q] = n_prod >= 2 ? (local << pk_shift) | last : local;
    for (int a = 1; a + 1 < n_prod; ++a)
      pk[(int64_t)a * nstream + q] = (uint32_t)((key >> L.shift[ko + a]) & L.mask[ko + a]);
    const uint32_t o = ord[p];
    if (perm) {
      val[q] = val_in[o];
      perm[q] = o;
    } else {
      val[q] = __uint_as_float(o);
    }
  } else {
    for (int a = 0; a < n_words; ++a) pk[(int64_t)a * nstream + q] = 0u;
    val[q] = 0.0f;
    if (perm) perm[q] = 0xffffffffu;
  }
  const uint32_t word = __ballot_sync(0xffffffffu, head);
  if ((threadIdx.x & 31) == 0) {
    bf[q >> 5] = word;
    wcount[q >> 5] = __popc(word);
  }
}

template <class K>
__global__ void k_seg_coord_blocked(const K* __restrict__ keys, const uint32_t* __restrict__ qmap,
                                    const uint32_t* __restrict__ bf, const uint32_t* __restrict__ wbase, KeyLayout L,
                                    int64_t nstream, uint32_t* __restrict__ seg_coord) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nstream) return;
  const uint32_t word = bf[q >> 5];
  const int b = (int)(q & 31);
  if (!((word >> b) & 1u)) return;
  const uint32_t s = wbase[q >> 5] + __popc(word & ((1u << b) - 1u));
  const K key = keys[qmap[q]];
  for (int a = 0; a < L.n_idx; ++a) seg_coord[(int64_t)s * L.n_idx + a] = (uint32_t)((key >> L.shift[a]) & L.mask[a]);
}

// ---- blocked SpTTM (op TTM): the fibre (output row) of each blocked segment ----
// A fibre's nonzeros are spread over the blocks of U rows, so the blocked stream holds one segment
// per (block, fibre); the SpTTM output keeps one row per fibre (Eq.(3)) in lexicographic
// order of the index tuple, as the plain F-COO does.  The segments' tuples are sorted (key = the
// index part of the build key, payload = segment ordinal); a new tuple in sorted order starts a
// fibre; seg_row[s] = fibre ordinal of segment s and fib_coord[r] = tuple of fibre r.
template <class K>
__global__ void k_fib_keys(const uint32_t* __restrict__ seg_coord, KeyLayout L, int64_t nsegs, K* __restrict__ keys,
                           uint32_t* __restrict__ ids) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsegs) return;
  K key = 0;
  for (int a = 0; a < L.n_idx; ++a) key |= (K)seg_coord[s * L.n_idx + a] << (L.shift[a] - L.prod_bits);
  keys[s] = key;
  ids[s] = (uint32_t)s;
}

template <class K>
__global__ void k_fib_heads(const K* __restrict__ keys, int64_t n, uint32_t* __restrict__ head) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  head[p] = p == n ? 0u : (p == 0 || keys[p] != keys[p - 1]) ? 1u : 0u;
}

// excl = exclusive scan of head: fibre ordinal of sorted position p = excl[p] + head[p] - 1
__global__ void k_fib_scatter(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ head,
                              const uint32_t* __restrict__ excl, const uint32_t* __restrict__ seg_coord, int n_idx,
                              int64_t n, uint32_t* __restrict__ seg_row, uint32_t* __restrict__ fib_coord) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t r = excl[p] + head[p] - 1u, s = ids[p];
  seg_row[s] = r;
  if (head[p])
    for (int a = 0; a < n_idx; ++a) fib_coord[(int64_t)r * n_idx + a] = seg_coord[(int64_t)s * n_idx + a];
}

int bits_for(int64_t n) {
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < n) ++b;
  return b;
}

template <class T>
T* grab(fcoo_s* f, size_t bytes, cudaStream_t s, size_t* rec) {
  *rec = bytes;
  return reinterpret_cast<T*>(f->alloc.get(bytes, s));
}

void free_handle_arrays(fcoo_s* f) {
  cudaStream_t s = f->build_stream;
  if (f->pidx) f->alloc.put(f->pidx, f->bytes_pidx, s);
  if (f->val) f->alloc.put(f->val, f->bytes_val, s);
  if (f->bf) f->alloc.put(f->bf, f->bytes_bf, s);
  if (f->sf) f->alloc.put(f->sf, f->bytes_sf, s);
  if (f->seg_base) f->alloc.put(f->seg_base, f->bytes_seg_base, s);
  if (f->seg_coord) f->alloc.put(f->seg_coord, f->bytes_seg_coord, s);
  if (f->perm) f->alloc.put(f->perm, f->bytes_perm, s);
  if (f->blk_start) f->alloc.put(f->blk_start, f->bytes_blk, s);
  if (f->seg_row) f->alloc.put(f->seg_row, f->bytes_seg_row, s);
  if (f->fib_coord) f->alloc.put(f->fib_coord, f->bytes_fib, s);
  if (f->bf2) f->alloc.put(f->bf2, f->bytes_l2, s);
  if (f->dpart) f->alloc.put(f->dpart, f->bytes_dpart, s);
  f->dpart = nullptr;
  f->bytes_dpart = 0;
  for (int k = 0; k < 10; ++k)
    if (f->items[k]) f->alloc.put(f->items[k], sizeof(int2) * f->h_items[k].size(), s);
  for (int k = 0; k < 10; ++k) f->items[k] = nullptr;
  f->blk_start = nullptr; f->blk_end = nullptr;
  f->pidx = nullptr; f->val = nullptr; f->bf = nullptr; f->sf = nullptr;
  f->seg_base = nullptr; f->seg_coord = nullptr; f->perm = nullptr;
  f->seg_row = nullptr; f->fib_coord = nullptr;
  f->bf2 = nullptr; f->sf2 = nullptr; f->seg_base2 = nullptr;
}

}  // namespace

// Automatic tile length (tile_nnz == 0): enough tiles that the MTTKRP/TTM launch fills the GPU
// about four times over at R=32 (148 SMs x 16 resident warps x 4 lane-groups per warp x 4 waves),
// rounded to the nearest power of two in [32, 2048] (power-of-two tiles measured 5-12% faster than
// neighbouring multiples of 32, profiles/round1/README.md).  Large tensors get T = 2048 (nell-2);
// brainq-sized ones 256, where short fibres need more lane-groups in flight.
int auto_tile(int64_t nnz) {
  const double x = (double)nnz / (148.0 * 16 * 4 * 4);
  int t = 32;
  while (t < 2048 && (double)t * 1.41421356 < x) t <<= 1;
  return t;
}

// Host-side mode taxonomy (Table I) and key layout; used by fcoo_build.
fcoo_status plan_modes(fcoo_s* f, int order, const int64_t* dims, int op, int mode, bool desc = false) {
  if (order < 2 || order > kMaxOrder) return fail(FCOO_ERR_ORDER, "order %d outside [2,8]", order);
  if (mode < 0 || mode >= order) return fail(FCOO_ERR_MODE, "mode %d outside [0,%d)", mode, order);
  if (op != FCOO_OP_MTTKRP && op != FCOO_OP_TTM) return fail(FCOO_ERR_ARG, "unknown op %d", op);
  f->order = order; f->op = op; f->mode = mode;
  for (int m = 0; m < order; ++m) {
    if (dims[m] < 1 || dims[m] > 4294967295LL) return fail(FCOO_ERR_ARG, "dims[%d]=%lld outside [1,2^32)", m, (long long)dims[m]);
    f->dims[m] = dims[m];
  }
  int ni = 0, np = 0;
  if (op == FCOO_OP_MTTKRP) {
    f->idx_modes[ni++] = mode;
    for (int m = 0; m < order; ++m) if (m != mode) f->prod_modes[np++] = m;
    // reading Q5: ascending extent, ties by mode id (stable); FCOO_BUILD_PRODUCT_DESC: descending
    auto before = [&](int x, int y) { return desc ? dims[x] > dims[y] : dims[x] < dims[y]; };
    for (int a = 1; a < np; ++a)
      for (int b = a; b > 0 && before(f->prod_modes[b], f->prod_modes[b - 1]); --b) {
        int t = f->prod_modes[b]; f->prod_modes[b] = f->prod_modes[b - 1]; f->prod_modes[b - 1] = t;
      }
  } else {
    for (int m = 0; m < order; ++m) if (m != mode) f->idx_modes[ni++] = m;
    f->prod_modes[np++] = mode;
  }
  f->n_idx = ni; f->n_prod = np;
  return FCOO_OK;
}

// Key packing, radix sort, flags, tiles, the one host sync and seg_coord, for sort keys of type K
// (uint64_t up to 64 key bits; unsigned __int128 up to 128, e.g. nell1 = 69 bits, Table IV).
// Returns a status; the caller frees the handle on failure.  Scratch is freed stream-ordered.
template <class K>
fcoo_status sort_and_flag(fcoo_s* f, const fcoo_coo* coo, const KeyLayout& L, const IdxPtrs& ip, int total,
                          unsigned flags, cudaStream_t s) {
  const int64_t nnz = f->nnz, nnz_pad = f->nnz_pad, nwords = nnz_pad / 32, ntiles = f->ntiles;
  const int64_t T = f->T;
  Buf keys0(&f->alloc, sizeof(K) * nnz, s), keys1(&f->alloc, sizeof(K) * nnz, s);
  Buf ord0(&f->alloc, sizeof(uint32_t) * nnz, s), ord1(&f->alloc, sizeof(uint32_t) * nnz, s);
  Buf wcount(&f->alloc, sizeof(uint32_t) * (nwords + 1), s), wbase(&f->alloc, sizeof(uint32_t) * (nwords + 1), s);
  Buf errb(&f->alloc, sizeof(uint32_t) * 2, s);
  if (!keys0.ok() || !keys1.ok() || !ord0.ok() || !ord1.ok() || !wcount.ok() || !wbase.ok() || !errb.ok())
    return fail(FCOO_ERR_OOM, "build scratch allocation failed");
  cudaError_t ce;
  if ((ce = cudaMemsetAsync(errb.p, 0, sizeof(uint32_t) * 2, s)) != cudaSuccess ||
      (ce = cudaMemsetAsync(wcount.p, 0, sizeof(uint32_t) * (nwords + 1), s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));

  const int TB = 256;
  const bool keep_perm = (flags & FCOO_BUILD_KEEP_PERM) != 0;
  k_pack_keys<<<(unsigned)((nnz + TB - 1) / TB), TB, 0, s>>>(ip, L, nnz, keep_perm ? nullptr : coo->val,
                                                             keys0.as<K>(), ord0.as<uint32_t>(),
                                                             errb.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_pack_keys: %s", cudaGetErrorString(ce));

  cub::DoubleBuffer<K> dk(keys0.as<K>(), keys1.as<K>());
  cub::DoubleBuffer<uint32_t> dv(ord0.as<uint32_t>(), ord1.as<uint32_t>());
  int end_bit = total > 0 ? total : 1;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int64_t)nnz, 0, end_bit, s);
  {
    Buf cubtmp(&f->alloc, tmp_bytes, s);
    if (!cubtmp.ok()) return fail(FCOO_ERR_OOM, "radix sort scratch");
    if ((ce = cub::DeviceRadixSort::SortPairs(cubtmp.p, tmp_bytes, dk, dv, (int64_t)nnz, 0, end_bit, s)) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "radix sort: %s", cudaGetErrorString(ce));
    count_launch(2 + (end_bit + 7) / 8);
  }
  const K* keys = dk.Current();
  const uint32_t* ord = dv.Current();

  k_flags<<<(unsigned)((nnz_pad + TB - 1) / TB), TB, 0, s>>>(keys, ord, coo->val, L, f->n_prod, nnz, nnz_pad, f->pidx,
                                                            f->val, f->bf, wcount.as<uint32_t>(), f->perm,
                                                            errb.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_flags: %s", cudaGetErrorString(ce));

  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, wcount.as<uint32_t>(), wbase.as<uint32_t>(), (int64_t)(nwords + 1), s);
  {
    Buf scantmp(&f->alloc, scan_bytes, s);
    if (!scantmp.ok()) return fail(FCOO_ERR_OOM, "scan scratch");
    if ((ce = cub::DeviceScan::ExclusiveSum(scantmp.p, scan_bytes, wcount.as<uint32_t>(), wbase.as<uint32_t>(),
                                            (int64_t)(nwords + 1), s)) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "scan: %s", cudaGetErrorString(ce));
    count_launch(2);
  }
  int64_t tthreads = ((ntiles + 1 + 31) / 32) * 32;
  k_tiles<<<(unsigned)((tthreads + TB - 1) / TB), TB, 0, s>>>(f->bf, wbase.as<uint32_t>(), ntiles, T / 32, nwords,
                                                             f->sf, f->seg_base);
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_tiles: %s", cudaGetErrorString(ce));

  uint32_t host[2] = {0, 0};
  if ((ce = cudaMemcpyAsync(&host[0], errb.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (ce = cudaMemcpyAsync(&host[1], wbase.as<uint32_t>() + nwords, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (ce = cudaStreamSynchronize(s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "build sync: %s", cudaGetErrorString(ce));
  if (host[0] & ERRF_INDEX_RANGE) return fail(FCOO_ERR_INDEX_RANGE, "a coordinate is >= its mode extent");
  if (host[0] & ERRF_DUPLICATE) return fail(FCOO_ERR_DUPLICATE, "duplicate coordinates");
  f->nsegs = host[1];
  f->dense_rows = (f->op == FCOO_OP_MTTKRP && f->nsegs == f->dims[f->mode]) ? 1 : 0;

  f->seg_coord = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)std::max<int64_t>(1, f->nsegs * f->n_idx), s,
                                &f->bytes_seg_coord);
  if (!f->seg_coord) return fail(FCOO_ERR_OOM, "seg_coord allocation");
  k_seg_coord<<<(unsigned)((nnz + TB - 1) / TB), TB, 0, s>>>(keys, f->bf, wbase.as<uint32_t>(), L, nnz, f->seg_coord);
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_seg_coord: %s", cudaGetErrorString(ce));
  if (!(flags & FCOO_BUILD_FIBRE_FLAGS)) return FCOO_OK;
  // the second flag level on the same sorted stream (one more host sync for the fibre count)
  f->fibre_flags = 1;
  const size_t w4 = sizeof(uint32_t);
  f->bytes_l2 = w4 * ((size_t)nwords + (size_t)((ntiles + 31) / 32 + 1) + (size_t)(ntiles + 1));
  f->bf2 = reinterpret_cast<uint32_t*>(f->alloc.get(f->bytes_l2, s));
  if (!f->bf2) return fail(FCOO_ERR_OOM, "second flag level allocation");
  f->sf2 = f->bf2 + nwords;
  f->seg_base2 = f->sf2 + (ntiles + 31) / 32 + 1;
  if ((ce = cudaMemsetAsync(wcount.p, 0, sizeof(uint32_t) * (nwords + 1), s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  const int fib_shift = L.shift[L.order - 2];
  k_fibre_flags<K><<<(unsigned)((nnz_pad + TB - 1) / TB), TB, 0, s>>>(keys, fib_shift, nnz, nnz_pad, f->bf2,
                                                                       wcount.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_fibre_flags: %s", cudaGetErrorString(ce));
  {
    Buf scantmp(&f->alloc, scan_bytes, s);
    if (!scantmp.ok()) return fail(FCOO_ERR_OOM, "scan scratch");
    if ((ce = cub::DeviceScan::ExclusiveSum(scantmp.p, scan_bytes, wcount.as<uint32_t>(), wbase.as<uint32_t>(),
                                            (int64_t)(nwords + 1), s)) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "scan: %s", cudaGetErrorString(ce));
    count_launch(2);
  }
  k_tiles<<<(unsigned)((tthreads + TB - 1) / TB), TB, 0, s>>>(f->bf2, wbase.as<uint32_t>(), ntiles, T / 32, nwords,
                                                             f->sf2, f->seg_base2);
  count_launch();
  uint32_t nfib = 0;
  if ((ce = cudaMemcpyAsync(&nfib, wbase.as<uint32_t>() + nwords, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (ce = cudaStreamSynchronize(s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "build sync: %s", cudaGetErrorString(ce));
  f->nfib = nfib;
  f->fib_coord = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)std::max<int64_t>(1, (int64_t)nfib * (L.order - 1)), s,
                                &f->bytes_fib);
  if (!f->fib_coord) return fail(FCOO_ERR_OOM, "fibre table allocation");
  k_fib_coord_l2<K><<<(unsigned)((nnz + TB - 1) / TB), TB, 0, s>>>(keys, f->bf2, wbase.as<uint32_t>(), L, nnz,
                                                                    f->fib_coord);
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_fib_coord_l2: %s", cudaGetErrorString(ce));
  return FCOO_OK;
}

// Work tables of the blocked SpMTTKRP: for gpc = 1 << k, one item (b, t0) per run of up to gpc
// consecutive tiles of block b (every tile of a blocked stream lies in exactly one block).
static fcoo_status make_items(fcoo_s* f, cudaStream_t s) {
  for (int k = 3; k < 10; ++k) {
    const int64_t gpc = (int64_t)1 << k;
    std::vector<int2>& v = f->h_items[k];
    v.clear();
    for (int64_t b = 0; b < f->nblocks; ++b)
      for (int64_t t = f->h_blk_start[b] / f->T; t < f->h_blk_start[b + 1] / f->T; t += gpc)
        v.push_back(make_int2((int)b, (int)t));
    if (v.empty()) continue;
    f->items[k] = reinterpret_cast<int2*>(f->alloc.get(sizeof(int2) * v.size(), s));
    if (!f->items[k]) return fail(FCOO_ERR_OOM, "work table allocation");
    FCOO_CUDA_TRY(cudaMemcpyAsync(f->items[k], v.data(), sizeof(int2) * v.size(), cudaMemcpyHostToDevice, s));
  }
  return FCOO_OK;
}

// Blocked build (FCOO_BUILD_BLOCKED): keys carry the block id above every coordinate; after the sort
// one host sync reads the block boundaries, the stream is laid out with every block padded to a
// multiple of T, and the flags/segment steps run over the padded stream through qmap.
template <class K>
fcoo_status sort_and_flag_blocked(fcoo_s* f, const fcoo_coo* coo, const KeyLayout& L, const IdxPtrs& ip, int total,
                                  unsigned flags, cudaStream_t s) {
  const int64_t nnz = f->nnz, T = f->T, nblocks = f->nblocks;
  Buf keys0(&f->alloc, sizeof(K) * nnz, s), keys1(&f->alloc, sizeof(K) * nnz, s);
  Buf ord0(&f->alloc, sizeof(uint32_t) * nnz, s), ord1(&f->alloc, sizeof(uint32_t) * nnz, s);
  Buf errb(&f->alloc, sizeof(uint32_t) * 2, s);
  Buf startb(&f->alloc, sizeof(int64_t) * (nblocks + 1), s);
  if (!keys0.ok() || !keys1.ok() || !ord0.ok() || !ord1.ok() || !errb.ok() || !startb.ok())
    return fail(FCOO_ERR_OOM, "build scratch allocation failed");
  cudaError_t ce;
  if ((ce = cudaMemsetAsync(errb.p, 0, sizeof(uint32_t) * 2, s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  const int TB = 256;
  const bool keep_perm = (flags & FCOO_BUILD_KEEP_PERM) != 0;
  k_pack_keys<<<(unsigned)((nnz + TB - 1) / TB), TB, 0, s>>>(ip, L, nnz, keep_perm ? nullptr : coo->val,
                                                             keys0.as<K>(), ord0.as<uint32_t>(), errb.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_pack_keys: %s", cudaGetErrorString(ce));
  cub::DoubleBuffer<K> dk(keys0.as<K>(), keys1.as<K>());
  cub::DoubleBuffer<uint32_t> dv(ord0.as<uint32_t>(), ord1.as<uint32_t>());
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int64_t)nnz, 0, total, s);
  {
    Buf cubtmp(&f->alloc, tmp_bytes, s);
    if (!cubtmp.ok()) return fail(FCOO_ERR_OOM, "radix sort scratch");
    if ((ce = cub::DeviceRadixSort::SortPairs(cubtmp.p, tmp_bytes, dk, dv, (int64_t)nnz, 0, total, s)) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "radix sort: %s", cudaGetErrorString(ce));
    count_launch(2 + (total + 7) / 8);
  }
  const K* keys = dk.Current();
  const uint32_t* ord = dv.Current();
  k_blk_bounds<K><<<(unsigned)((nnz + 1 + TB - 1) / TB), TB, 0, s>>>(keys, nnz, L.blk_shift, nblocks,
                                                                      startb.as<int64_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_blk_bounds: %s", cudaGetErrorString(ce));
  // host sync 1 of 2: block boundaries and the index-range flag
  std::vector<int64_t> start(nblocks + 1);
  uint32_t err0 = 0;
  if ((ce = cudaMemcpyAsync(start.data(), startb.p, sizeof(int64_t) * (nblocks + 1), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (ce = cudaMemcpyAsync(&err0, errb.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (ce = cudaStreamSynchronize(s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "build sync: %s", cudaGetErrorString(ce));
  if (err0 & ERRF_INDEX_RANGE) return fail(FCOO_ERR_INDEX_RANGE, "a coordinate is >= its mode extent");
  f->h_blk_start.assign(nblocks + 1, 0);
  f->h_blk_end.assign(nblocks, 0);
  for (int64_t b = 0; b < nblocks; ++b) {
    const int64_t nb = start[b + 1] - start[b];
    f->h_blk_end[b] = f->h_blk_start[b] + nb;
    f->h_blk_start[b + 1] = f->h_blk_start[b] + (nb + T - 1) / T * T;
  }
  const int64_t ns = f->h_blk_start[nblocks], nwords = ns / 32;
  if (ns >= 4294967295LL) return fail(FCOO_ERR_ARG, "blocked stream of %lld positions needs < 2^32", (long long)ns);
  f->nnz_pad = ns;
  f->ntiles = ns / T;
  f->tile_begin = 0;
  f->tile_end = f->ntiles;
  const int64_t ntiles = f->ntiles;
  const int n_words = f->n_words;
  f->pidx = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)(n_words * ns), s, &f->bytes_pidx);
  f->val = grab<float>(f, sizeof(float) * (size_t)ns, s, &f->bytes_val);
  f->bf = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)nwords, s, &f->bytes_bf);
  f->sf = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)((ntiles + 31) / 32 + 1), s, &f->bytes_sf);
  f->seg_base = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)(ntiles + 1), s, &f->bytes_seg_base);
  f->blk_start = grab<int64_t>(f, sizeof(int64_t) * (size_t)(2 * nblocks + 1), s, &f->bytes_blk);
  if (keep_perm) f->perm = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)ns, s, &f->bytes_perm);
  if (!f->pidx || !f->val || !f->bf || !f->sf || !f->seg_base || !f->blk_start || (keep_perm && !f->perm))
    return fail(FCOO_ERR_OOM, "handle allocation failed");
  f->blk_end = f->blk_start + nblocks + 1;
  FCOO_CUDA_TRY(cudaMemcpyAsync(f->blk_start, f->h_blk_start.data(), sizeof(int64_t) * (nblocks + 1),
                                cudaMemcpyHostToDevice, s));
  FCOO_CUDA_TRY(cudaMemcpyAsync(f->blk_end, f->h_blk_end.data(), sizeof(int64_t) * nblocks, cudaMemcpyHostToDevice, s));
  fcoo_status st = make_items(f, s);
  if (st) return st;

  Buf qmap(&f->alloc, sizeof(uint32_t) * ns, s);
  Buf wcount(&f->alloc, sizeof(uint32_t) * (nwords + 1), s), wbase(&f->alloc, sizeof(uint32_t) * (nwords + 1), s);
  if (!qmap.ok() || !wcount.ok() || !wbase.ok()) return fail(FCOO_ERR_OOM, "build scratch allocation failed");
  if ((ce = cudaMemsetAsync(wcount.p, 0, sizeof(uint32_t) * (nwords + 1), s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "memset: %s", cudaGetErrorString(ce));
  k_blk_qmap<<<(unsigned)((ns + TB - 1) / TB), TB, 0, s>>>(f->blk_start, startb.as<int64_t>(), nblocks, ns,
                                                          qmap.as<uint32_t>());
  count_launch();
  k_flags_blocked<K><<<(unsigned)((ns + TB - 1) / TB), TB, 0, s>>>(keys, ord, coo->val, L, f->n_prod, f->pk_shift,
                                                                    qmap.as<uint32_t>(), ns, f->pidx, f->val, f->bf,
                                                                    wcount.as<uint32_t>(), f->perm, errb.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_flags_blocked: %s", cudaGetErrorString(ce));
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, wcount.as<uint32_t>(), wbase.as<uint32_t>(), (int64_t)(nwords + 1), s);
  {
    Buf scantmp(&f->alloc, scan_bytes, s);
    if (!scantmp.ok()) return fail(FCOO_ERR_OOM, "scan scratch");
    if ((ce = cub::DeviceScan::ExclusiveSum(scantmp.p, scan_bytes, wcount.as<uint32_t>(), wbase.as<uint32_t>(),
                                            (int64_t)(nwords + 1), s)) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "scan: %s", cudaGetErrorString(ce));
    count_launch(2);
  }
  const int64_t tthreads = ((ntiles + 1 + 31) / 32) * 32;
  k_tiles<<<(unsigned)((tthreads + TB - 1) / TB), TB, 0, s>>>(f->bf, wbase.as<uint32_t>(), ntiles, T / 32, nwords,
                                                             f->sf, f->seg_base);
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_tiles: %s", cudaGetErrorString(ce));
  // host sync 2 of 2: duplicates and the segment count
  uint32_t host[2] = {0, 0};
  if ((ce = cudaMemcpyAsync(&host[0], errb.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (ce = cudaMemcpyAsync(&host[1], wbase.as<uint32_t>() + nwords, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (ce = cudaStreamSynchronize(s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "build sync: %s", cudaGetErrorString(ce));
  if (host[0] & ERRF_DUPLICATE) return fail(FCOO_ERR_DUPLICATE, "duplicate coordinates");
  f->nsegs = host[1];
  f->dense_rows = 0;  // a row recurs once per block: seg_coord is always used
  f->seg_coord = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)std::max<int64_t>(1, f->nsegs * f->n_idx), s,
                                &f->bytes_seg_coord);
  if (!f->seg_coord) return fail(FCOO_ERR_OOM, "seg_coord allocation");
  k_seg_coord_blocked<K><<<(unsigned)((ns + TB - 1) / TB), TB, 0, s>>>(keys, qmap.as<uint32_t>(), f->bf,
                                                                        wbase.as<uint32_t>(), L, ns, f->seg_coord);
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_seg_coord_blocked: %s", cudaGetErrorString(ce));
  return FCOO_OK;
}

// Fibre table of a blocked SpTTM handle (k_fib_*): one more sort over the segments' index tuples
// and a third host synchronisation (the fibre count sizes fib_coord).
template <class K>
fcoo_status fibre_table(fcoo_s* f, const KeyLayout& L, cudaStream_t s) {
  const int64_t n = f->nsegs;
  const int idx_bits = L.blk_shift - L.prod_bits;
  const int TB = 256;
  Buf k0(&f->alloc, sizeof(K) * n, s), k1(&f->alloc, sizeof(K) * n, s);
  Buf i0(&f->alloc, sizeof(uint32_t) * n, s), i1(&f->alloc, sizeof(uint32_t) * n, s);
  Buf head(&f->alloc, sizeof(uint32_t) * (n + 1), s), excl(&f->alloc, sizeof(uint32_t) * (n + 1), s);
  if (!k0.ok() || !k1.ok() || !i0.ok() || !i1.ok() || !head.ok() || !excl.ok())
    return fail(FCOO_ERR_OOM, "fibre table scratch allocation failed");
  f->seg_row = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)n, s, &f->bytes_seg_row);
  if (!f->seg_row) return fail(FCOO_ERR_OOM, "seg_row allocation");
  cudaError_t ce;
  k_fib_keys<K><<<(unsigned)((n + TB - 1) / TB), TB, 0, s>>>(f->seg_coord, L, n, k0.as<K>(), i0.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_fib_keys: %s", cudaGetErrorString(ce));
  cub::DoubleBuffer<K> dk(k0.as<K>(), k1.as<K>());
  cub::DoubleBuffer<uint32_t> dv(i0.as<uint32_t>(), i1.as<uint32_t>());
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, n, 0, std::max(1, idx_bits), s);
  {
    Buf cubtmp(&f->alloc, tmp_bytes, s);
    if (!cubtmp.ok()) return fail(FCOO_ERR_OOM, "radix sort scratch");
    if ((ce = cub::DeviceRadixSort::SortPairs(cubtmp.p, tmp_bytes, dk, dv, n, 0, std::max(1, idx_bits), s)) !=
        cudaSuccess)
      return fail(FCOO_ERR_CUDA, "fibre sort: %s", cudaGetErrorString(ce));
    count_launch(2 + (idx_bits + 7) / 8);
  }
  k_fib_heads<K><<<(unsigned)((n + 1 + TB - 1) / TB), TB, 0, s>>>(dk.Current(), n, head.as<uint32_t>());
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_fib_heads: %s", cudaGetErrorString(ce));
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, head.as<uint32_t>(), excl.as<uint32_t>(), n + 1, s);
  {
    Buf scantmp(&f->alloc, scan_bytes, s);
    if (!scantmp.ok()) return fail(FCOO_ERR_OOM, "scan scratch");
    if ((ce = cub::DeviceScan::ExclusiveSum(scantmp.p, scan_bytes, head.as<uint32_t>(), excl.as<uint32_t>(), n + 1,
                                            s)) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "scan: %s", cudaGetErrorString(ce));
    count_launch(2);
  }
  uint32_t nfib = 0;
  if ((ce = cudaMemcpyAsync(&nfib, excl.as<uint32_t>() + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (ce = cudaStreamSynchronize(s)) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "build sync: %s", cudaGetErrorString(ce));
  f->nfib = nfib;
  f->fib_coord = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)std::max<int64_t>(1, (int64_t)nfib * f->n_idx), s,
                                &f->bytes_fib);
  if (!f->fib_coord) return fail(FCOO_ERR_OOM, "fib_coord allocation");
  k_fib_scatter<<<(unsigned)((n + TB - 1) / TB), TB, 0, s>>>(dv.Current(), head.as<uint32_t>(), excl.as<uint32_t>(),
                                                            f->seg_coord, f->n_idx, n, f->seg_row, f->fib_coord);
  count_launch();
  if ((ce = cudaGetLastError()) != cudaSuccess) return fail(FCOO_ERR_CUDA, "k_fib_scatter: %s", cudaGetErrorString(ce));
  return FCOO_OK;
}

fcoo_status build_impl(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, const fcoo_allocator* alloc,
                       cudaStream_t s, fcoo_t* out) {
  Nvtx range("fcoo_build");
  if (!coo || !out) return fail(FCOO_ERR_ARG, "NULL coo/out");
  *out = nullptr;
  int op = opts ? opts->op : FCOO_OP_MTTKRP;
  int T = opts ? opts->tile_nnz : 0;
  unsigned flags = opts ? opts->flags : 0u;
  if (T == 0 && coo->nnz > 0) T = auto_tile(coo->nnz);
  if (T < 32 || T > 8192 || (T % 32) != 0) return fail(FCOO_ERR_ARG, "tile_nnz %d must be a multiple of 32 in [32,8192]", T);
  if (!coo->dims || !coo->idx || !coo->val) return fail(FCOO_ERR_ARG, "NULL dims/idx/val");
  fcoo_s tmp;
  fcoo_status st = plan_modes(&tmp, coo->order, coo->dims, op, mode, (flags & FCOO_BUILD_PRODUCT_DESC) != 0);
  if (st) return st;
  const bool blocked = (flags & FCOO_BUILD_BLOCKED) != 0;
  if (flags & FCOO_BUILD_FIBRE_FLAGS) {
    if (op != FCOO_OP_MTTKRP || blocked || (flags & FCOO_BUILD_DETERMINISTIC) || tmp.n_prod < 2)
      return fail(FCOO_ERR_ARG, "FCOO_BUILD_FIBRE_FLAGS needs a plain, non-deterministic MTTKRP handle of order >= 3");
  }
  int BR = 0;
  if (blocked) {
    BR = (opts && opts->block_rows) ? opts->block_rows : 512;
    if (coo->order > 5) return fail(FCOO_ERR_ARG, "FCOO_BUILD_BLOCKED supports order <= 5 (got %d)", coo->order);
    if (flags & (FCOO_BUILD_DETERMINISTIC | FCOO_BUILD_PRODUCT_DESC))
      return fail(FCOO_ERR_ARG, "FCOO_BUILD_BLOCKED excludes DETERMINISTIC and PRODUCT_DESC");
    if (BR < 32 || BR > 65536) return fail(FCOO_ERR_ARG, "block_rows %d outside [32, 65536]", BR);
    tmp.blocked = 1;
    tmp.block_rows = BR;
    tmp.nblocks = (coo->dims[tmp.prod_modes[0]] + BR - 1) / BR;
    tmp.n_words = tmp.n_prod >= 2 ? tmp.n_prod - 1 : 1;
    const int ib = tmp.n_prod >= 2 ? bits_for(coo->dims[tmp.prod_modes[tmp.n_prod - 1]]) : 0;
    tmp.pk_shift = ib;
    if (tmp.n_prod >= 2 && bits_for(BR) + ib > 32)
      return fail(FCOO_ERR_ARG, "blocked word needs ceil(log2 %d) + %d > 32 bits", BR, ib);
  }
  if (coo->nnz <= 0) return fail(FCOO_ERR_EMPTY, "nnz == 0");
  if (coo->nnz >= 4294967295LL) return fail(FCOO_ERR_ARG, "nnz must be < 2^32");
  for (int m = 0; m < coo->order; ++m) if (!coo->idx[m]) return fail(FCOO_ERR_ARG, "idx[%d] is NULL", m);

  // key layout: key position a -> mode; first position most significant
  KeyLayout L{};
  L.order = coo->order;
  L.n_idx = tmp.n_idx;
  for (int a = 0; a < tmp.n_idx; ++a) L.key_modes[a] = tmp.idx_modes[a];
  for (int a = 0; a < tmp.n_prod; ++a) L.key_modes[tmp.n_idx + a] = tmp.prod_modes[a];
  int total = 0, bits[kMaxOrder];
  for (int a = 0; a < L.order; ++a) { bits[a] = bits_for(coo->dims[L.key_modes[a]]); total += bits[a]; }
  const int blk_bits = blocked ? bits_for(tmp.nblocks) : 0;
  if (total + blk_bits > 128) return fail(FCOO_ERR_KEY_BITS, "sort key needs %d bits > 128", total + blk_bits);
  int sh = 0;
  for (int a = L.order - 1; a >= 0; --a) {
    L.shift[a] = sh;
    L.mask[a] = bits[a] >= 64 ? ~0ull : ((1ull << bits[a]) - 1ull);
    int64_t d = coo->dims[L.key_modes[a]];
    L.dims[a] = d >= 4294967296LL ? 0u : (uint32_t)d;
    sh += bits[a];
  }
  L.prod_bits = 0;
  for (int a = tmp.n_idx; a < L.order; ++a) L.prod_bits += bits[a];
  L.BR = (uint32_t)BR;
  L.blk_shift = total;
  IdxPtrs ip{};
  for (int a = 0; a < L.order; ++a) ip.p[a] = coo->idx[L.key_modes[a]];

  fcoo_s* f = new fcoo_s(tmp);
  if (alloc && alloc->alloc && alloc->free) { f->alloc.a = *alloc; f->alloc.custom = true; }
  f->build_stream = s;
  cudaGetDevice(&f->device);
  f->T = T;
  f->deterministic = (flags & FCOO_BUILD_DETERMINISTIC) ? 1 : 0;
  f->nnz = coo->nnz;
  f->ntiles = (f->nnz + T - 1) / T;
  f->nnz_pad = f->ntiles * T;
  f->tile_begin = 0; f->tile_end = f->ntiles;
  const int64_t nnz = f->nnz, nnz_pad = f->nnz_pad, nwords = nnz_pad / 32, ntiles = f->ntiles;

  auto bail = [&](fcoo_status e) { free_handle_arrays(f); delete f; return e; };
  if (blocked) {
    const int tb = total + blk_bits;
    st = tb <= 64 ? sort_and_flag_blocked<uint64_t>(f, coo, L, ip, tb, flags, s)
                  : sort_and_flag_blocked<unsigned __int128>(f, coo, L, ip, tb, flags, s);
    if (st) return bail(st);
    if (op == FCOO_OP_TTM) {
      st = tb <= 64 ? fibre_table<uint64_t>(f, L, s) : fibre_table<unsigned __int128>(f, L, s);
      if (st) return bail(st);
    }
    *out = f;
    return FCOO_OK;
  }

  f->pidx = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)(f->n_prod * nnz_pad), s, &f->bytes_pidx);
  f->val = grab<float>(f, sizeof(float) * (size_t)nnz_pad, s, &f->bytes_val);
  f->bf = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)nwords, s, &f->bytes_bf);
  f->sf = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)((ntiles + 31) / 32 + 1), s, &f->bytes_sf);
  f->seg_base = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)(ntiles + 1), s, &f->bytes_seg_base);
  if (flags & FCOO_BUILD_KEEP_PERM) f->perm = grab<uint32_t>(f, sizeof(uint32_t) * (size_t)nnz, s, &f->bytes_perm);
  if (!f->pidx || !f->val || !f->bf || !f->sf || !f->seg_base || ((flags & FCOO_BUILD_KEEP_PERM) && !f->perm))
    return bail(fail(FCOO_ERR_OOM, "handle allocation failed"));

  if (total <= 64) st = sort_and_flag<uint64_t>(f, coo, L, ip, total, flags, s);
  else st = sort_and_flag<unsigned __int128>(f, coo, L, ip, total, flags, s);
  if (st) return bail(st);
  *out = f;
  return FCOO_OK;
}

fcoo_status build_empty(int order, const int64_t* dims, int op, int mode, const fcoo_allocator* alloc, cudaStream_t s,
                        fcoo_t* out) {
  if (!dims || !out) return fail(FCOO_ERR_ARG, "NULL dims/out");
  fcoo_s tmp;
  fcoo_status st = plan_modes(&tmp, order, dims, op, mode);
  if (st) return st;
  fcoo_s* f = new fcoo_s(tmp);
  if (alloc && alloc->alloc && alloc->free) { f->alloc.a = *alloc; f->alloc.custom = true; }
  f->build_stream = s;
  cudaGetDevice(&f->device);
  f->T = 32;
  f->nnz = f->nnz_pad = f->ntiles = f->nsegs = 0;
  f->tile_begin = f->tile_end = 0;
  *out = f;
  return FCOO_OK;
}

void destroy_impl(fcoo_s* f) {
  if (!f) return;
  free_handle_arrays(f);
  delete f;
}

}  // namespace fcoo
