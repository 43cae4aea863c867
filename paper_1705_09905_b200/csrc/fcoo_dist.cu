// fcoo_dist.cu — the distributed (row-partitioned) build and the owned-rows combine (SURVEY §8(e)
// alternative to the all-reduce, §8(f)-4 "distributed sample-sort build"; "multiple-GPUs can
// be used").
//
// Each rank starts from its own chunk of the COO.  For mode n the index-mode rows are split into
// nranks contiguous ranges balanced by nonzero count — the sample sort's splitter step, taken from
// the exact slice histogram (the index-mode key is dense: one counter per slice, all-reduced)
// instead of from samples; each rank buckets its nonzeros by destination (a stable radix sort on
// the destination rank), the buckets are exchanged in one grouped NCCL send/recv, and every rank
// builds the F-COO of ITS rows only.  Slices (the MTTKRP segments) never cross ranks, so
// each rank's SpMTTKRP rows are complete and the combine is an all-gather of owned row ranges
// (comm_gather_rows) instead of a sum all-reduce: about half the bytes, no redundant sort, and
// 1/nranks of the stream per rank.
#include <cub/cub.cuh>

#include "fcoo_internal.cuh"

namespace fcoo {

fcoo_status build_impl(const fcoo_coo* coo, int mode, const fcoo_build_opts* opts, const fcoo_allocator* alloc,
                       cudaStream_t s, fcoo_t* out);

namespace {

__global__ void k_slice_hist(const uint32_t* __restrict__ idx, int64_t nnz, uint32_t I, uint32_t* __restrict__ hist,
                             uint32_t* __restrict__ err) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const uint32_t i = idx[q];
  if (i >= I) {
    atomicOr(err, 1u);
    return;
  }
  atomicAdd(&hist[i], 1u);
}

// destination rank of nonzero q: the k with bounds[k] <= i_n < bounds[k+1]; its input ordinal
// rides along as the payload of the (stable) radix sort by destination
__global__ void k_dest(const uint32_t* __restrict__ idx, int64_t nnz, const int64_t* __restrict__ bounds, int nranks,
                       uint32_t* __restrict__ dest, uint32_t* __restrict__ ord, uint32_t* __restrict__ err) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const int64_t i = idx[q];
  if (i >= bounds[nranks]) atomicOr(err, 1u);
  int lo = 0, hi = nranks;  // bounds[lo] <= i < bounds[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= i) lo = mid; else hi = mid;
  }
  dest[q] = (uint32_t)lo;
  ord[q] = (uint32_t)q;
}

// counts[k] = number of sorted destination keys equal to k (binary searches, one thread per rank:
// no contended atomics over the nnz threads)
__global__ void k_dest_counts(const uint32_t* __restrict__ sorted, int64_t n, int nranks, uint32_t* __restrict__ counts) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nranks) return;
  auto lower = [&](uint32_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  counts[k] = (uint32_t)(lower((uint32_t)k + 1u) - lower((uint32_t)k));
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ ord, int64_t n,
                             uint32_t* __restrict__ dst) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) dst[p] = src[ord[p]];
}

int bits_for_n(int64_t n) {
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < n) ++b;
  return b;
}

fcoo_status check_coo_arrays(const fcoo_coo* coo, int mode) {
  if (!coo || !coo->dims || !coo->idx) return fail(FCOO_ERR_ARG, "NULL coo/dims/idx");
  if (coo->order < 2 || coo->order > kMaxOrder) return fail(FCOO_ERR_ORDER, "order %d outside [2,8]", coo->order);
  if (mode < 0 || mode >= coo->order) return fail(FCOO_ERR_MODE, "mode %d outside [0,%d)", mode, coo->order);
  if (coo->nnz < 0 || coo->nnz >= 4294967295LL) return fail(FCOO_ERR_ARG, "nnz must be in [0, 2^32)");
  if (coo->nnz > 0) {
    if (!coo->val) return fail(FCOO_ERR_ARG, "NULL val");
    for (int m = 0; m < coo->order; ++m)
      if (!coo->idx[m]) return fail(FCOO_ERR_ARG, "idx[%d] is NULL", m);
  }
  for (int m = 0; m < coo->order; ++m)
    if (coo->dims[m] < 1 || coo->dims[m] > 4294967295LL) return fail(FCOO_ERR_ARG, "dims[%d] outside [1,2^32)", m);
  return FCOO_OK;
}

fcoo_status slice_hist(const fcoo_coo* coo, int mode, uint32_t* hist, const Alloc& al, cudaStream_t s) {
  const uint32_t I = (uint32_t)coo->dims[mode];
  FCOO_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)I, s));
  if (coo->nnz == 0) return FCOO_OK;
  Buf err(&al, sizeof(uint32_t), s);
  if (!err.ok()) return fail(FCOO_ERR_OOM, "histogram scratch");
  FCOO_CUDA_TRY(cudaMemsetAsync(err.p, 0, sizeof(uint32_t), s));
  k_slice_hist<<<(unsigned)((coo->nnz + 255) / 256), 256, 0, s>>>(coo->idx[mode], coo->nnz, I, hist, err.as<uint32_t>());
  FCOO_LAUNCH_CHECK();
  uint32_t e = 0;
  FCOO_CUDA_TRY(cudaMemcpyAsync(&e, err.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  FCOO_CUDA_TRY(cudaStreamSynchronize(s));
  if (e) return fail(FCOO_ERR_INDEX_RANGE, "a mode-%d coordinate is >= %u", mode, I);
  return FCOO_OK;
}

fcoo_status row_partition(const uint32_t* hist, int64_t I, int nranks, int64_t* bounds) {
  if (!hist || !bounds || I < 1 || nranks < 1) return fail(FCOO_ERR_ARG, "bad row partition arguments");
  int64_t nnz = 0;
  for (int64_t i = 0; i < I; ++i) nnz += hist[i];
  bounds[0] = 0;
  int64_t r = 0, pre = 0;  // pre = sum of hist[0..r)
  for (int k = 1; k < nranks; ++k) {
    const int64_t target = (k * nnz + nranks - 1) / nranks;  // ceil(k * nnz / nranks)
    while (r < I && pre < target) pre += hist[r++];
    bounds[k] = r;
  }
  bounds[nranks] = I;
  return FCOO_OK;
}

// Stable partition of the local nonzeros by destination rank (grouped in rank order, input order
// kept inside a group) into idx_out / val_out; counts[k] = nonzeros for rank k.  Synchronises.
fcoo_status bucket_rows(const fcoo_coo* coo, int mode, const int64_t* bounds, int nranks, uint32_t* const* idx_out,
                        float* val_out, int64_t* counts, const Alloc& al, cudaStream_t s) {
  const int64_t nnz = coo->nnz;
  for (int k = 0; k < nranks; ++k) counts[k] = 0;
  if (nnz == 0) return FCOO_OK;
  Buf db(&al, sizeof(int64_t) * (nranks + 1), s), cnt(&al, sizeof(uint32_t) * (nranks + 1), s);
  Buf d0(&al, sizeof(uint32_t) * nnz, s), d1(&al, sizeof(uint32_t) * nnz, s);
  Buf o0(&al, sizeof(uint32_t) * nnz, s), o1(&al, sizeof(uint32_t) * nnz, s);
  if (!db.ok() || !cnt.ok() || !d0.ok() || !d1.ok() || !o0.ok() || !o1.ok())
    return fail(FCOO_ERR_OOM, "bucket scratch allocation failed");
  FCOO_CUDA_TRY(cudaMemcpyAsync(db.p, bounds, sizeof(int64_t) * (nranks + 1), cudaMemcpyHostToDevice, s));
  FCOO_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * (nranks + 1), s));
  uint32_t* err = cnt.as<uint32_t>() + nranks;
  const unsigned grid = (unsigned)((nnz + 255) / 256);
  k_dest<<<grid, 256, 0, s>>>(coo->idx[mode], nnz, db.as<int64_t>(), nranks, d0.as<uint32_t>(), o0.as<uint32_t>(), err);
  FCOO_LAUNCH_CHECK();
  cub::DoubleBuffer<uint32_t> dk(d0.as<uint32_t>(), d1.as<uint32_t>()), dv(o0.as<uint32_t>(), o1.as<uint32_t>());
  const int bits = std::max(1, bits_for_n(nranks));
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, nnz, 0, bits, s);
  {
    Buf tmp(&al, tmp_bytes, s);
    if (!tmp.ok()) return fail(FCOO_ERR_OOM, "radix sort scratch");
    cudaError_t ce = cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, dk, dv, nnz, 0, bits, s);
    if (ce != cudaSuccess) return fail(FCOO_ERR_CUDA, "bucket sort: %s", cudaGetErrorString(ce));
    count_launch(2 + (bits + 7) / 8);
  }
  const uint32_t* ord = dv.Current();
  k_dest_counts<<<(unsigned)((nranks + 127) / 128), 128, 0, s>>>(dk.Current(), nnz, nranks, cnt.as<uint32_t>());
  FCOO_LAUNCH_CHECK();
  for (int m = 0; m < coo->order; ++m) {
    k_gather_u32<<<grid, 256, 0, s>>>(coo->idx[m], ord, nnz, idx_out[m]);
    FCOO_LAUNCH_CHECK();
  }
  k_gather_u32<<<grid, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(coo->val), ord, nnz,
                                    reinterpret_cast<uint32_t*>(val_out));
  FCOO_LAUNCH_CHECK();
  std::vector<uint32_t> h(nranks + 1);
  FCOO_CUDA_TRY(cudaMemcpyAsync(h.data(), cnt.p, sizeof(uint32_t) * (nranks + 1), cudaMemcpyDeviceToHost, s));
  FCOO_CUDA_TRY(cudaStreamSynchronize(s));
  if (h[nranks]) return fail(FCOO_ERR_INDEX_RANGE, "a mode-%d coordinate is beyond the last row bound", mode);
  for (int k = 0; k < nranks; ++k) counts[k] = h[k];
  return FCOO_OK;
}

__global__ void k_row_minmax(const uint32_t* __restrict__ seg_coord, int64_t nsegs, int n_idx,
                             uint32_t* __restrict__ mm) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t lo = 0xffffffffu, hi = 0u;
  if (s < nsegs) lo = hi = seg_coord[s * n_idx];
  for (int o = 16; o > 0; o >>= 1) {  // warp reduction, one atomic pair per warp
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

}  // namespace

fcoo_status set_row_shard(fcoo_s* f, int rank, int nranks, const int64_t* bounds, fcoo_comm_t comm) {
  if (!f || !bounds || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FCOO_ERR_ARG, "bad row shard %d/%d", rank, nranks);
  if (f->op != FCOO_OP_MTTKRP) return fail(FCOO_ERR_SHAPE, "row shards are for SpMTTKRP handles");
  if (f->nshards > 1) return fail(FCOO_ERR_ARG, "handle is already tile-sharded (fcoo_set_shard)");
  const int64_t I = f->dims[f->mode];
  if (bounds[0] != 0 || bounds[nranks] != I) return fail(FCOO_ERR_ARG, "row bounds must run from 0 to I_n = %lld", (long long)I);
  for (int k = 0; k < nranks; ++k)
    if (bounds[k + 1] < bounds[k]) return fail(FCOO_ERR_ARG, "row bounds must be non-decreasing");
  if (comm) {
    int cr = 0, cn = 1;
    comm_rank_size(comm, &cr, &cn);
    if (cr != rank || cn != nranks) return fail(FCOO_ERR_ARG, "row shard %d/%d does not match comm rank %d/%d", rank, nranks, cr, cn);
  }
  // every nonzero of the handle must lie in the rank's rows, or the gather would drop it
  if (f->nnz > 0) {
    uint32_t mm[2] = {0, 0};
    if (f->dense_rows) {
      mm[0] = 0;
      mm[1] = (uint32_t)(I - 1);
    } else {
      Buf d(&f->alloc, sizeof(uint32_t) * 2, f->build_stream);
      if (!d.ok()) return fail(FCOO_ERR_OOM, "row check scratch");
      const uint32_t init[2] = {0xffffffffu, 0u};
      FCOO_CUDA_TRY(cudaMemcpyAsync(d.p, init, sizeof(init), cudaMemcpyHostToDevice, f->build_stream));
      k_row_minmax<<<(unsigned)((f->nsegs + 255) / 256), 256, 0, f->build_stream>>>(f->seg_coord, f->nsegs, f->n_idx,
                                                                                   d.as<uint32_t>());
      FCOO_LAUNCH_CHECK();
      FCOO_CUDA_TRY(cudaMemcpyAsync(mm, d.p, sizeof(mm), cudaMemcpyDeviceToHost, f->build_stream));
      FCOO_CUDA_TRY(cudaStreamSynchronize(f->build_stream));
    }
    if ((int64_t)mm[0] < bounds[rank] || (int64_t)mm[1] >= bounds[rank + 1])
      return fail(FCOO_ERR_ARG, "handle has rows [%u, %u], outside the shard's [%lld, %lld)", mm[0], mm[1],
                  (long long)bounds[rank], (long long)bounds[rank + 1]);
  }
  f->row_sharded = nranks > 1 ? 1 : 0;
  f->row_rank = rank;
  f->row_nranks = nranks;
  f->row_bounds.assign(bounds, bounds + nranks + 1);
  f->row_comm = nranks > 1 ? comm : nullptr;
  return FCOO_OK;
}

}  // namespace fcoo

extern "C" {

fcoo_status fcoo_slice_histogram(const fcoo_coo* coo, int mode, uint32_t* hist, void* stream) {
  fcoo_status st = fcoo::check_coo_arrays(coo, mode);
  if (st) return st;
  if (!hist) return fcoo::fail(FCOO_ERR_ARG, "NULL hist");
  fcoo::Alloc al;
  return fcoo::slice_hist(coo, mode, hist, al, (cudaStream_t)stream);
}

fcoo_status fcoo_row_partition(const uint32_t* hist, int64_t I, int nranks, int64_t* bounds) {
  return fcoo::row_partition(hist, I, nranks, bounds);
}

fcoo_status fcoo_bucket_rows(const fcoo_coo* coo, int mode, const int64_t* bounds, int nranks,
                             uint32_t* const* idx_out, float* val_out, int64_t* counts, const fcoo_allocator* alloc,
                             void* stream) {
  fcoo_status st = fcoo::check_coo_arrays(coo, mode);
  if (st) return st;
  if (!bounds || nranks < 1 || !counts || (coo->nnz > 0 && (!idx_out || !val_out)))
    return fcoo::fail(FCOO_ERR_ARG, "NULL bounds/idx_out/val_out/counts or nranks < 1");
  if (coo->nnz > 0)
    for (int m = 0; m < coo->order; ++m)
      if (!idx_out[m]) return fcoo::fail(FCOO_ERR_ARG, "idx_out[%d] is NULL", m);
  fcoo::Alloc al;
  if (alloc && alloc->alloc && alloc->free) { al.a = *alloc; al.custom = true; }
  return fcoo::bucket_rows(coo, mode, bounds, nranks, idx_out, val_out, counts, al, (cudaStream_t)stream);
}

fcoo_status fcoo_set_row_shard(fcoo_t f, int rank, int nranks, const int64_t* bounds, fcoo_comm_t comm) {
  return fcoo::set_row_shard(f, rank, nranks, bounds, comm);
}

fcoo_status fcoo_build_distributed(const fcoo_coo* local, int mode, const fcoo_build_opts* opts, fcoo_comm_t comm,
                                   const fcoo_allocator* alloc, void* stream, fcoo_t* out) {
  using namespace fcoo;
  Nvtx range("fcoo_build_distributed");
  if (!comm || !out) return fail(FCOO_ERR_ARG, "NULL comm/out");
  *out = nullptr;
  fcoo_status st = check_coo_arrays(local, mode);
  if (st) return st;
  if (opts && opts->op != FCOO_OP_MTTKRP) return fail(FCOO_ERR_SHAPE, "the distributed build is for SpMTTKRP handles");
  // a permutation would index this rank's RECEIVED nonzeros, not the caller's chunk: not offered
  if (opts && (opts->flags & FCOO_BUILD_KEEP_PERM)) return fail(FCOO_ERR_ARG, "KEEP_PERM is not available in the distributed build");
  cudaStream_t s = (cudaStream_t)stream;
  int rank = 0, nranks = 1;
  comm_rank_size(comm, &rank, &nranks);
  Alloc al;
  if (alloc && alloc->alloc && alloc->free) { al.a = *alloc; al.custom = true; }
  const int order = local->order;
  const int64_t I = local->dims[mode], nnz = local->nnz;
  // 1. global slice histogram -> row bounds (identical on every rank)
  std::vector<int64_t> bounds(nranks + 1);
  {
    Buf hist(&al, sizeof(uint32_t) * (size_t)I, s);
    st = hist.ok() ? slice_hist(local, mode, hist.as<uint32_t>(), al, s) : fail(FCOO_ERR_OOM, "histogram allocation");
    st = comm_agree(comm, st, s);  // a bad coordinate on one rank stops every rank here
    if (st) return st;
    st = comm_allreduce_u32(comm, hist.as<uint32_t>(), (size_t)I, s);
    if (st) return st;
    std::vector<uint32_t> h(I);
    FCOO_CUDA_TRY(cudaMemcpyAsync(h.data(), hist.p, sizeof(uint32_t) * (size_t)I, cudaMemcpyDeviceToHost, s));
    FCOO_CUDA_TRY(cudaStreamSynchronize(s));
    st = row_partition(h.data(), I, nranks, bounds.data());
    if (st) return st;
  }
  // 2. bucket the local nonzeros by destination rank
  std::vector<Buf*> bufs;
  auto release = [&]() { for (Buf* b : bufs) delete b; bufs.clear(); };
  auto buf = [&](size_t bytes) { bufs.push_back(new Buf(&al, bytes, s)); return bufs.back(); };
  std::vector<uint32_t*> sidx(order), ridx(order);
  for (int m = 0; m < order; ++m) sidx[m] = buf(sizeof(uint32_t) * (size_t)nnz)->as<uint32_t>();
  float* sval = buf(sizeof(float) * (size_t)nnz)->as<float>();
  std::vector<int64_t> send(nranks, 0), recv(nranks, 0);
  st = FCOO_OK;
  for (Buf* b : bufs) if (!b->ok()) st = fail(FCOO_ERR_OOM, "send buffers");
  if (!st) st = bucket_rows(local, mode, bounds.data(), nranks, sidx.data(), sval, send.data(), al, s);
  Buf sc(&al, sizeof(uint64_t) * nranks, s), all(&al, sizeof(uint64_t) * (size_t)nranks * nranks, s);
  if (!st && (!sc.ok() || !all.ok())) st = fail(FCOO_ERR_OOM, "count buffers");
  st = comm_agree(comm, st, s);
  if (st) { release(); return st; }
  // 3. who sends how much to whom: all-gather of every rank's per-destination counts
  {
    std::vector<uint64_t> h(send.begin(), send.end()), ha((size_t)nranks * nranks);
    if (cudaMemcpyAsync(sc.p, h.data(), sizeof(uint64_t) * nranks, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      release();
      return fail(FCOO_ERR_CUDA, "count upload");
    }
    st = comm_allgather_u64(comm, sc.as<uint64_t>(), all.as<uint64_t>(), (size_t)nranks, s);
    if (st) { release(); return st; }
    if (cudaMemcpyAsync(ha.data(), all.p, sizeof(uint64_t) * ha.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      release();
      return fail(FCOO_ERR_CUDA, "count download");
    }
    for (int j = 0; j < nranks; ++j) recv[j] = (int64_t)ha[(size_t)j * nranks + rank];
  }
  int64_t total = 0;
  for (int j = 0; j < nranks; ++j) total += recv[j];
  st = total >= 4294967295LL ? fail(FCOO_ERR_ARG, "rank %d would receive %lld >= 2^32 nonzeros", rank, (long long)total)
                             : FCOO_OK;
  // 4. the exchange: one grouped send/recv per array (the own bucket by a device copy)
  float* rval = nullptr;
  if (!st) {
    for (int m = 0; m < order; ++m) ridx[m] = buf(sizeof(uint32_t) * (size_t)total)->as<uint32_t>();
    rval = buf(sizeof(float) * (size_t)total)->as<float>();
    for (Buf* b : bufs) if (!b->ok()) st = fail(FCOO_ERR_OOM, "receive buffers");
  }
  st = comm_agree(comm, st, s);
  if (st) { release(); return st; }
  for (int m = 0; m < order && !st; ++m)
    st = comm_exchange(comm, sidx[m], send.data(), ridx[m], recv.data(), sizeof(uint32_t), s);
  if (!st) st = comm_exchange(comm, sval, send.data(), rval, recv.data(), sizeof(float), s);
  if (st) { release(); return st; }
  // 5. the F-COO of this rank's rows (an empty handle if a heavy slice left it none)
  fcoo_t f = nullptr;
  if (total == 0) {
    st = build_empty(order, local->dims, FCOO_OP_MTTKRP, mode, alloc, s, &f);
  } else {
    const uint32_t* ip[kMaxOrder];
    for (int m = 0; m < order; ++m) ip[m] = ridx[m];
    fcoo_coo mine{order, local->dims, total, ip, rval};
    st = build_impl(&mine, mode, opts, alloc, s, &f);
  }
  if (!st) {
    // the exchanged buffers are freed on the stream after the build's last use (stream order)
    st = set_row_shard(f, rank, nranks, bounds.data(), comm);
    if (st) fcoo_destroy(f);
  }
  release();
  if (st) return st;
  *out = f;
  return FCOO_OK;
}

}  // extern "C"
