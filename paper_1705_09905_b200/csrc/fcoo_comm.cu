// fcoo_comm.cu — multi-GPU combine: the only cross-GPU step of the
// path is a per-mode sum all-reduce of the partial MTTKRP output over NVLink/NVSwitch (NCCL picks
// NVLS in-switch reduction where available).  One process per GPU; the 128-byte NCCL unique id
// is broadcast by the caller (torch.distributed in the Python binding).
#include <cuda.h>  // driver API types only; entry points come from cudaGetDriverEntryPoint
#include <nccl.h>
#include <string.h>

#include "fcoo_internal.cuh"

struct fcoo_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int device = 0;
  int* scratch = nullptr;  // one device int: the payload of the stream-ordered barrier
};

// An output buffer bound to an NVLink SHARP (NVLS) multicast object: every rank of the comm owns
// `bytes` of its own HBM (`uc`, its unicast view) and all ranks share one multicast address range
// (`mc`): a multimem.st there writes every rank's copy, a multimem.red.add is reduced in the
// NVSwitch and lands in every copy.  SURVEY §8(f)-2.
struct fcoo_mc_s {
  fcoo_comm_t comm = nullptr;
  size_t bytes = 0, size = 0;  // requested, and rounded to the multicast granularity
  CUmemGenericAllocationHandle mem = 0, mcobj = 0;
  CUdeviceptr uc = 0, mc = 0;
  bool bound = false, uc_mapped = false, mc_mapped = false;
};

namespace fcoo {

// Status of an enqueued NCCL call: the immediate result, then the communicator's asynchronous
// error state (ncclCommGetAsyncError, non-blocking: a peer failure or a network error surfaces
// here on the next collective instead of as a hang) -> FCOO_ERR_NCCL.
static fcoo_status nccl_status(fcoo_comm_t c, ncclResult_t r, const char* what) {
  if (r != ncclSuccess && r != ncclInProgress) return fail(FCOO_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
  ncclResult_t ae = ncclSuccess;
  if (ncclCommGetAsyncError(c->comm, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress))
    return fail(FCOO_ERR_NCCL, "%s: communicator error: %s", what, ncclGetErrorString(ae));
  count_launch();
  return FCOO_OK;
}

fcoo_status comm_allreduce(fcoo_comm_t c, float* buf, size_t count, cudaStream_t s) {
  Nvtx range("ncclAllReduce");
  if (!c || !c->comm) return FCOO_OK;
  return nccl_status(c, ncclAllReduce(buf, buf, count, ncclFloat, ncclSum, c->comm, s), "ncclAllReduce");
}

fcoo_status comm_allreduce_f64(fcoo_comm_t c, double* buf, size_t count, cudaStream_t s) {
  Nvtx range("ncclAllReduce(f64)");
  if (!c || !c->comm) return FCOO_OK;
  return nccl_status(c, ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c->comm, s), "ncclAllReduce(f64)");
}

// Stream-ordered barrier over the comm: a one-element all-reduce completes on a rank only after
// every rank has reached it (and, by stream order, finished the work enqueued before it).
fcoo_status comm_barrier(fcoo_comm_t c, cudaStream_t s) {
  if (!c || !c->comm) return FCOO_OK;
  return nccl_status(c, ncclAllReduce(c->scratch, c->scratch, 1, ncclInt, ncclSum, c->comm, s), "barrier");
}

// Owned-rows combine ("boundary-row fixup + all-gather of owned rows, which halves
// the bytes" of the all-reduce): on a row-sharded handle no row is partial on two ranks, so rank k
// broadcasts its complete rows [bounds[k], bounds[k+1]) in place; the nranks broadcasts form one
// NCCL group (one launch).  Every rank calls it with the same bounds.
template <class T>
static fcoo_status gather_rows_t(fcoo_comm_t c, T* out, const std::vector<int64_t>& bounds, int R, ncclDataType_t ty,
                                 cudaStream_t s) {
  Nvtx range("owned-rows gather");
  if (!c || !c->comm || c->nranks == 1) return FCOO_OK;
  if ((int)bounds.size() != c->nranks + 1) return fail(FCOO_ERR_ARG, "row bounds for %d ranks, comm has %d",
                                                       (int)bounds.size() - 1, c->nranks);
  ncclResult_t r = ncclGroupStart();
  for (int k = 0; k < c->nranks && r == ncclSuccess; ++k) {
    const size_t n = (size_t)(bounds[k + 1] - bounds[k]) * (size_t)R;
    if (n == 0) continue;
    T* p = out + (size_t)bounds[k] * (size_t)R;
    r = ncclBroadcast(p, p, n, ty, k, c->comm, s);
  }
  const ncclResult_t r2 = ncclGroupEnd();
  return nccl_status(c, r != ncclSuccess ? r : r2, "owned-rows gather (ncclBroadcast group)");
}

fcoo_status comm_gather_rows(fcoo_comm_t c, float* out, const std::vector<int64_t>& bounds, int R, cudaStream_t s) {
  return gather_rows_t<float>(c, out, bounds, R, ncclFloat, s);
}

fcoo_status comm_gather_rows_f64(fcoo_comm_t c, double* out, const std::vector<int64_t>& bounds, int R,
                                 cudaStream_t s) {
  return gather_rows_t<double>(c, out, bounds, R, ncclDouble, s);
}

// Collective status agreement: every rank passes its local status and all return the largest one
// (FCOO_OK only if every rank succeeded), so a local failure before a collective step makes every
// rank stop instead of leaving the others blocked in that collective.  Synchronises `s`.
fcoo_status comm_agree(fcoo_comm_t c, fcoo_status local, cudaStream_t s) {
  if (!c || !c->comm || c->nranks == 1) return local;
  int v = (int)local;
  if (cudaMemcpyAsync(c->scratch, &v, sizeof(int), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "status agreement upload");
  fcoo_status st = nccl_status(c, ncclAllReduce(c->scratch, c->scratch, 1, ncclInt, ncclMax, c->comm, s), "agree");
  if (st) return st;
  if (cudaMemcpyAsync(&v, c->scratch, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemsetAsync(c->scratch, 0, sizeof(int), s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "status agreement download");
  if (v != (int)FCOO_OK && local == FCOO_OK) return fail((fcoo_status)v, "another rank failed (status %d)", v);
  return v == (int)FCOO_OK ? FCOO_OK : local;
}

fcoo_status comm_allreduce_u32(fcoo_comm_t c, uint32_t* buf, size_t count, cudaStream_t s) {
  if (!c || !c->comm) return FCOO_OK;
  return nccl_status(c, ncclAllReduce(buf, buf, count, ncclUint32, ncclSum, c->comm, s), "ncclAllReduce(u32)");
}

fcoo_status comm_allgather_u64(fcoo_comm_t c, const uint64_t* send, uint64_t* recv, size_t count, cudaStream_t s) {
  if (!c || !c->comm) return fail(FCOO_ERR_ARG, "all-gather needs a comm");
  return nccl_status(c, ncclAllGather(send, recv, count, ncclUint64, c->comm, s), "ncclAllGather(u64)");
}

// Grouped point-to-point exchange (the all-to-all of the distributed build): items of `elem`
// bytes, send_counts[j] of them to rank j from consecutive ranges of sendbuf, recv_counts[j] from
// rank j into consecutive ranges of recvbuf (the own bucket by a device copy).  Counts must agree pairwise.
fcoo_status comm_exchange(fcoo_comm_t c, const void* sendbuf, const int64_t* send_counts, void* recvbuf,
                          const int64_t* recv_counts, size_t elem, cudaStream_t s) {
  if (!c || !c->comm) return fail(FCOO_ERR_ARG, "exchange needs a comm");
  const char* sb = static_cast<const char*>(sendbuf);
  char* rb = static_cast<char*>(recvbuf);
  size_t so = 0, ro = 0, self_so = 0, self_ro = 0, self_n = 0;
  ncclResult_t r = ncclGroupStart();
  for (int j = 0; j < c->nranks && r == ncclSuccess; ++j) {
    const size_t ns = (size_t)send_counts[j] * elem, nr = (size_t)recv_counts[j] * elem;
    if (j == c->rank) {  // this rank's own bucket: a device copy, not a NCCL self send/recv
      self_so = so, self_ro = ro, self_n = ns;
    } else {
      if (ns) r = ncclSend(sb + so, ns, ncclUint8, j, c->comm, s);
      if (r == ncclSuccess && nr) r = ncclRecv(rb + ro, nr, ncclUint8, j, c->comm, s);
    }
    so += ns;
    ro += nr;
  }
  const ncclResult_t r2 = ncclGroupEnd();
  if (self_n && cudaMemcpyAsync(rb + self_ro, sb + self_so, self_n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(FCOO_ERR_CUDA, "exchange: own bucket copy");
  return nccl_status(c, r != ncclSuccess ? r : r2, "exchange (ncclSend/ncclRecv group)");
}

void comm_rank_size(fcoo_comm_t c, int* rank, int* nranks) {
  *rank = c ? c->rank : 0;
  *nranks = c ? c->nranks : 1;
}

}  // namespace fcoo

extern "C" {

fcoo_status fcoo_comm_unique_id(void* out128) {
  if (!out128) return fcoo::fail(FCOO_ERR_ARG, "NULL out");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fcoo::fail(FCOO_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return FCOO_OK;
}

fcoo_status fcoo_comm_init(int rank, int nranks, const void* uid128, fcoo_comm_t* out) {
  if (!out || !uid128 || nranks < 1 || rank < 0 || rank >= nranks) return fcoo::fail(FCOO_ERR_ARG, "bad comm args");
  fcoo_comm_s* c = new fcoo_comm_s();
  c->rank = rank;
  c->nranks = nranks;
  // a 1-rank communicator is a real NCCL communicator too (the handles never attach it: sharding
  // into one shard drops the comm), so the NCCL path can be exercised on a single GPU
  {
    cudaGetDevice(&c->device);
    if (cudaMalloc(&c->scratch, sizeof(int)) != cudaSuccess || cudaMemset(c->scratch, 0, sizeof(int)) != cudaSuccess) {
      delete c;
      return fcoo::fail(FCOO_ERR_OOM, "comm scratch");
    }
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      cudaFree(c->scratch);
      delete c;
      return fcoo::fail(FCOO_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = c;
  return FCOO_OK;
}

fcoo_status fcoo_comm_destroy(fcoo_comm_t c) {
  if (!c) return FCOO_OK;
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->scratch) cudaFree(c->scratch);
  delete c;
  return FCOO_OK;
}

fcoo_status fcoo_allreduce_sum(fcoo_comm_t c, float* buf, size_t count, void* stream) {
  if (!c || !buf) return fcoo::fail(FCOO_ERR_ARG, "NULL comm/buf");
  return fcoo::comm_allreduce(c, buf, count, (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// NVLS multicast output buffers
namespace fcoo {
namespace {

struct Drv {
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) allocGranularity = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceAttr = nullptr;
  bool ok = false;
};

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
          !*fn)
        ok = false;
    };
    get("cuMulticastCreate", (void**)&x.mcCreate);
    get("cuMulticastAddDevice", (void**)&x.mcAddDevice);
    get("cuMulticastBindMem", (void**)&x.mcBindMem);
    get("cuMulticastUnbind", (void**)&x.mcUnbind);
    get("cuMulticastGetGranularity", (void**)&x.mcGranularity);
    get("cuMemCreate", (void**)&x.memCreate);
    get("cuMemRelease", (void**)&x.memRelease);
    get("cuMemAddressReserve", (void**)&x.addrReserve);
    get("cuMemAddressFree", (void**)&x.addrFree);
    get("cuMemMap", (void**)&x.memMap);
    get("cuMemUnmap", (void**)&x.memUnmap);
    get("cuMemSetAccess", (void**)&x.setAccess);
    get("cuMemGetAllocationGranularity", (void**)&x.allocGranularity);
    get("cuMemExportToShareableHandle", (void**)&x.exportHandle);
    get("cuMemImportFromShareableHandle", (void**)&x.importHandle);
    get("cuDeviceGet", (void**)&x.deviceGet);
    get("cuDeviceGetAttribute", (void**)&x.deviceAttr);
    x.ok = ok;
    return x;
  }();
  return d;
}

void mc_release(fcoo_mc_s* m) {
  const Drv& d = drv();
  if (!d.ok || !m) return;
  if (m->mc_mapped) d.memUnmap(m->mc, m->size);
  if (m->mc) d.addrFree(m->mc, m->size);
  if (m->uc_mapped) d.memUnmap(m->uc, m->size);
  if (m->uc) d.addrFree(m->uc, m->size);
  if (m->bound) {
    CUdevice dev;
    if (d.deviceGet(&dev, m->comm->device) == CUDA_SUCCESS) d.mcUnbind(m->mcobj, dev, 0, m->size);
  }
  if (m->mem) d.memRelease(m->mem);
  if (m->mcobj) d.memRelease(m->mcobj);
}

// Host-level collective step: every rank's enqueued work done, then a barrier, then wait for it.
fcoo_status host_barrier(fcoo_comm_t c) {
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return fail(FCOO_ERR_CUDA, "barrier stream");
  fcoo_status st = comm_barrier(c, s);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (st) return st;
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "barrier: %s", cudaGetErrorString(e));
  return FCOO_OK;
}

// Collective agreement: 1 on every rank iff `ok` is nonzero on every rank (min all-reduce on a
// private stream, host-synchronous).  fcoo_mc_alloc calls it after every step that can fail on one
// rank only, so all ranks bail out together instead of leaving the others blocked in a collective.
bool agree_ok(fcoo_comm_t c, int ok) {
  if (c->nranks == 1) return ok != 0;
  int* d = nullptr;
  cudaStream_t s = nullptr;
  int res = 0;
  if (cudaMalloc(&d, sizeof(int)) == cudaSuccess && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
      cudaMemcpyAsync(d, &ok, sizeof(int), cudaMemcpyHostToDevice, s) == cudaSuccess &&
      ncclAllReduce(d, d, 1, ncclInt, ncclMin, c->comm, s) == ncclSuccess &&
      cudaMemcpyAsync(&res, d, sizeof(int), cudaMemcpyDeviceToHost, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess) {
  } else {
    res = 0;
  }
  if (s) cudaStreamDestroy(s);
  if (d) cudaFree(d);
  return res != 0;
}

// rank `root`'s n bytes to every rank (ncclBroadcast through a device staging buffer)
fcoo_status bcast_bytes(fcoo_comm_t c, void* host, size_t n, int root) {
  if (c->nranks == 1) return FCOO_OK;
  void* dbuf = nullptr;
  cudaStream_t s = nullptr;
  if (cudaMalloc(&dbuf, n) != cudaSuccess) return fail(FCOO_ERR_OOM, "bcast staging");
  fcoo_status st = FCOO_OK;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) st = fail(FCOO_ERR_CUDA, "bcast stream");
  if (!st && cudaMemcpyAsync(dbuf, host, n, cudaMemcpyHostToDevice, s) != cudaSuccess) st = fail(FCOO_ERR_CUDA, "bcast h2d");
  if (!st) {
    ncclResult_t r = ncclBroadcast(dbuf, dbuf, n, ncclChar, root, c->comm, s);
    if (r != ncclSuccess) st = fail(FCOO_ERR_NCCL, "ncclBroadcast: %s", ncclGetErrorString(r));
  }
  if (!st && cudaMemcpyAsync(host, dbuf, n, cudaMemcpyDeviceToHost, s) != cudaSuccess) st = fail(FCOO_ERR_CUDA, "bcast d2h");
  if (!st && cudaStreamSynchronize(s) != cudaSuccess) st = fail(FCOO_ERR_CUDA, "bcast sync");
  if (s) cudaStreamDestroy(s);
  cudaFree(dbuf);
  return st;
}

}  // namespace
}  // namespace fcoo

extern "C" {

fcoo_status fcoo_mc_alloc(fcoo_comm_t c, size_t bytes, fcoo_mc_t* out) {
  using namespace fcoo;
  if (!c || !out || bytes == 0) return fail(FCOO_ERR_ARG, "fcoo_mc_alloc: NULL comm/out or zero bytes");
  if (!c->comm) return fail(FCOO_ERR_ARG, "fcoo_mc_alloc: comm has no NCCL communicator");
  const Drv& d = drv();
  if (!d.ok) return fail(FCOO_ERR_CUDA, "fcoo_mc_alloc: driver entry points unavailable");
  CUdevice dev;
  if (d.deviceGet(&dev, c->device) != CUDA_SUCCESS) return fail(FCOO_ERR_CUDA, "cuDeviceGet");
  int mcs = 0;
  d.deviceAttr(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  if (!agree_ok(c, mcs)) return fail(FCOO_ERR_ARG, "fcoo_mc_alloc: a device of the comm does not support NVLS multicast");
  const bool shared = c->nranks > 1;
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)c->nranks;
  mp.handleTypes = shared ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_NONE;
  mp.size = bytes;
  size_t g_mc = 0, g_mem = 0;
  if (d.mcGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
    return fail(FCOO_ERR_CUDA, "cuMulticastGetGranularity");
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
  if (d.allocGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS)
    return fail(FCOO_ERR_CUDA, "cuMemGetAllocationGranularity");
  const size_t g = g_mc > g_mem ? g_mc : g_mem;
  fcoo_mc_s* m = new fcoo_mc_s();
  m->comm = c;
  m->bytes = bytes;
  m->size = mp.size = (bytes + g - 1) / g * g;
  auto bail = [&](fcoo_status st) {
    mc_release(m);
    delete m;
    return st;
  };
  // rank 0 creates the multicast object and shares it as a fabric handle (bytes over NCCL)
  CUmemFabricHandle fh;
  memset(&fh, 0, sizeof(fh));
  int ok0 = 1;
  CUresult cr = CUDA_SUCCESS;
  if (c->rank == 0) {
    cr = d.mcCreate(&m->mcobj, &mp);
    if (cr != CUDA_SUCCESS && !shared) {  // some drivers want a shareable handle type even for one device
      mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
      cr = d.mcCreate(&m->mcobj, &mp);
    }
    ok0 = cr == CUDA_SUCCESS;
    if (ok0 && shared) {
      cr = d.exportHandle(&fh, m->mcobj, CU_MEM_HANDLE_TYPE_FABRIC, 0);
      ok0 = cr == CUDA_SUCCESS;
    }
  }
  // from here on every failure point is agreed on by all ranks (agree_ok) before anyone bails,
  // so a failure on one rank never leaves the others blocked in a later collective
  fcoo_status err = FCOO_OK;
  auto failed_somewhere = [&](fcoo_status local) {
    if (local && !err) err = local;
    if (agree_ok(c, local == FCOO_OK)) return false;
    if (!err) err = fail(FCOO_ERR_CUDA, "fcoo_mc_alloc: a step failed on another rank");
    return true;
  };
  if (shared) {
    struct { CUmemFabricHandle h; int ok; } msg;
    msg.h = fh;
    msg.ok = ok0;
    fcoo_status st = bcast_bytes(c, &msg, sizeof(msg), 0);
    if (st) return bail(st);
    if (!msg.ok) return bail(fail(FCOO_ERR_CUDA, "cuMulticastCreate/export failed on rank 0 (CUresult %d)", (int)cr));
    fcoo_status imp = FCOO_OK;
    if (c->rank != 0 && d.importHandle(&m->mcobj, &msg.h, CU_MEM_HANDLE_TYPE_FABRIC) != CUDA_SUCCESS)
      imp = fail(FCOO_ERR_CUDA, "cuMemImportFromShareableHandle (multicast)");
    if (failed_somewhere(imp)) return bail(err);
  } else if (!ok0) {
    return bail(fail(FCOO_ERR_CUDA, "cuMulticastCreate: CUresult %d", (int)cr));
  }
  fcoo_status add = FCOO_OK;
  if ((cr = d.mcAddDevice(m->mcobj, dev)) != CUDA_SUCCESS) add = fail(FCOO_ERR_CUDA, "cuMulticastAddDevice: CUresult %d", (int)cr);
  if (failed_somewhere(add)) return bail(err);
  // every device must be added before any rank binds memory
  fcoo_status st = host_barrier(c);
  if (st) return bail(st);
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  auto setup = [&]() -> fcoo_status {  // local steps; the first failure is reported
    if (d.memCreate(&m->mem, m->size, &ap, 0) != CUDA_SUCCESS) return fail(FCOO_ERR_OOM, "cuMemCreate");
    if ((cr = d.mcBindMem(m->mcobj, 0, m->mem, 0, m->size, 0)) != CUDA_SUCCESS)
      return fail(FCOO_ERR_CUDA, "cuMulticastBindMem: CUresult %d", (int)cr);
    m->bound = true;
    if (d.addrReserve(&m->uc, m->size, g, 0, 0) != CUDA_SUCCESS) return fail(FCOO_ERR_OOM, "VA reserve (unicast)");
    if (d.memMap(m->uc, m->size, 0, m->mem, 0) != CUDA_SUCCESS) return fail(FCOO_ERR_CUDA, "cuMemMap (unicast)");
    m->uc_mapped = true;
    if (d.setAccess(m->uc, m->size, &acc, 1) != CUDA_SUCCESS) return fail(FCOO_ERR_CUDA, "cuMemSetAccess (unicast)");
    if (d.addrReserve(&m->mc, m->size, g, 0, 0) != CUDA_SUCCESS) return fail(FCOO_ERR_OOM, "VA reserve (multicast)");
    if (d.memMap(m->mc, m->size, 0, m->mcobj, 0) != CUDA_SUCCESS) return fail(FCOO_ERR_CUDA, "cuMemMap (multicast)");
    m->mc_mapped = true;
    if (d.setAccess(m->mc, m->size, &acc, 1) != CUDA_SUCCESS) return fail(FCOO_ERR_CUDA, "cuMemSetAccess (multicast)");
    if (cudaMemset((void*)m->uc, 0, m->size) != cudaSuccess) return fail(FCOO_ERR_CUDA, "zero multicast buffer");
    return FCOO_OK;
  };
  if (failed_somewhere(setup())) return bail(err);
  st = host_barrier(c);  // every rank bound and mapped before anyone writes through mc
  if (st) return bail(st);
  *out = m;
  return FCOO_OK;
}

fcoo_status fcoo_mc_ptr(fcoo_mc_t m, void** local, size_t* bytes) {
  if (!m || !local) return fcoo::fail(FCOO_ERR_ARG, "fcoo_mc_ptr: NULL");
  *local = (void*)m->uc;
  if (bytes) *bytes = m->bytes;
  return FCOO_OK;
}

fcoo_status fcoo_mc_free(fcoo_mc_t m) {
  if (!m) return FCOO_OK;
  cudaDeviceSynchronize();
  fcoo::mc_release(m);
  delete m;
  return FCOO_OK;
}

}  // extern "C"

namespace fcoo {
void mc_views(fcoo_mc_t m, float** uc, float** mc, size_t* bytes, fcoo_comm_t* comm) {
  *uc = reinterpret_cast<float*>(m->uc);
  *mc = reinterpret_cast<float*>(m->mc);
  *bytes = m->bytes;
  *comm = m->comm;
}
}  // namespace fcoo
