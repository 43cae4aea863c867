"""Thin ctypes binding over libfcoo.so (include/fcoo.h) — argument marshalling only.

Every step of the path runs in the library's CUDA kernels; PyTorch supplies device memory
(the caching allocator, through fcoo_allocator callbacks), streams and torch.distributed (to
broadcast the NCCL unique id).  There is no CPU fallback: if libfcoo.so is missing or no CUDA
device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCOO_LIB") or os.path.join(_PKG, "libfcoo.so")  # FCOO_LIB: experiment builds

OK = 0
ERR_ARG, ERR_ORDER, ERR_MODE, ERR_INDEX_RANGE, ERR_DUPLICATE, ERR_EMPTY, ERR_KEY_BITS, ERR_RANK, ERR_SHAPE, \
    ERR_ALIGN, ERR_OOM, ERR_CUDA, ERR_NCCL, ERR_NOT_FINITE, ERR_IO = range(1, 16)
OP_MTTKRP, OP_TTM = 0, 1
BUILD_KEEP_PERM = 1
BUILD_PRODUCT_DESC = 2
BUILD_DETERMINISTIC = 4
BUILD_BLOCKED = 8
BUILD_FIBRE_FLAGS = 16


class FcooError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str):
        super().__init__(f"{where}: status {code} ({detail})")
        self.code = code


class _Coo(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int), ("dims", ctypes.POINTER(ctypes.c_int64)), ("nnz", ctypes.c_int64),
                ("idx", ctypes.POINTER(ctypes.c_void_p)), ("val", ctypes.c_void_p)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


class _Allocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", ctypes.c_void_p)]


class _BuildOpts(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int), ("tile_nnz", ctypes.c_int), ("flags", ctypes.c_uint), ("block_rows", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int), ("op", ctypes.c_int), ("mode", ctypes.c_int), ("n_idx", ctypes.c_int),
                ("n_prod", ctypes.c_int), ("idx_modes", ctypes.c_int * 8), ("prod_modes", ctypes.c_int * 8),
                ("dims", ctypes.c_int64 * 8), ("nnz", ctypes.c_int64), ("nsegs", ctypes.c_int64),
                ("ntiles", ctypes.c_int64), ("tile_nnz", ctypes.c_int64), ("dense_rows", ctypes.c_int),
                ("storage_bytes", ctypes.c_int64), ("seg_table_bytes", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("shard", ctypes.c_int), ("nshards", ctypes.c_int),
                ("tile_begin", ctypes.c_int64), ("tile_end", ctypes.c_int64), ("blocked", ctypes.c_int),
                ("block_rows", ctypes.c_int), ("nblocks", ctypes.c_int64), ("nstream", ctypes.c_int64),
                ("pk_shift", ctypes.c_int), ("n_words", ctypes.c_int), ("nfib", ctypes.c_int64),
                ("row_sharded", ctypes.c_int), ("row_rank", ctypes.c_int), ("row_nranks", ctypes.c_int),
                ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64), ("fibre_flags", ctypes.c_int)]


class _HostView(ctypes.Structure):
    _fields_ = [("perm", ctypes.c_void_p), ("bf", ctypes.c_void_p), ("sf", ctypes.c_void_p),
                ("seg_base", ctypes.c_void_p), ("seg_coord", ctypes.c_void_p), ("pidx", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("pk", ctypes.c_void_p), ("blk_start", ctypes.c_void_p),
                ("blk_end", ctypes.c_void_p), ("seg_row", ctypes.c_void_p), ("fib_coord", ctypes.c_void_p),
                ("bf2", ctypes.c_void_p)]


class _CpOpts(ctypes.Structure):
    _fields_ = [("R", ctypes.c_int), ("iters", ctypes.c_int), ("tol", ctypes.c_double), ("tile_nnz", ctypes.c_int),
                ("comm", ctypes.c_void_p), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("seed", ctypes.c_uint64), ("deterministic", ctypes.c_int), ("layout", ctypes.c_int),
                ("dist", ctypes.c_int)]


# The exported symbols (every one declared in include/fcoo.h).
SYMBOLS = ["fcoo_build", "fcoo_build_sharded", "fcoo_mttkrp", "fcoo_ttm", "fcoo_ttmc", "fcoo_info", "fcoo_export", "fcoo_destroy",
           "fcoo_comm_unique_id", "fcoo_comm_init", "fcoo_comm_destroy", "fcoo_allreduce_sum", "fcoo_set_shard",
           "fcoo_mc_alloc", "fcoo_mc_ptr", "fcoo_mc_free", "fcoo_mttkrp_mc",
           "fcoo_shard_range", "cp_als", "fcoo_tns_read", "fcoo_tns_info", "fcoo_tns_copy", "fcoo_tns_destroy",
           "fcoo_tns_write", "fcoo_debug_flip_bit", "fcoo_slice_histogram", "fcoo_row_partition", "fcoo_bucket_rows",
           "fcoo_set_row_shard", "fcoo_build_distributed", "fcoo_status_str", "fcoo_last_error", "fcoo_launch_count"]

_lib = None


def load_library():
    """Load libfcoo.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, ci, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.fcoo_build.argtypes = [ctypes.POINTER(_Coo), ci, ctypes.POINTER(_BuildOpts), ctypes.POINTER(_Allocator), vp,
                             ctypes.POINTER(vp)]
    L.fcoo_build_sharded.argtypes = [ctypes.POINTER(_Coo), ci, ctypes.POINTER(_BuildOpts), vp,
                                     ctypes.POINTER(_Allocator), vp, ctypes.POINTER(vp)]
    L.fcoo_mttkrp.argtypes = [vp, ctypes.POINTER(vp), ci, vp, vp]
    L.fcoo_ttm.argtypes = [vp, vp, ci, vp, vp]
    L.fcoo_ttmc.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(ci), vp, vp]
    L.fcoo_info.argtypes = [vp, ctypes.POINTER(_Info)]
    L.fcoo_export.argtypes = [vp, ctypes.POINTER(_HostView), vp]
    L.fcoo_destroy.argtypes = [vp]
    L.fcoo_debug_flip_bit.argtypes = [vp, ci, i64]
    L.fcoo_comm_unique_id.argtypes = [vp]
    L.fcoo_comm_init.argtypes = [ci, ci, vp, ctypes.POINTER(vp)]
    L.fcoo_comm_destroy.argtypes = [vp]
    L.fcoo_allreduce_sum.argtypes = [vp, vp, ctypes.c_size_t, vp]
    L.fcoo_set_shard.argtypes = [vp, ci, ci, vp]
    L.fcoo_mc_alloc.argtypes = [vp, ctypes.c_size_t, ctypes.POINTER(vp)]
    L.fcoo_mc_ptr.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)]
    L.fcoo_mc_free.argtypes = [vp]
    L.fcoo_mttkrp_mc.argtypes = [vp, ctypes.POINTER(vp), ci, vp, vp]
    L.fcoo_shard_range.argtypes = [i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.cp_als.argtypes = [ctypes.POINTER(_Coo), ctypes.POINTER(_CpOpts), ctypes.POINTER(vp), vp,
                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ci), ctypes.POINTER(_Allocator), vp]
    L.fcoo_tns_read.argtypes = [ctypes.c_char_p, ci, ctypes.POINTER(i64), ctypes.POINTER(vp)]
    L.fcoo_tns_info.argtypes = [vp, ctypes.POINTER(ci), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.fcoo_tns_copy.argtypes = [vp, ctypes.POINTER(vp), vp]
    L.fcoo_tns_destroy.argtypes = [vp]
    L.fcoo_tns_write.argtypes = [ctypes.c_char_p, ci, i64, ctypes.POINTER(vp), vp]
    L.fcoo_slice_histogram.argtypes = [ctypes.POINTER(_Coo), ci, vp, vp]
    L.fcoo_row_partition.argtypes = [vp, i64, ci, vp]
    L.fcoo_bucket_rows.argtypes = [ctypes.POINTER(_Coo), ci, vp, ci, ctypes.POINTER(vp), vp, vp,
                                   ctypes.POINTER(_Allocator), vp]
    L.fcoo_set_row_shard.argtypes = [vp, ci, ci, vp, vp]
    L.fcoo_build_distributed.argtypes = [ctypes.POINTER(_Coo), ci, ctypes.POINTER(_BuildOpts), vp,
                                         ctypes.POINTER(_Allocator), vp, ctypes.POINTER(vp)]
    L.fcoo_status_str.restype = ctypes.c_char_p
    L.fcoo_status_str.argtypes = [ci]
    L.fcoo_last_error.restype = ctypes.c_char_p
    L.fcoo_launch_count.restype = ctypes.c_uint64
    for name in SYMBOLS[:-3]:
        getattr(L, name).restype = ci
    _lib = L
    return L


def _check(rc: int, where: str):
    if rc != OK:
        L = load_library()
        raise FcooError(rc, where, f"{L.fcoo_status_str(rc).decode()}: {L.fcoo_last_error().decode()}")


def launch_count() -> int:
    return int(load_library().fcoo_launch_count())


# ---- torch caching allocator behind fcoo_allocator ----
_live = {}


@_ALLOC_FN
def _torch_alloc(nbytes, stream, ctx):
    try:
        p = torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
        _live[p] = nbytes
        return p
    except Exception:  # surfaces as FCOO_ERR_OOM
        return None


@_FREE_FN
def _torch_free(ptr, nbytes, stream, ctx):
    if ptr:
        _live.pop(ptr, None)
        torch.cuda.caching_allocator_delete(ptr)


_ALLOCATOR = _Allocator(_torch_alloc, _torch_free, None)


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _require_cuda(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def read_tns(path: str, nthreads: int = 0, dims=None):
    """FROSTT .tns text -> (dims, idx (order, nnz) uint32 0-based, val (nnz,) float32) host arrays,
    parsed by the library's native reader (fcoo_tns_read).  Coo.from_numpy uploads them."""
    import numpy as np
    L = load_library()
    t = ctypes.c_void_p()
    ov = None if dims is None else (ctypes.c_int64 * len(dims))(*[int(d) for d in dims])
    _check(L.fcoo_tns_read(os.fsencode(path), int(nthreads), ov, ctypes.byref(t)), "fcoo_tns_read")
    try:
        order, nnz = ctypes.c_int(), ctypes.c_int64()
        d = (ctypes.c_int64 * 8)()
        _check(L.fcoo_tns_info(t, ctypes.byref(order), d, ctypes.byref(nnz)), "fcoo_tns_info")
        idx = np.empty((order.value, nnz.value), np.uint32)
        val = np.empty(nnz.value, np.float32)
        ptrs = (ctypes.c_void_p * order.value)(*[idx[m].ctypes.data for m in range(order.value)])
        _check(L.fcoo_tns_copy(t, ptrs, val.ctypes.data), "fcoo_tns_copy")
        return tuple(int(d[m]) for m in range(order.value)), idx, val
    finally:
        L.fcoo_tns_destroy(t)


def write_tns(path: str, idx, val):
    """Write host arrays (idx (order, nnz) 0-based, val (nnz,)) as 1-based FROSTT text (fcoo_tns_write)."""
    import numpy as np
    L = load_library()
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float32)
    order, nnz = idx.shape
    ptrs = (ctypes.c_void_p * order)(*[idx[m].ctypes.data for m in range(order)])
    _check(L.fcoo_tns_write(os.fsencode(path), order, nnz, ptrs, val.ctypes.data), "fcoo_tns_write")


class Coo:
    """Device COO tensor: idx (order, nnz) int32-viewed-as-uint32 CUDA tensor, val (nnz,) float32."""

    def __init__(self, dims, idx: torch.Tensor, val: torch.Tensor):
        _require_cuda(idx, torch.int32, "idx")
        _require_cuda(val, torch.float32, "val")
        self.dims = [int(d) for d in dims]
        self.idx, self.val = idx, val
        self._dims = (ctypes.c_int64 * len(self.dims))(*self.dims)
        self._ptrs = (ctypes.c_void_p * len(self.dims))(*[idx[m].data_ptr() for m in range(len(self.dims))])
        self.c = _Coo(len(self.dims), self._dims, int(val.shape[0]), self._ptrs, val.data_ptr())

    @property
    def order(self):
        return len(self.dims)

    @property
    def nnz(self):
        return int(self.val.shape[0])

    @staticmethod
    def from_numpy(dims, idx_np, val_np, device=None):
        import numpy as np
        idx = torch.from_numpy(np.ascontiguousarray(idx_np).view(np.int32)).to(device or "cuda")
        val = torch.from_numpy(np.ascontiguousarray(val_np, dtype=np.float32)).to(device or "cuda")
        return Coo(dims, idx, val)


@dataclass
class Info:
    order: int
    op: int
    mode: int
    n_idx: int
    n_prod: int
    idx_modes: list
    prod_modes: list
    dims: list
    nnz: int
    nsegs: int
    ntiles: int
    tile_nnz: int
    dense_rows: bool
    storage_bytes: int
    seg_table_bytes: int
    device_bytes: int
    shard: int
    nshards: int
    tile_begin: int
    tile_end: int
    blocked: bool = False
    block_rows: int = 0
    nblocks: int = 0
    nstream: int = 0
    pk_shift: int = 0
    n_words: int = 0
    nfib: int = 0  # SpTTM: output rows (fibres)
    row_sharded: bool = False
    row_rank: int = 0
    row_nranks: int = 1
    row_begin: int = 0
    row_end: int = 0
    fibre_flags: bool = False


class Fcoo:
    """Owning wrapper of an fcoo_t handle (fcoo_build ... fcoo_destroy)."""

    def __init__(self, handle: int, keep: Coo):
        self.h = ctypes.c_void_p(handle)
        self._coo = keep  # the build borrows the COO only until the build returns; kept for clarity
        self.info = self._info()

    def _info(self) -> Info:
        inf = _Info()
        _check(load_library().fcoo_info(self.h, ctypes.byref(inf)), "fcoo_info")
        o = inf.order
        return Info(o, inf.op, inf.mode, inf.n_idx, inf.n_prod, list(inf.idx_modes[: inf.n_idx]),
                    list(inf.prod_modes[: inf.n_prod]), list(inf.dims[:o]), inf.nnz, inf.nsegs, inf.ntiles,
                    inf.tile_nnz, bool(inf.dense_rows), inf.storage_bytes, inf.seg_table_bytes, inf.device_bytes,
                    inf.shard, inf.nshards, inf.tile_begin, inf.tile_end, bool(inf.blocked), inf.block_rows,
                    inf.nblocks, inf.nstream, inf.pk_shift, inf.n_words, inf.nfib, bool(inf.row_sharded),
                    inf.row_rank, inf.row_nranks, inf.row_begin, inf.row_end, bool(inf.fibre_flags))

    def destroy(self):
        if self.h:
            load_library().fcoo_destroy(self.h)
            self.h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def _flags(keep_perm=False, product_desc=False, deterministic=False, blocked=False) -> int:
    return ((BUILD_KEEP_PERM if keep_perm else 0) | (BUILD_PRODUCT_DESC if product_desc else 0)
            | (BUILD_DETERMINISTIC if deterministic else 0) | (BUILD_BLOCKED if blocked else 0))


def fcoo_build(coo: Coo, mode: int, op: int = OP_MTTKRP, tile_nnz: int = 0, keep_perm: bool = False,
               product_desc: bool = False, stream=None, deterministic: bool = False, blocked: bool = False,
               block_rows: int = 0, fibre_flags: bool = False) -> Fcoo:
    """blocked=True: the blocked F-COO of FCOO_BUILD_BLOCKED (block_rows 0 = the library default).
    fibre_flags=True (MTTKRP, plain): the second flag level, so fcoo_ttm runs SpTTM on the handle's
    last product mode (Fig. 2)."""
    L = load_library()
    opts = _BuildOpts(op, tile_nnz, _flags(keep_perm, product_desc, deterministic, blocked)
                      | (BUILD_FIBRE_FLAGS if fibre_flags else 0), block_rows)
    out = ctypes.c_void_p()
    _check(L.fcoo_build(ctypes.byref(coo.c), mode, ctypes.byref(opts), ctypes.byref(_ALLOCATOR),
                        ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(out)), "fcoo_build")
    return Fcoo(out.value, coo)


def fcoo_build_sharded(coo: Coo, mode: int, comm: "Comm", op: int = OP_MTTKRP, tile_nnz: int = 0,
                       keep_perm: bool = False, stream=None, deterministic: bool = False, blocked: bool = False,
                       block_rows: int = 0) -> Fcoo:
    """fcoo_build + fcoo_set_shard(comm.rank, comm.nranks, comm) in one C call."""
    L = load_library()
    opts = _BuildOpts(op, tile_nnz, _flags(keep_perm, False, deterministic, blocked), block_rows)
    out = ctypes.c_void_p()
    _check(L.fcoo_build_sharded(ctypes.byref(coo.c), mode, ctypes.byref(opts), comm.h, ctypes.byref(_ALLOCATOR),
                                ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(out)), "fcoo_build_sharded")
    return Fcoo(out.value, coo)


def fcoo_slice_histogram(coo: Coo, mode: int, stream=None) -> torch.Tensor:
    """Nonzeros per index-mode row (device int32 tensor holding the u32 counts)."""
    hist = torch.empty(coo.dims[mode], dtype=torch.int32, device=coo.val.device)
    _check(load_library().fcoo_slice_histogram(ctypes.byref(coo.c), mode, ctypes.c_void_p(hist.data_ptr()),
                                               ctypes.c_void_p(_stream_ptr(stream))), "fcoo_slice_histogram")
    return hist


def fcoo_row_partition(hist, nranks: int):
    """Row bounds (numpy int64[nranks + 1]) balancing the nonzeros of a host slice histogram over
    nranks contiguous row ranges (host arithmetic in the library, no device)."""
    import numpy as np
    h = np.ascontiguousarray(hist, dtype=np.uint32)
    bounds = np.zeros(nranks + 1, np.int64)
    _check(load_library().fcoo_row_partition(h.ctypes.data, int(h.shape[0]), int(nranks), bounds.ctypes.data),
           "fcoo_row_partition")
    return bounds


def fcoo_bucket_rows(coo: Coo, mode: int, bounds, stream=None):
    """Nonzeros of coo grouped by destination rank of `bounds` -> (Coo of the grouped nonzeros,
    numpy int64 counts per rank)."""
    import numpy as np
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    nranks = int(b.shape[0]) - 1
    idx = torch.empty_like(coo.idx)
    val = torch.empty_like(coo.val)
    ptrs = (ctypes.c_void_p * coo.order)(*[idx[m].data_ptr() for m in range(coo.order)])
    counts = np.zeros(nranks, np.int64)
    _check(load_library().fcoo_bucket_rows(ctypes.byref(coo.c), mode, b.ctypes.data, nranks, ptrs,
                                           ctypes.c_void_p(val.data_ptr()), counts.ctypes.data,
                                           ctypes.byref(_ALLOCATOR), ctypes.c_void_p(_stream_ptr(stream))),
           "fcoo_bucket_rows")
    return Coo(coo.dims, idx, val), counts


def fcoo_set_row_shard(f: "Fcoo", rank: int, bounds, comm: "Comm" = None):
    """Declare f as holding exactly rows [bounds[rank], bounds[rank+1]) of its mode (owned-rows
    combine over comm in fcoo_mttkrp; comm None: no combine)."""
    import numpy as np
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    _check(load_library().fcoo_set_row_shard(f.h, int(rank), int(b.shape[0]) - 1, b.ctypes.data,
                                             comm.h if comm is not None else None), "fcoo_set_row_shard")
    f.info = f._info()


def fcoo_build_distributed(local: Coo, mode: int, comm: "Comm", tile_nnz: int = 0, blocked: bool = False,
                           block_rows: int = 0, stream=None) -> "Fcoo":
    """Collective: every rank passes its own chunk of the tensor and receives the F-COO of its
    nnz-balanced range of mode rows (histogram, all-reduce, partition, bucket, NCCL exchange, build)."""
    L = load_library()
    opts = _BuildOpts(OP_MTTKRP, tile_nnz, _flags(False, False, False, blocked), block_rows)
    out = ctypes.c_void_p()
    _check(L.fcoo_build_distributed(ctypes.byref(local.c), mode, ctypes.byref(opts), comm.h, ctypes.byref(_ALLOCATOR),
                                    ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(out)), "fcoo_build_distributed")
    return Fcoo(out.value, local)


def _factor_ptrs(f: "Fcoo", factors, R: int, skip_mode: int):
    """Device pointers of `order` factors, each checked to be a contiguous fp32 CUDA (dims[m], R)
    tensor (the C ABI carries no sizes: a wrong shape would read out of bounds)."""
    i = f.info
    if len(factors) != i.order:
        raise ValueError(f"expected {i.order} factors, got {len(factors)}")
    ptrs = []
    for m, U in enumerate(factors):
        if U is None:
            if m != skip_mode:
                raise ValueError(f"factors[{m}] is None")
            ptrs.append(None)
            continue
        _require_cuda(U, torch.float32, f"factors[{m}]")
        if m != skip_mode and tuple(U.shape) != (i.dims[m], R):
            raise ValueError(f"factors[{m}] has shape {tuple(U.shape)}, expected {(i.dims[m], R)}")
        ptrs.append(U.data_ptr())
    return ptrs


def _check_out(out: torch.Tensor, rows: int, cols: int, name: str = "out"):
    _require_cuda(out, torch.float32, name)
    if out.numel() < rows * cols:
        raise ValueError(f"{name} holds {out.numel()} elements, needs {rows} x {cols}")


def fcoo_mttkrp(f: Fcoo, factors, R: int, out: torch.Tensor, stream=None) -> torch.Tensor:
    """factors: list of `order` CUDA fp32 (I_m, R) tensors (entry [mode] may be None)."""
    L = load_library()
    ptrs = _factor_ptrs(f, factors, R, f.info.mode)
    _check_out(out, f.info.dims[f.info.mode], R)
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    _check(L.fcoo_mttkrp(f.h, arr, R, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))),
           "fcoo_mttkrp")
    return out


def fcoo_ttm(f: Fcoo, U: torch.Tensor, R: int, out: torch.Tensor, stream=None) -> torch.Tensor:
    L = load_library()
    _require_cuda(U, torch.float32, "U")
    # an MTTKRP handle with the second flag level runs SpTTM on its last product mode
    m = f.info.mode if f.info.op == OP_TTM else f.info.prod_modes[-1]
    if tuple(U.shape) != (f.info.dims[m], R):
        raise ValueError(f"U has shape {tuple(U.shape)}, expected {(f.info.dims[m], R)}")
    _check_out(out, f.info.nfib, R)
    _check(L.fcoo_ttm(f.h, ctypes.c_void_p(U.data_ptr()), R, ctypes.c_void_p(out.data_ptr()),
                      ctypes.c_void_p(_stream_ptr(stream))), "fcoo_ttm")
    return out


def fcoo_ttmc(f: Fcoo, factors, out: torch.Tensor, stream=None) -> torch.Tensor:
    """SpTTMc (Eq.(4)) on an MTTKRP handle of an order-3 tensor.  factors: list of `order` CUDA fp32
    (I_m, R_m) tensors (entry [mode] may be None); out: (I_mode, prod of the other R_m)."""
    L = load_library()
    i = f.info
    if len(factors) != i.order:
        raise ValueError(f"expected {i.order} factors, got {len(factors)}")
    ptrs, ranks = [], []
    for m, U in enumerate(factors):
        if U is None:
            ptrs.append(None)
            ranks.append(0)
            continue
        _require_cuda(U, torch.float32, f"factors[{m}]")
        if U.dim() != 2 or (m != i.mode and U.shape[0] != i.dims[m]):
            raise ValueError(f"factors[{m}] has shape {tuple(U.shape)}, expected ({i.dims[m]}, R_{m})")
        ptrs.append(U.data_ptr())
        ranks.append(int(U.shape[1]))
    ncol = 1
    for m in range(i.order):
        if m != i.mode:
            ncol *= ranks[m]
    _check_out(out, i.dims[i.mode], ncol)
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    rk = (ctypes.c_int * len(ranks))(*ranks)
    _check(L.fcoo_ttmc(f.h, arr, rk, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stream))),
           "fcoo_ttmc")
    return out


def fcoo_debug_flip_bit(f: Fcoo, which: str, bit: int):
    """TEST SUPPORT: flip one bit of the handle's device bf ("bf") or sf ("sf") array."""
    _check(load_library().fcoo_debug_flip_bit(f.h, {"bf": 0, "sf": 1}[which], int(bit)), "fcoo_debug_flip_bit")


def fcoo_export(f: Fcoo, perm: bool = False, stream=None) -> dict:
    """Host copies of the handle's arrays (stream length = info.nstream: nnz, or nnz + padding on a
    blocked handle, whose export also has the packed words "pk" and the block tables)."""
    import numpy as np
    i = f.info
    ns = i.nstream
    d = {
        "bf": np.zeros((ns + 7) // 8, np.uint8),
        "sf": np.zeros((i.ntiles + 31) // 32, np.uint32),
        "seg_base": np.zeros(i.ntiles, np.uint32),
        "seg_coord": np.zeros((i.nsegs, i.n_idx), np.uint32),
        "pidx": np.zeros((i.n_prod, ns), np.uint32),
        "val": np.zeros(ns, np.float32),
    }
    if i.blocked:
        d["pk"] = np.zeros((i.n_words, ns), np.uint32)
        d["blk_start"] = np.zeros(i.nblocks + 1, np.int64)
        d["blk_end"] = np.zeros(i.nblocks, np.int64)
        if i.op == OP_TTM:
            d["seg_row"] = np.zeros(i.nsegs, np.uint32)
    if i.op == OP_TTM:
        d["fib_coord"] = np.zeros((i.nfib, i.n_idx), np.uint32)
    elif i.fibre_flags:
        d["fib_coord"] = np.zeros((i.nfib, i.order - 1), np.uint32)
        d["bf2"] = np.zeros((ns + 7) // 8, np.uint8)
    if perm:
        d["perm"] = np.zeros(ns, np.uint32)
    v = _HostView(*(d[k].ctypes.data if k in d else None
                    for k in ("perm", "bf", "sf", "seg_base", "seg_coord", "pidx", "val", "pk", "blk_start",
                              "blk_end", "seg_row", "fib_coord", "bf2")))
    _check(load_library().fcoo_export(f.h, ctypes.byref(v), ctypes.c_void_p(_stream_ptr(stream))), "fcoo_export")
    return d


class Comm:
    def __init__(self, handle: int, rank: int, nranks: int):
        self.h = ctypes.c_void_p(handle)
        self.rank, self.nranks = rank, nranks

    def destroy(self):
        if self.h:
            load_library().fcoo_comm_destroy(self.h)
            self.h = ctypes.c_void_p(None)


def fcoo_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().fcoo_comm_unique_id(buf), "fcoo_comm_unique_id")
    return buf.raw


def fcoo_comm_init(rank: int, nranks: int, uid: bytes) -> Comm:
    out = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(load_library().fcoo_comm_init(rank, nranks, buf, ctypes.byref(out)), "fcoo_comm_init")
    return Comm(out.value, rank, nranks)


def comm_from_process_group(group=None) -> Comm:
    """NCCL communicator of the library, unique id broadcast over torch.distributed."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [fcoo_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return fcoo_comm_init(rank, world, obj[0])


def fcoo_allreduce_sum(comm: Comm, buf: torch.Tensor, stream=None):
    _require_cuda(buf, torch.float32, "buf")
    _check(load_library().fcoo_allreduce_sum(comm.h, ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                             ctypes.c_void_p(_stream_ptr(stream))), "fcoo_allreduce_sum")


def fcoo_shard_range(ntiles: int, shard: int, nshards: int):
    """Tile range [begin, end) of shard `shard` (host arithmetic in the library, no device)."""
    b, e = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(load_library().fcoo_shard_range(ntiles, shard, nshards, ctypes.byref(b), ctypes.byref(e)),
           "fcoo_shard_range")
    return b.value, e.value


def fcoo_set_shard(f: Fcoo, shard: int, nshards: int, comm: Comm | None = None):
    _check(load_library().fcoo_set_shard(f.h, shard, nshards, comm.h if comm else None), "fcoo_set_shard")
    f.info = f._info()


class McBuffer:
    """Output buffer bound to an NVLS multicast object across the ranks of a Comm (fcoo_mc_alloc).
    `local` is this rank's copy as a CUDA fp32 tensor of `numel` elements (a view, not owning)."""

    def __init__(self, comm: "Comm", numel: int):
        L = load_library()
        out = ctypes.c_void_p()
        _check(L.fcoo_mc_alloc(comm.h, ctypes.c_size_t(4 * numel), ctypes.byref(out)), "fcoo_mc_alloc")
        self.h = out
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(L.fcoo_mc_ptr(self.h, ctypes.byref(p), ctypes.byref(n)), "fcoo_mc_ptr")
        self.numel = numel
        self.ptr = p.value
        self.local = _tensor_view(p.value, numel)

    def free(self):
        if self.h:
            load_library().fcoo_mc_free(self.h)
            self.h = ctypes.c_void_p(None)
            self.local = None


def _tensor_view(ptr: int, numel: int) -> torch.Tensor:
    """Non-owning CUDA fp32 tensor over device memory the library owns (via __cuda_array_interface__)."""
    class _A:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_A(), device="cuda")


def fcoo_mttkrp_mc(f: Fcoo, factors, R: int, out: McBuffer, stream=None) -> torch.Tensor:
    """SpMTTKRP with the cross-rank combine fused into the epilogue; returns out.local[:I_n*R] as (I_n, R)."""
    L = load_library()
    ptrs = _factor_ptrs(f, factors, R, f.info.mode)
    if out.numel < f.info.dims[f.info.mode] * R:
        raise ValueError(f"multicast buffer holds {out.numel} floats, output needs {f.info.dims[f.info.mode] * R}")
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    _check(L.fcoo_mttkrp_mc(f.h, arr, R, out.h, ctypes.c_void_p(_stream_ptr(stream))), "fcoo_mttkrp_mc")
    I = f.info.dims[f.info.mode]
    return out.local[: I * R].view(I, R)


def cp_als(coo: Coo, R: int, iters: int, factors, tol: float = 0.0, tile_nnz: int = 0, comm: Comm | None = None,
           stream=None, seed: int = 0, deterministic: bool = False, layout: str = "auto", dist: bool = False):
    """In-place CP-ALS: `factors` (list of CUDA fp32 (I_m, R)) hold the initial factors (or, with
    seed != 0, are seeded on the device by the library) and receive the result.  layout "auto": the
    blocked F-COO where the build allows it; "fcoo": the plain F-COO for every mode.  dist=True (with
    a comm): `coo` is this rank's chunk of the nonzeros and every mode runs on row shards
    (fcoo_build_distributed, owned-rows all-gather).  Returns (lambda CUDA fp32 (R,), fit_trace list)."""
    import numpy as np
    L = load_library()
    if len(factors) != coo.order:
        raise ValueError(f"expected {coo.order} factors, got {len(factors)}")
    for m, U in enumerate(factors):
        _require_cuda(U, torch.float32, f"factors[{m}]")
        if tuple(U.shape) != (coo.dims[m], R):
            raise ValueError(f"factors[{m}] has shape {tuple(U.shape)}, expected {(coo.dims[m], R)}")
    lam = torch.empty(R, dtype=torch.float32, device=factors[0].device)
    trace = np.zeros(iters, np.float64)
    done = ctypes.c_int(0)
    opts = _CpOpts(R, iters, tol, tile_nnz, comm.h if comm else None, comm.rank if comm else 0,
                   comm.nranks if comm else 1, seed, 1 if deterministic else 0, 1 if layout == "fcoo" else 0,
                   1 if dist else 0)
    arr = (ctypes.c_void_p * len(factors))(*[U.data_ptr() for U in factors])
    _check(L.cp_als(ctypes.byref(coo.c), ctypes.byref(opts), arr, ctypes.c_void_p(lam.data_ptr()),
                    trace.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(done),
                    ctypes.byref(_ALLOCATOR), ctypes.c_void_p(_stream_ptr(stream))), "cp_als")
    return lam, list(trace[: done.value])
