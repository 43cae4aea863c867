"""fp64 CPU oracle for the F-COO hot path (arXiv 1705.09905) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with paper_1705_09905_b200/ (the
CUDA product path) and the product path never imports it.  See fcoo_oracle.cpp for
the passage each function follows and the pins that check it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fcoo_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, ERR_ARG, ERR_ORDER, ERR_MODE, ERR_INDEX_RANGE, ERR_DUPLICATE, ERR_EMPTY = range(7)
OP_MTTKRP, OP_TTM = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c++17", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.orc_mode_spec.argtypes = [ci, vp, ci, ci, vp, vp, vp, vp]
        L.orc_storage_bytes.restype = i64
        L.orc_storage_bytes.argtypes = [i64, ci, i64]
        L.orc_build.argtypes = [ci, vp, i64, vp, vp, ci, ci, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_build_ex.argtypes = [ci, vp, i64, vp, vp, ci, ci, i64, ci, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_build_blocked.argtypes = [ci, vp, i64, vp, vp, ci, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                        i64, vp, vp, vp]
        L.orc_build_blocked_ex.argtypes = [ci, vp, i64, vp, vp, ci, ci, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                           vp, i64, vp, vp, vp, vp, vp]
        L.orc_mode_spec_ex.argtypes = [ci, vp, ci, ci, ci, vp, vp, vp, vp]
        L.orc_mttkrp.argtypes = [ci, vp, i64, vp, vp, ci, vp, ci, vp, vp, ci]
        L.orc_ttm.argtypes = [ci, vp, i64, vp, vp, ci, vp, ci, vp, vp, vp, vp]
        L.orc_ttmc.argtypes = [ci, vp, i64, vp, vp, ci, vp, vp, vp, vp]
        L.orc_gram.argtypes = [i64, ci, vp, vp]
        L.orc_pinv_sym.argtypes = [ci, vp, vp]
        L.orc_normalize.argtypes = [i64, ci, vp, vp]
        L.orc_cp_als.argtypes = [ci, vp, i64, vp, vp, ci, ci, ctypes.c_double, vp, vp, vp, vp]
        L.orc_cp_als_mt.argtypes = [ci, vp, i64, vp, vp, ci, ci, ctypes.c_double, vp, vp, vp, vp, ci]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data


def _coo(dims, idx, val):
    d = np.ascontiguousarray(dims, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float32)
    assert idx.ndim == 2 and idx.shape[0] == len(d) and idx.shape[1] == val.shape[0]
    return d, idx, val


def mode_spec(dims, op: int, mode: int, desc: bool = False):
    L = _load()
    d = np.ascontiguousarray(dims, dtype=np.int64)
    im, pm = np.zeros(8, np.int32), np.zeros(8, np.int32)
    ni, npr = ctypes.c_int(0), ctypes.c_int(0)
    rc = L.orc_mode_spec_ex(len(d), _ptr(d), op, mode, int(desc), _ptr(im), ctypes.byref(ni), _ptr(pm),
                            ctypes.byref(npr))
    if rc:
        raise OracleError(rc, "mode_spec")
    return list(im[: ni.value]), list(pm[: npr.value])


def storage_bytes(nnz: int, n_prod: int, T: int) -> int:
    return int(_load().orc_storage_bytes(nnz, n_prod, T))


@dataclass
class Fcoo:
    """Oracle F-COO build result (numpy arrays, exact bytes)."""
    index_modes: list
    product_modes: list
    perm: np.ndarray        # u32[nnz]
    bf: np.ndarray          # u8[ceil(nnz/8)]
    sf: np.ndarray          # u32[ceil(ntiles/32)]
    seg_base: np.ndarray    # u32[ntiles]
    seg_coord: np.ndarray   # u32[nsegs, n_idx]
    pidx: np.ndarray        # u32[n_prod, nnz]
    val: np.ndarray         # f32[nnz]
    nsegs: int
    T: int

    def bf_bits(self) -> np.ndarray:
        return np.unpackbits(self.bf, bitorder="little")[: self.val.shape[0]]


def build_fcoo(dims, idx, val, op: int, mode: int, T: int, desc: bool = False) -> Fcoo:
    L = _load()
    d, idx, val = _coo(dims, idx, val)
    nnz = val.shape[0]
    order = len(d)
    if order < 2 or order > 8:
        raise OracleError(ERR_ORDER, "build")
    im, pm = mode_spec(d, op, mode, desc)
    ntiles = max(1, (nnz + T - 1) // T)
    perm = np.zeros(nnz, np.uint32)
    bf = np.zeros(max(1, (nnz + 7) // 8), np.uint8)
    sf = np.zeros(max(1, (ntiles + 31) // 32), np.uint32)
    seg_base = np.zeros(ntiles, np.uint32)
    seg_coord = np.zeros((max(1, nnz), len(im)), np.uint32)
    pidx = np.zeros((len(pm), nnz), np.uint32)
    pval = np.zeros(nnz, np.float32)
    ns = ctypes.c_int64(0)
    rc = L.orc_build_ex(order, _ptr(d), nnz, _ptr(idx), _ptr(val), op, mode, T, int(desc), _ptr(perm), _ptr(bf), _ptr(sf),
                     _ptr(seg_base), _ptr(seg_coord), _ptr(pidx), _ptr(pval), ctypes.byref(ns))
    if rc:
        raise OracleError(rc, "build")
    nsegs = ns.value
    return Fcoo(im, pm, perm, bf[: (nnz + 7) // 8], sf[: (((nnz + T - 1) // T) + 31) // 32],
                seg_base[: (nnz + T - 1) // T], seg_coord[:nsegs].copy(), pidx, pval, nsegs, T)


@dataclass
class FcooBlocked:
    """Oracle blocked F-COO (orc_build_blocked): stream arrays have nstream positions."""
    index_modes: list
    product_modes: list
    perm: np.ndarray        # u32[nstream], 0xFFFFFFFF at padding
    bf: np.ndarray          # u8[ceil(nstream/8)]
    sf: np.ndarray          # u32[ceil(ntiles/32)]
    seg_base: np.ndarray    # u32[ntiles]
    seg_coord: np.ndarray   # u32[nsegs, n_idx]
    pidx: np.ndarray        # u32[n_prod, nstream] (global product coords, 0 at padding)
    val: np.ndarray         # f32[nstream] (0 at padding)
    pk: np.ndarray          # u32[nstream] packed (outer_local << IB) | last
    blk_start: np.ndarray   # i64[nblocks + 1]
    blk_end: np.ndarray     # i64[nblocks]
    nsegs: int
    nstream: int
    nblocks: int
    T: int
    BR: int
    IB: int
    seg_row: np.ndarray = None   # SpTTM: fibre (output row) of each blocked segment
    nfib: int = 0

    def bf_bits(self) -> np.ndarray:
        return np.unpackbits(self.bf, bitorder="little")[: self.nstream]


def build_fcoo_blocked(dims, idx, val, mode: int, T: int, BR: int, op: int = OP_MTTKRP) -> FcooBlocked:
    L = _load()
    d, idx, val = _coo(dims, idx, val)
    nnz = val.shape[0]
    order = len(d)
    if order < 2 or order > 8:
        raise OracleError(ERR_ORDER, "build_blocked")
    im, pm = mode_spec(d, op, mode)
    nblocks = max(1, (int(d[pm[0]]) + BR - 1) // BR)
    cap = nnz + nblocks * (T - 1)
    ntiles_cap = max(1, cap // T + 1)
    perm = np.zeros(cap, np.uint32)
    bf = np.zeros(max(1, (cap + 7) // 8), np.uint8)
    sf = np.zeros(max(1, (ntiles_cap + 31) // 32), np.uint32)
    seg_base = np.zeros(ntiles_cap, np.uint32)
    seg_coord = np.zeros((max(1, nnz), len(im)), np.uint32)
    pidx = np.zeros(len(pm) * cap, np.uint32)
    pval = np.zeros(cap, np.float32)
    pk = np.zeros(cap, np.uint32)
    bs = np.zeros(nblocks + 1, np.int64)
    be = np.zeros(nblocks, np.int64)
    nsg, nst, nbl, nfb = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    seg_row = np.zeros(max(1, nnz), np.uint32)
    rc = L.orc_build_blocked_ex(order, _ptr(d), nnz, _ptr(idx), _ptr(val), op, mode, T, BR, _ptr(perm), _ptr(bf),
                                _ptr(sf), _ptr(seg_base), _ptr(seg_coord), _ptr(pidx), _ptr(pval), _ptr(pk), _ptr(bs),
                                _ptr(be), cap, ctypes.byref(nsg), ctypes.byref(nst), ctypes.byref(nbl),
                                _ptr(seg_row), ctypes.byref(nfb))
    if rc:
        raise OracleError(rc, "build_blocked")
    ns, ntiles = nst.value, nst.value // T
    IB = 0
    while (1 << IB) < int(d[pm[-1]]):
        IB += 1
    return FcooBlocked(im, pm, perm[:ns].copy(), bf[: (ns + 7) // 8].copy(), sf[: (ntiles + 31) // 32].copy(),
                       seg_base[:ntiles].copy(), seg_coord[: nsg.value].copy(),
                       pidx[: len(pm) * ns].reshape(len(pm), ns).copy(), pval[:ns].copy(), pk[:ns].copy(), bs, be,
                       nsg.value, ns, nbl.value, T, BR, IB if len(pm) >= 2 else 0,
                       seg_row[: nsg.value].copy() if op == OP_TTM else None, nfb.value)


def mttkrp(dims, idx, val, mode: int, factors, R: int | None = None, with_D: bool = True, nthreads: int = 1):
    """Returns (M, D) fp64 I_mode x R (D None if with_D False)."""
    L = _load()
    d, idx, val = _coo(dims, idx, val)
    fs = [np.ascontiguousarray(f, dtype=np.float32) for f in factors]
    R = fs[(mode + 1) % len(d)].shape[1] if R is None else R
    ptrs = (ctypes.c_void_p * len(d))(*[_ptr(f) for f in fs])
    M = np.zeros((int(d[mode]), R), np.float64)
    D = np.zeros_like(M) if with_D else None
    rc = L.orc_mttkrp(len(d), _ptr(d), val.shape[0], _ptr(idx), _ptr(val), mode, ptrs, R, _ptr(M),
                      _ptr(D) if with_D else None, nthreads)
    if rc:
        raise OracleError(rc, "mttkrp")
    return M, D


def ttm(dims, idx, val, mode: int, U):
    """Returns (coords u32[nfib, order-1], Y fp64[nfib, R], D fp64[nfib, R])."""
    L = _load()
    d, idx, val = _coo(dims, idx, val)
    U = np.ascontiguousarray(U, dtype=np.float32)
    R = U.shape[1]
    nnz = val.shape[0]
    cap = max(1, nnz)
    coords = np.zeros((cap, len(d) - 1), np.uint32)
    Y = np.zeros((cap, R), np.float64)
    D = np.zeros((cap, R), np.float64)
    nf = ctypes.c_int64(0)
    rc = L.orc_ttm(len(d), _ptr(d), nnz, _ptr(idx), _ptr(val), mode, _ptr(U), R, ctypes.byref(nf), _ptr(coords),
                   _ptr(Y), _ptr(D))
    if rc:
        raise OracleError(rc, "ttm")
    n = nf.value
    return coords[:n].copy(), Y[:n].copy(), D[:n].copy()


def ttmc(dims, idx, val, mode: int, factors, with_D: bool = True):
    """SpTTMc, Eq.(4): returns (Y, D) fp64 I_mode x prod_{m != mode} R_m (Kronecker of the other
    modes' rows in ascending mode order; factors[mode] may be None)."""
    L = _load()
    d, idx, val = _coo(dims, idx, val)
    order = len(d)
    fs = [np.ascontiguousarray(f, dtype=np.float32) if f is not None else np.zeros((1, 1), np.float32)
          for f in factors]
    ranks = np.array([f.shape[1] for f in fs], np.int32)
    W = int(np.prod([ranks[m] for m in range(order) if m != mode]))
    ptrs = (ctypes.c_void_p * order)(*[_ptr(f) for f in fs])
    Y = np.zeros((int(d[mode]), W), np.float64)
    D = np.zeros_like(Y) if with_D else None
    rc = L.orc_ttmc(order, _ptr(d), val.shape[0], _ptr(idx), _ptr(val), mode, ptrs, _ptr(ranks), _ptr(Y),
                    _ptr(D) if with_D else None)
    if rc:
        raise OracleError(rc, "ttmc")
    return Y, D


def gram(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    G = np.zeros((A.shape[1], A.shape[1]), np.float64)
    _load().orc_gram(A.shape[0], A.shape[1], _ptr(A), _ptr(G))
    return G


def pinv_sym(G):
    G = np.ascontiguousarray(G, dtype=np.float64)
    P = np.zeros_like(G)
    rc = _load().orc_pinv_sym(G.shape[0], _ptr(G), _ptr(P))
    if rc < 0:
        raise OracleError(ERR_ARG, "pinv_sym (not symmetric)")
    return P


def normalize(A):
    A = np.array(A, dtype=np.float64, order="C")
    lam = np.zeros(A.shape[1], np.float64)
    _load().orc_normalize(A.shape[0], A.shape[1], _ptr(A), _ptr(lam))
    return A, lam


def cp_als(dims, idx, val, R: int, iters: int, init, tol: float = 0.0, nthreads: int = 1):
    """Returns (factors fp64 list, lambda fp64[R], fit_trace fp64[iters_done]).  nthreads > 1 splits
    each MTTKRP over host threads (private partials merged in thread order)."""
    L = _load()
    d, idx, val = _coo(dims, idx, val)
    ins = [np.ascontiguousarray(f, dtype=np.float32) for f in init]
    outs = [np.zeros((int(I), R), np.float64) for I in d]
    ip = (ctypes.c_void_p * len(d))(*[_ptr(f) for f in ins])
    op = (ctypes.c_void_p * len(d))(*[_ptr(f) for f in outs])
    lam = np.zeros(R, np.float64)
    trace = np.zeros(iters, np.float64)
    n = L.orc_cp_als_mt(len(d), _ptr(d), val.shape[0], _ptr(idx), _ptr(val), R, iters, tol, ip, op, _ptr(lam),
                        _ptr(trace), int(nthreads))
    if n < 0:
        raise OracleError(-n, "cp_als")
    return outs, lam, trace[:n].copy()
