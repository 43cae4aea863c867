"""Seeded synthetic input generator (shared by the oracle and the CUDA path).

This module holds none of the method's arithmetic (no sort keys, flags,
MTTKRP/TTM/CP maths): it draws coordinates, values and dense factor entries
from a counter-based generator (see tensorgen.c for the recipe) plus the
paper-shaped workload table used by tests and bench.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tensorgen.c")
_LIB = os.path.join(_HERE, "libtensorgen.so")
_lib = None


def build(force: bool = False) -> str:
    deps = [_SRC, os.path.join(os.path.dirname(_SRC), "tensorgen_dedup.h")]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(d) for d in deps):
        # -mcx16: lock-free 16-byte compare-and-swap for the 128-bit tuple table
        subprocess.check_call(["gcc", "-O2", "-mcx16", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.tg_coo.restype = ctypes.c_int
        lib.tg_coo.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_uint64,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.tg_uniform_f32.restype = None
        lib.tg_uniform_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_void_p]
        lib.tg_hash.restype = ctypes.c_uint64
        lib.tg_hash.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = lib
    return _lib


def coo(dims, nnz: int, alpha=None, seed: int = 1):
    """Duplicate-free synthetic COO tensor in draw order.

    Returns (idx, val): idx is uint32 (order, nnz) C-contiguous (SoA), val float32 (nnz,).
    """
    lib = _load()
    order = len(dims)
    d = np.asarray(dims, dtype=np.int64)
    a = np.asarray(alpha if alpha is not None else [0.0] * order, dtype=np.float64)
    idx = np.empty((order, nnz), dtype=np.uint32)
    val = np.empty((nnz,), dtype=np.float32)
    draws = ctypes.c_int64(0)
    rc = lib.tg_coo(order, d.ctypes.data, nnz, a.ctypes.data, seed, idx.ctypes.data, val.ctypes.data,
                    ctypes.byref(draws))
    if rc != 0:
        raise ValueError(f"tensorgen.tg_coo failed rc={rc} dims={list(dims)} nnz={nnz}")
    return idx, val


def uniform(shape, seed: int, stream: int = 0, signed: bool = False) -> np.ndarray:
    """Counter-based uniform fp32 entries in [0,1) (or [-1,1) if signed), 24-bit exact."""
    lib = _load()
    out = np.empty(shape, dtype=np.float32)
    lib.tg_uniform_f32(seed, stream, 0, out.size, 1 if signed else 0, out.ctypes.data)
    return out


def factors(dims, R: int, seed: int, signed: bool = False):
    """One I_m x R row-major fp32 factor matrix per mode (stream = 1000 + m)."""
    return [uniform((int(I), R), seed, 1000 + m, signed) for m, I in enumerate(dims)]


def hash64(seed: int, stream: int, ctr: int) -> int:
    return int(_load().tg_hash(seed, stream, ctr))


def kruskal_coo(factors_list, lam, coords):
    """Values of a known Kruskal model sum_r lam_r prod_m U_m(i_m, r) at given coordinates.

    Test-data synthesis for the CP recovery inputs (the model the tensor is drawn
    from), evaluated in fp64 and rounded once to fp32.  coords: (order, nnz) uint32.
    """
    acc = np.zeros((coords.shape[1], len(lam)), dtype=np.float64)
    acc[:] = np.asarray(lam, dtype=np.float64)[None, :]
    for m, U in enumerate(factors_list):
        acc *= np.asarray(U, dtype=np.float64)[coords[m].astype(np.int64)]
    return acc.sum(axis=1).astype(np.float32)


@dataclass(frozen=True)
class Workload:
    name: str
    dims: tuple
    nnz: int
    alpha: tuple
    seed: int


# SURVEY.md §8(d) table; shapes follow PAPER.md Table IV (L406-419) and BASELINE.json configs.
WORKLOADS = {
    "tiny": Workload("tiny", (50, 40, 30), 1000, (0.0, 0.0, 0.0), 101),
    "nell2": Workload("nell2", (12092, 9184, 28818), 76879419, (0.5, 0.5, 0.5), 102),
    "netflix": Workload("netflix", (480189, 17770, 2182), 100480507, (0.5, 0.5, 0.2), 103),
    "brainq": Workload("brainq", (60, 70000, 9), 11000000, (0.0, 0.0, 0.0), 104),
    "order4": Workload("order4", (500000, 20000, 2000, 1000), 150000000, (0.5, 0.5, 0.5, 0.5), 105),
    # SURVEY §8(d) "stress variant": heavy power law, one slice of ~7M nonzeros (reading Q16)
    "netflix_stress": Workload("netflix_stress", (480189, 17770, 2182), 100480507, (1.0, 1.0, 0.5), 106),
    # Table IV's two large tensors (FROSTT extents): 67- and 69-bit sort keys, so the
    # device build takes the 128-bit key path
    "delicious": Workload("delicious", (532924, 17262471, 2480308), 140126181, (0.5, 0.5, 0.5), 107),
    "nell1": Workload("nell1", (2902330, 2143368, 25495389), 143599552, (0.5, 0.5, 0.5), 108),
}


def workload(name: str, nnz: int | None = None):
    w = WORKLOADS[name]
    idx, val = coo(w.dims, nnz if nnz is not None else w.nnz, w.alpha, w.seed)
    return w, idx, val


def planted_sparse(dims, R: int, s: int, seed: int, disjoint_mode: int = 0):
    """Test-data synthesis (no method arithmetic): a rank-R tensor with sparse-support factors,
    X = sum_r lam_r U_0(:,r) o U_1(:,r) o ... (SURVEY §8(c) c4 "exact recovery" family at
    configuration-5 shape).  Column r of mode m is nonzero on s distinct rows, values in [0.5, 1.5);
    in `disjoint_mode` the supports of different columns are disjoint (needs R*s <= dims[mode]), so
    every stored cell belongs to exactly one rank-1 term and its value is that term's product,
    evaluated in fp64 and rounded once to fp32.  nnz = R * s**order.
    Returns (idx (order, nnz) uint32, val fp32, factors fp64 list, lam fp64)."""
    rng = np.random.default_rng(seed)
    order = len(dims)
    assert R * s <= dims[disjoint_mode]
    lam = 1.0 + rng.random(R)
    facs = [np.zeros((int(I), R)) for I in dims]
    sup = [[None] * R for _ in range(order)]
    for m, I in enumerate(dims):
        dis = rng.permutation(int(I))[: R * s] if m == disjoint_mode else None
        for r in range(R):
            rows = np.sort(dis[r * s:(r + 1) * s]) if m == disjoint_mode else np.sort(rng.choice(int(I), s, replace=False))
            sup[m][r] = rows
            facs[m][rows, r] = 0.5 + rng.random(s)
    n_term = s ** order
    idx = np.empty((order, R * n_term), np.uint32)
    val = np.empty(R * n_term, np.float32)
    for r in range(R):
        grids = np.meshgrid(*[sup[m][r] for m in range(order)], indexing="ij")
        prod = np.full(grids[0].shape, lam[r])
        for m in range(order):
            prod = prod * facs[m][grids[m], r]
        for m in range(order):
            idx[m, r * n_term:(r + 1) * n_term] = grids[m].ravel()
        val[r * n_term:(r + 1) * n_term] = prod.ravel().astype(np.float32)
    return idx, val, facs, lam
