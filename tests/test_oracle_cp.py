"""Pins for the oracle CP-ALS (Algorithm 1): helper hand
cases, Penrose conditions, exact recovery of known low-rank tensors, monotone fit, and the
fit identity against a dense reconstruction."""
import numpy as np
import pytest

import gen
import oracle
from dense_defs import dense_from_coo, kruskal_dense


def test_helper_hand_cases(golden):
    c = golden["cp"]
    assert np.array_equal(oracle.gram(np.array(c["gram"]["A"], float)), np.array(c["gram"]["G"], float))
    assert np.allclose(oracle.pinv_sym(np.array(c["pinv"]["G"], float)), np.array(c["pinv"]["P"]), atol=1e-15)
    A, lam = oracle.normalize(np.array(c["normalize"]["A"], float))
    assert np.allclose(A, c["normalize"]["out"], rtol=1e-15) and np.allclose(lam, c["normalize"]["lambda"])
    A, lam = oracle.normalize(np.zeros((3, 2)))
    assert np.array_equal(A, np.zeros((3, 2))) and np.array_equal(lam, [0, 0])
    assert np.allclose(oracle.pinv_sym(np.eye(4)), np.eye(4), atol=1e-15)


@pytest.mark.parametrize("rank", [6, 4, 1])
def test_pinv_penrose(rank):
    """The four Penrose conditions for SPD (rank 6) and PSD rank-deficient inputs."""
    B = gen.uniform((6, rank), 7, rank, signed=True).astype(np.float64)
    G = B @ B.T
    P = oracle.pinv_sym(G)
    n = np.linalg.norm(G)
    assert np.linalg.norm(G @ P @ G - G) <= 1e-9 * n
    assert np.linalg.norm(P @ G @ P - P) <= 1e-9 * max(1.0, np.linalg.norm(P))
    assert np.linalg.norm((G @ P).T - G @ P) <= 1e-9
    assert np.linalg.norm((P @ G).T - P @ G) <= 1e-9


def _dense_coo(dims):
    return np.array(list(np.ndindex(*dims)), np.uint32).T.copy()


def _init(dims, R, seed):
    return gen.factors(dims, R, seed)


@pytest.mark.parametrize("dims,R", [((30, 20, 10), 5), ((12, 10, 8, 6), 4)])
def test_recovery_dense(dims, R):
    A = [gen.uniform((d, R), 300 + m, 1, signed=True) for m, d in enumerate(dims)]
    lam = np.linspace(1.0, 2.0, R)
    cells = _dense_coo(dims)
    val = gen.kruskal_coo(A, lam, cells)
    _, _, trace = oracle.cp_als(dims, cells, val, R, 200, _init(dims, R, 301), tol=1e-10)
    assert trace[-1] >= 0.999


def test_recovery_sparse_support():
    """Rank-8 tensor whose factor columns each have 20 random nonzero rows: the tensor is
    sparse (union of 8 blocks of 20^3 cells, many empty slices) and exactly low-rank.
    (With signed factor entries ALS from a positive start stalls in a local minimum near
    fit 0.805 for this support pattern — an ALS property, not an oracle error; the
    non-negative model is recovered from every seed tried.)"""
    dims, R, s = (200, 150, 100), 8, 20
    A, sup = [], []
    for m, d in enumerate(dims):
        U = np.zeros((d, R), np.float32)
        S = []
        for r in range(R):
            rows = np.argsort(gen.uniform((d,), 400 + m, r))[:s]
            U[rows, r] = gen.uniform((s,), 410 + m, r) + 0.5  # entries in [0.5, 1.5)
            S.append(rows)
        A.append(U)
        sup.append(S)
    cells = set()
    for r in range(R):
        for i in sup[0][r]:
            for j in sup[1][r]:
                for k in sup[2][r]:
                    cells.add((int(i), int(j), int(k)))
    coords = np.array(sorted(cells), np.uint32).T.copy()
    val = gen.kruskal_coo(A, np.ones(R), coords)
    _, _, trace = oracle.cp_als(dims, coords, val, R, 200, _init(dims, R, 401), tol=1e-10)
    assert trace[-1] >= 0.999


def test_recovery_rank1():
    dims = (6, 5, 4)
    A = [gen.uniform((d, 1), 500 + m, 0) + 0.5 for m, d in enumerate(dims)]
    cells = _dense_coo(dims)
    val = gen.kruskal_coo(A, [1.0], cells)
    _, _, trace = oracle.cp_als(dims, cells, val, 1, 25, _init(dims, 1, 501))
    assert trace[-1] >= 0.999


def test_monotone_fit_and_identity():
    """ALS never increases the residual: the fit trace is non-decreasing; and the
    identity-based fit equals 1 - ||X - Xhat|| / ||X|| from a dense reconstruction."""
    dims = (9, 8, 7)
    idx, val = gen.coo(dims, 200, None, 601)
    R = 4
    facs, lam, trace = oracle.cp_als(dims, idx, val, R, 30, _init(dims, R, 602))
    assert np.all(np.diff(trace) >= -1e-7)
    X = dense_from_coo(dims, idx, val)
    Xh = kruskal_dense(lam, facs)
    fit = 1 - np.linalg.norm(X - Xh) / np.linalg.norm(X)
    assert abs(fit - trace[-1]) <= 1e-9
    # columns are unit norm, lambda non-negative
    for U in facs:
        assert np.allclose(np.linalg.norm(U, axis=0), 1.0, atol=1e-12)
    assert np.all(lam >= 0)


def test_rank_above_extent():
    """Q15 / P:L564: R larger than a mode extent gives a deficient V; pinv handles it."""
    dims = (10, 9, 3)
    idx, val = gen.coo(dims, 120, None, 701)
    _, _, trace = oracle.cp_als(dims, idx, val, 5, 10, _init(dims, 5, 702))
    assert np.all(np.isfinite(trace)) and np.all(np.diff(trace) >= -1e-7)


def test_threads_agree():
    """The multi-threaded CP oracle (private per-thread MTTKRP partials merged in thread order, used
    at configuration-5 scale) computes the same iteration as the single-threaded one up to rounding
    order: fit traces within 1e-12, factors and lambda within 1e-9 relative."""
    dims = (60, 50, 40, 30)
    idx, val = gen.coo(dims, 20000, (0.5, 0.5, 0.5, 0.5), 61)
    R = 8
    init = gen.factors(dims, R, 62)
    f1, l1, t1 = oracle.cp_als(dims, idx, val, R, 4, init, nthreads=1)
    f4, l4, t4 = oracle.cp_als(dims, idx, val, R, 4, init, nthreads=4)
    assert np.allclose(t1, t4, rtol=0, atol=1e-12)
    assert np.allclose(l1, l4, rtol=1e-9, atol=0)
    for a, b in zip(f1, f4):
        assert np.allclose(a, b, rtol=1e-9, atol=1e-12)
