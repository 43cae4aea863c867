"""Pins for the oracle SpMTTKRP and SpTTM: hand cases, dense
unfolding x explicit Khatri-Rao (Eq.(5)), the CP-loss gradient, the Kruskal closed form,
inner-product and slice-sum invariants, dense TTM and the Fig. 3 equivalence."""
import numpy as np
import pytest

import gen
import oracle
from dense_defs import (dense_from_coo, kronecker, khatri_rao, kruskal_dense, mttkrp_dense, ttm_dense, unfold)


# ---- the textbook helpers themselves are pinned to the worked cases first ----

def test_helpers_match_worked_cases(golden):
    kr = golden["khatri_rao"]
    assert np.array_equal(khatri_rao(np.array(kr["A"], float), np.array(kr["B"], float)), np.array(kr["out"]))
    kc = golden["kronecker"]
    assert np.array_equal(kronecker(np.array(kc["A"], float), np.array(kc["B"], float)), np.array(kc["out"]))
    m0, m1 = golden["matricize"]
    X = np.zeros(m0["dims"])
    for i, j, k in np.ndindex(*m0["dims"]):
        X[i, j, k] = 1 + i + 2 * j + 4 * k
    assert np.array_equal(unfold(X, 0), np.array(m0["rows"]))
    X = np.zeros(m1["dims"])
    X[tuple(m1["coord"])] = 1
    assert np.argmax(unfold(X, 0)[0]) == m1["col"]


# ---- MTTKRP ----

def test_mttkrp_hand_cases(golden):
    for case in golden["mttkrp"]:
        dims = case["dims"]
        if case.get("dense_ones"):
            cells = np.array(list(np.ndindex(*dims)), np.uint32).T.copy()
            idx, val = cells, np.ones(cells.shape[1], np.float32)
        else:
            idx = np.array(case["coords"], np.uint32).T.copy()
            val = np.array(case["vals"], np.float32)
        fs = [np.array(f, np.float32) for f in case["factors"]]
        M, D = oracle.mttkrp(dims, idx, val, case["mode"], fs)
        assert np.array_equal(M, np.array(case["M"], float)), case["cite"]


@pytest.mark.parametrize("dims", [(8, 7, 6), (5, 4, 3, 3), (6, 9)])
def test_mttkrp_vs_unfold_khatri_rao(dims):
    """Eq.(5): M = X_(n) (KR of the other factors), for every mode; also pins Q8/Q9."""
    nnz = int(np.prod(dims) * 0.4)
    idx, val = gen.coo(dims, nnz, None, 21)
    R = 5
    fs = gen.factors(dims, R, 22, signed=True)
    X = dense_from_coo(dims, idx, val)
    for n in range(len(dims)):
        M, _ = oracle.mttkrp(dims, idx, val, n, fs)
        ref = mttkrp_dense(X, fs, n)
        assert np.allclose(M, ref, rtol=1e-12, atol=1e-12)


def test_mttkrp_is_cp_gradient_term():
    """grad_{U_n} 1/2 ||X - [[U]]||^2 = U_n (Hadamard_{m!=n} U_m^T U_m) - M_n; the loss is
    quadratic in U_n so central differences are exact up to rounding."""
    dims = (5, 4, 3)
    R = 3
    idx, val = gen.coo(dims, 30, None, 31)
    X = dense_from_coo(dims, idx, val)
    fs = [f.astype(np.float64) for f in gen.factors(dims, R, 32, signed=True)]

    def loss(factors):
        return 0.5 * np.sum((X - kruskal_dense(np.ones(R), factors)) ** 2)

    for n in range(3):
        M, _ = oracle.mttkrp(dims, idx, val, n, [f.astype(np.float32) for f in fs])
        # factors given to the oracle are fp32-rounded; use those exact values in the loss too
        f32 = [f.astype(np.float32).astype(np.float64) for f in fs]
        V = np.ones((R, R))
        for m in range(3):
            if m != n:
                V *= f32[m].T @ f32[m]
        grad = f32[n] @ V - M
        h = 1e-3
        num = np.zeros_like(grad)
        for i in range(dims[n]):
            for r in range(R):
                up = [f.copy() for f in f32]
                dn = [f.copy() for f in f32]
                up[n][i, r] += h
                dn[n][i, r] -= h
                num[i, r] = (loss(up) - loss(dn)) / (2 * h)
        assert np.allclose(grad, num, rtol=1e-7, atol=1e-9)


def test_mttkrp_kruskal_closed_form():
    """X = [[lam; A_1..A_N]] stored densely: MTTKRP_n(V) = A_n diag(lam) Hadamard_{m!=n}(A_m^T V_m)."""
    for dims, Rx, R in (((6, 5, 4), 2, 3), ((4, 3, 3, 2), 2, 2)):
        A = [gen.uniform((d, Rx), 40 + m, 0, signed=True).astype(np.float64) for m, d in enumerate(dims)]
        lam = np.array([1.5, 0.75])
        cells = np.array(list(np.ndindex(*dims)), np.uint32).T.copy()
        val = gen.kruskal_coo(A, lam, cells)  # fp32-rounded values of the model
        Vs = gen.factors(dims, R, 41, signed=True)
        for n in range(len(dims)):
            M, _ = oracle.mttkrp(dims, cells, val, n, Vs)
            H = np.ones((Rx, R))
            Habs = np.ones((Rx, R))
            for m in range(len(dims)):
                if m != n:
                    H *= A[m].T @ Vs[m].astype(np.float64)
                    Habs *= np.abs(A[m]).T @ np.abs(Vs[m].astype(np.float64))
            ref = A[n] @ np.diag(lam) @ H
            # values carry one fp32 rounding each: relative 2^-24 per term
            scale = np.abs(A[n]) @ np.diag(lam) @ Habs + 1e-30
            assert np.all(np.abs(M - ref) <= 1e-6 * scale + 1e-12)


def test_mttkrp_inner_product_invariant():
    """<M_n, U_n>_F = <X, [[U]]> = sum_q v_q sum_r prod_m U_m(i_m, r), the same for every n."""
    dims = (30, 20, 25, 7)
    idx, val = gen.coo(dims, 3000, (0.5, 0.5, 0.5, 0.0), 51)
    fs = gen.factors(dims, 8, 52, signed=True)
    direct = 0.0
    prod = np.ones((val.shape[0], 8))
    for m in range(4):
        prod *= fs[m].astype(np.float64)[idx[m]]
    direct = float(np.sum(val.astype(np.float64)[:, None] * prod))
    for n in range(4):
        M, _ = oracle.mttkrp(dims, idx, val, n, fs)
        assert abs(np.sum(M * fs[n]) - direct) <= 1e-10 * np.sum(np.abs(val[:, None] * prod))


def test_mttkrp_slice_sums_and_normaliser():
    dims = (13, 11, 9)
    idx, val = gen.coo(dims, 400, None, 61)
    ones = [np.ones((d, 1), np.float32) for d in dims]
    for n in range(3):
        M, D = oracle.mttkrp(dims, idx, val, n, ones)
        ref = np.bincount(idx[n], weights=val.astype(np.float64), minlength=dims[n])
        assert np.allclose(M[:, 0], ref, rtol=1e-14)
        assert np.array_equal(M, D)  # all contributions positive
    fs = gen.factors(dims, 4, 62, signed=True)
    M, D = oracle.mttkrp(dims, idx, val, 1, fs)
    assert np.all(D >= np.abs(M) - 1e-15)


def test_mttkrp_threads_agree():
    dims = (40, 30, 20)
    idx, val = gen.coo(dims, 5000, (0.5, 0.5, 0.5), 71)
    fs = gen.factors(dims, 16, 72)
    M1, D1 = oracle.mttkrp(dims, idx, val, 0, fs, nthreads=1)
    M4, D4 = oracle.mttkrp(dims, idx, val, 0, fs, nthreads=4)
    assert np.allclose(M1, M4, rtol=1e-13, atol=0)
    assert np.allclose(D1, D4, rtol=1e-13, atol=0)


def test_mttkrp_errors():
    with pytest.raises(oracle.OracleError):
        oracle.mttkrp((3, 3, 3), np.array([[0], [0], [3]], np.uint32), np.ones(1, np.float32), 0,
                      [np.ones((3, 2), np.float32)] * 3)


# ---- TTM ----

def test_ttm_hand_cases(golden):
    for case in golden["ttm"]:
        idx = np.array(case["coords"], np.uint32).T.copy()
        coords, Y, D = oracle.ttm(case["dims"], idx, np.array(case["vals"], np.float32), case["mode"],
                                  np.array(case["U"], np.float32))
        assert coords.tolist() == case["fibers"], case["cite"]
        assert np.array_equal(Y, np.array(case["Y"], float)), case["cite"]


@pytest.mark.parametrize("dims", [(7, 6, 5), (4, 5, 3, 3)])
def test_ttm_vs_dense(dims):
    idx, val = gen.coo(dims, int(np.prod(dims) * 0.3), None, 81)
    X = dense_from_coo(dims, idx, val)
    for n in range(len(dims)):
        U = gen.uniform((dims[n], 4), 82, n, signed=True)
        coords, Y, D = oracle.ttm(dims, idx, val, n, U)
        Yd = ttm_dense(X, U, n)
        others = [m for m in range(len(dims)) if m != n]
        nonempty = sorted({tuple(int(idx[m][q]) for m in others) for q in range(val.shape[0])})
        assert [tuple(c) for c in coords.tolist()] == nonempty  # lexicographic fibre order
        for f, c in enumerate(nonempty):
            assert np.allclose(Y[f], Yd[c], rtol=1e-12, atol=1e-13)


def test_fig3_ttm_then_hadamard_equals_mttkrp():
    """Fig. 3: TTM along mode k with C, then the fibre-wise Hadamard with B
    reduced over j, equals the one-shot MTTKRP on mode i."""
    dims = (9, 8, 7)
    idx, val = gen.coo(dims, 150, None, 91)
    fs = gen.factors(dims, 6, 92, signed=True)
    coords, Y, _ = oracle.ttm(dims, idx, val, 2, fs[2])  # Y(i,j,:) = sum_k X(i,j,k) C(k,:)
    M2 = np.zeros((dims[0], 6))
    for f, (i, j) in enumerate(coords.tolist()):
        M2[i] += Y[f] * fs[1][j].astype(np.float64)
    M, _ = oracle.mttkrp(dims, idx, val, 0, fs)
    assert np.allclose(M, M2, rtol=1e-12, atol=1e-13)


def test_segmented_scan_reading(golden):
    """S:L258 segmented scan semantics = the per-segment running sum of a build:
    with R=1 and unit factors the MTTKRP segment totals are the last scan value per segment."""
    c = golden["segmented_scan"]
    vals, heads = c["values"], c["heads"]
    out, acc = [], 0
    for v, h in zip(vals, heads):
        acc = v if h else acc + v
        out.append(acc)
    assert out == c["out"]
    # the same totals from the oracle: segments [0,1,2] and [3,4] as two slices
    idx = np.array([[0, 0, 0, 1, 1], [0, 1, 2, 0, 1], [0, 0, 0, 0, 0]], np.uint32)
    M, _ = oracle.mttkrp((2, 3, 1), idx, np.array(vals, np.float32), 0,
                         [np.ones((2, 1), np.float32), np.ones((3, 1), np.float32), np.ones((1, 1), np.float32)])
    assert M[:, 0].tolist() == [out[2], out[4]]
