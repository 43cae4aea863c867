"""Pins for the oracle SpTTMc (Eq.(4), Table I row 3 P:L233): the worked case, the rank-1
coincidence with MTTKRP, the dense unfolding x explicit Kronecker rows, and the TTM-chain
(X x_2 U2 x_3 U3) definition of P:L116."""
import json
import os

import numpy as np

import gen
import oracle
from dense_defs import dense_from_coo, kronecker, unfold

HERE = os.path.dirname(os.path.abspath(__file__))


def test_worked_case():
    for c in json.load(open(os.path.join(HERE, "golden", "ttmc_cases.json")))["cases"]:
        idx = np.array(c["coords"], np.uint32).T.copy()
        fs = [None if f is None else np.array(f, np.float32) for f in c["factors"]]
        Y, _ = oracle.ttmc(c["dims"], idx, np.array(c["vals"], np.float32), c["mode"], fs)
        assert np.array_equal(Y, np.array(c["Y"], float)), c["cite"]


def test_rank1_equals_mttkrp():
    """R_m = 1 for every other mode: the Kronecker row is the Hadamard row."""
    dims = (9, 7, 5, 4)
    idx, val = gen.coo(dims, 200, None, 91)
    fs = gen.factors(dims, 1, 92, signed=True)
    for n in range(4):
        Y, _ = oracle.ttmc(dims, idx, val, n, fs)
        M, _ = oracle.mttkrp(dims, idx, val, n, fs)
        assert np.allclose(Y, M, rtol=1e-14, atol=1e-15)


def _kron_row(factors, others, cell):
    row = np.ones((1, 1))
    for m in others:  # ascending mode order, first factor outermost (Eq.(1))
        row = kronecker(row, factors[m][cell[m]:cell[m] + 1].astype(np.float64))
    return row[0]


def test_dense_unfolding_times_kronecker_rows():
    dims = (5, 4, 3, 2)
    idx, val = gen.coo(dims, 80, None, 93)
    ranks = (2, 3, 2, 2)
    fs = [gen.uniform((d, r), 94, m, signed=True) for m, (d, r) in enumerate(zip(dims, ranks))]
    X = dense_from_coo(dims, idx, val)
    for n in range(4):
        others = [m for m in range(4) if m != n]
        Xn = unfold(X, n)
        # column z of X_(n): the other modes' indices with the first other mode fastest (Q8)
        K = []
        for z in range(Xn.shape[1]):
            cell, rem = {}, z
            for m in others:
                cell[m] = rem % dims[m]
                rem //= dims[m]
            K.append(_kron_row(fs, others, cell))
        ref = Xn @ np.array(K)
        Y, _ = oracle.ttmc(dims, idx, val, n, fs)
        assert np.allclose(Y, ref, rtol=1e-12, atol=1e-13)


def test_ttm_chain_definition():
    """mode-1 TTMc = X x_2 U2 x_3 U3; Y(i,p,q) = sum_jk X(i,j,k) U2(j,p) U3(k,q), p outer."""
    dims = (6, 5, 4)
    idx, val = gen.coo(dims, 60, None, 95)
    U2 = gen.uniform((5, 3), 96, 0, signed=True)
    U3 = gen.uniform((4, 2), 96, 1, signed=True)
    X = dense_from_coo(dims, idx, val)
    ref = np.einsum("ijk,jp,kq->ipq", X, U2.astype(np.float64), U3.astype(np.float64)).reshape(6, 6)
    Y, D = oracle.ttmc(dims, idx, val, 0, [None, U2, U3])
    assert np.allclose(Y, ref, rtol=1e-12, atol=1e-13)
    assert np.all(D >= np.abs(Y) - 1e-15)
