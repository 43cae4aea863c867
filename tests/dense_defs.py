"""Textbook definitions written out for pinning the oracle (independent of oracle/ and of
the CUDA path).  Each follows the cited passage literally with explicit loops."""
import itertools

import numpy as np


def dense_from_coo(dims, idx, val):
    X = np.zeros(dims, np.float64)
    for q in range(val.shape[0]):
        X[tuple(int(idx[m][q]) for m in range(len(dims)))] = float(val[q])
    return X


def unfold(X, n):
    """Mode-n matricization X_(n) (Fig. 1): columns are mode-n fibres; the other
    modes vary fastest in ascending mode order (Kolda; reading Q8: 0-based z = j + J*k)."""
    dims = X.shape
    others = [m for m in range(len(dims)) if m != n]
    ncol = int(np.prod([dims[m] for m in others]))
    out = np.zeros((dims[n], ncol), np.float64)
    for cell in itertools.product(*[range(d) for d in dims]):
        col, stride = 0, 1
        for m in others:
            col += cell[m] * stride
            stride *= dims[m]
        out[cell[n], col] = X[cell]
    return out


def kronecker(A, B):
    """Eq.(1): block (i,j) = a_ij * B."""
    I, J = A.shape
    K, L = B.shape
    out = np.zeros((I * K, J * L), np.float64)
    for i in range(I):
        for j in range(J):
            out[i * K:(i + 1) * K, j * L:(j + 1) * L] = A[i, j] * B
    return out


def khatri_rao(A, B):
    """Eq.(2): column r = a_r (x) b_r."""
    assert A.shape[1] == B.shape[1]
    cols = [kronecker(A[:, r:r + 1], B[:, r:r + 1]) for r in range(A.shape[1])]
    return np.concatenate(cols, axis=1)


def mttkrp_dense(X, factors, n):
    """Eq.(5) P:L133 generalised (Q9): X_(n) (U_{N-1} (.) ... (.) U_{n+1} (.) U_{n-1} (.) ... (.) U_0)."""
    others = [m for m in range(X.ndim) if m != n]
    kr = None
    for m in reversed(others):
        U = np.asarray(factors[m], np.float64)
        kr = U if kr is None else khatri_rao(kr, U)
    return unfold(X, n) @ kr


def kruskal_dense(lam, factors):
    dims = [U.shape[0] for U in factors]
    X = np.zeros(dims, np.float64)
    for r in range(len(lam)):
        t = np.array(lam[r], np.float64)
        for U in factors:
            t = np.multiply.outer(t, np.asarray(U[:, r], np.float64))
        X += t
    return X


def ttm_dense(X, U, n):
    """Eq.(3) P:L104 generalised to mode n: Y(..., :, ...) = sum_k X(..., k, ...) U(k, :),
    with the R axis moved to the end."""
    return np.moveaxis(np.tensordot(X, np.asarray(U, np.float64), axes=([n], [0])), -1, -1)
