"""Parity helpers for the GPU tests (compare the CUDA path with the oracle)."""
import numpy as np

# north_star: "max relative error <= 1e-4 per output element, normalised by that row's sum of
# |contributions|" — per element (i, r), the stricter reading.
TOL = 1e-4


def normalized_error(gpu: np.ndarray, ref: np.ndarray, D: np.ndarray):
    """Returns (max err over D > 0, all exact-zero where D == 0)."""
    gpu = gpu.astype(np.float64)
    pos = D > 0
    err = np.zeros_like(ref)
    err[pos] = np.abs(gpu[pos] - ref[pos]) / D[pos]
    zero_ok = bool(np.all(gpu[~pos] == 0.0))
    return float(err.max() if err.size else 0.0), zero_ok


def assert_parity(gpu, ref, D, tol=TOL, what=""):
    e, z = normalized_error(gpu, ref, D)
    assert z, f"{what}: nonzero output where the oracle has no contributions"
    assert e <= tol, f"{what}: normalized error {e:.3e} > {tol:g}"
    return e
