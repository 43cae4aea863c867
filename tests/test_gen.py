"""Input generator (gen/, shared by both sides; no method arithmetic): exact nnz, no duplicate
coordinates, coordinates in range, deterministic in the seed -- for 64-bit and 128-bit packed
tuples (nell-1 extents need 69 bits, Table IV)."""
import numpy as np
import pytest

import gen
import oracle

NELL1_DIMS = (2902330, 2143368, 25495389)


@pytest.mark.parametrize("dims,alpha", [((300, 200, 500), (0.5, 0.5, 0.5)),
                                        (NELL1_DIMS, (0.5, 0.5, 0.5)),
                                        ((1 << 22, 1 << 22, 1 << 22, 1 << 22), (1.0, 0.0, 0.5, 0.0))])
def test_distinct_in_range_deterministic(dims, alpha):
    idx, val = gen.coo(dims, 20000, alpha, 7)
    assert idx.shape == (len(dims), 20000) and val.shape == (20000,)
    assert all(int(idx[m].max()) < dims[m] for m in range(len(dims)))
    assert len(set(map(tuple, idx.T.tolist()))) == 20000
    assert np.all((val > 0) & (val <= 1))
    idx2, val2 = gen.coo(dims, 20000, alpha, 7)
    assert np.array_equal(idx, idx2) and np.array_equal(val, val2)


def test_skewed_small_extent_forces_duplicate_draws():
    # 40x40 cells, 1200 distinct tuples under Zipf(1.0): many draws repeat, all dropped
    idx, _ = gen.coo((40, 40), 1200, (1.0, 1.0), 3)
    assert len(set(map(tuple, idx.T.tolist()))) == 1200


def test_oracle_build_wide_key_tensor():
    """The oracle build sorts by coordinate tuples (no key-width limit): on a nell-1-shaped sample
    the sorted stream is lexicographically ordered by (index mode, product modes)."""
    idx, val = gen.coo(NELL1_DIMS, 5000, (0.5, 0.5, 0.5), 9)
    for mode in range(3):
        f = oracle.build_fcoo(NELL1_DIMS, idx, val, oracle.OP_MTTKRP, mode, 32)
        im, pm = oracle.mode_spec(NELL1_DIMS, oracle.OP_MTTKRP, mode)
        keys = np.stack([idx[m][f.perm].astype(np.int64) for m in im + pm])
        order = np.lexsort(keys[::-1])
        assert np.array_equal(order, np.arange(5000))
