"""Pins for the oracle F-COO build (oracle/fcoo_oracle.cpp: orc_mode_spec, orc_build,
orc_storage_bytes).  Each check is fixed by the paper or by a definition, not by the
oracle itself: Table I, Table II, the worked flag cases, brute-force permutations and
structural invariants."""
import itertools

import numpy as np
import pytest

import gen
import oracle


def _tensor_from_i(i_seq):
    """3-order tensor whose mode-0 coords follow i_seq in sorted order (j increasing)."""
    n = len(i_seq)
    idx = np.zeros((3, n), np.uint32)
    idx[0] = i_seq
    idx[1] = np.arange(n)
    idx[2] = 0
    return (max(i_seq) + 1, n, 1), idx, np.arange(1, n + 1, dtype=np.float32)


def test_table1_mode_spec():
    # Table I P:L229-233 (1-based modes in the paper; 0-based here)
    im, pm = oracle.mode_spec((4, 5, 6), oracle.OP_TTM, 2)          # SpTTM on mode-3
    assert im == [0, 1] and pm == [2]
    im, pm = oracle.mode_spec((4, 5, 6), oracle.OP_MTTKRP, 0)       # SpMTTKRP on mode-1
    assert im == [0] and sorted(pm) == [1, 2]
    # Q5: product modes by ascending extent, ties by mode id
    assert oracle.mode_spec((5, 9, 3), oracle.OP_MTTKRP, 0)[1] == [2, 1]
    assert oracle.mode_spec((5, 3, 3, 2), oracle.OP_MTTKRP, 0)[1] == [3, 1, 2]
    with pytest.raises(oracle.OracleError):
        oracle.mode_spec((4, 5, 6), oracle.OP_MTTKRP, 3)
    with pytest.raises(oracle.OracleError):
        oracle.mode_spec((4,), oracle.OP_MTTKRP, 0)


def test_hand_flag_cases(golden):
    for case in golden["build_flags"]:
        dims, idx, val = _tensor_from_i(case["i"])
        f = oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, 0, case["T"])
        assert list(f.bf_bits()) == case["bf"], case["cite"]
        ntiles = (len(case["i"]) + case["T"] - 1) // case["T"]
        sf_bits = [(int(f.sf[t >> 5]) >> (t & 31)) & 1 for t in range(ntiles)]
        assert sf_bits == case["sf"], case["cite"]
        assert list(f.seg_coord[:, 0]) == case["seg_coord"], case["cite"]
        assert list(f.seg_base) == case["seg_base"], case["cite"]


def test_table2_storage(golden):
    for case in golden["storage"]:
        if "bytes" in case:
            assert oracle.storage_bytes(case["nnz"], case["n_prod"], case["T"]) == case["bytes"], case["cite"]
        else:  # F-COO is smaller than COO for every op
            for n_prod in (1, 2):
                assert oracle.storage_bytes(case["nnz"], n_prod, 8) < case["coo_bytes"]


def _check_invariants(dims, idx, val, op, mode, T):
    f = oracle.build_fcoo(dims, idx, val, op, mode, T)
    nnz = val.shape[0]
    im, pm = f.index_modes, f.product_modes
    # perm is a bijection
    assert np.array_equal(np.sort(f.perm), np.arange(nnz, dtype=np.uint32))
    keys = np.stack([idx[m][f.perm] for m in im + pm]).astype(np.int64)
    # rows are strictly increasing under the key (lexicographic)
    for p in range(1, nnz):
        a, b = tuple(keys[:, p - 1]), tuple(keys[:, p])
        assert a < b
    # bf marks exactly the index-tuple changes; popcount = nsegs = #distinct tuples
    bits = f.bf_bits()
    heads = np.ones(nnz, bool)
    heads[1:] = np.any(keys[: len(im), 1:] != keys[: len(im), :-1], axis=0)
    assert np.array_equal(bits.astype(bool), heads)
    ntuples = len({tuple(idx[m][q] for m in im) for q in range(nnz)})
    assert int(bits.sum()) == f.nsegs == ntuples
    # pad bits of the last bf byte are 0
    assert np.unpackbits(f.bf, bitorder="little")[nnz:].sum() == 0
    # sf[t] = bf[t*T]; seg_base[t] = heads before t*T
    ntiles = (nnz + T - 1) // T
    for t in range(ntiles):
        assert ((int(f.sf[t >> 5]) >> (t & 31)) & 1) == bits[t * T]
        assert f.seg_base[t] == bits[: t * T].sum()
    # seg_coord = index coords at heads; permuted arrays are gathers of the input
    hp = np.nonzero(bits)[0]
    for a, m in enumerate(im):
        assert np.array_equal(f.seg_coord[:, a], idx[m][f.perm[hp]])
    for a, m in enumerate(pm):
        assert np.array_equal(f.pidx[a], idx[m][f.perm])
    assert np.array_equal(f.val.view(np.uint32), val[f.perm].view(np.uint32))
    # multiset of (coord, value) preserved
    got = sorted(zip(*(idx[m][f.perm].tolist() for m in range(len(dims))), f.val.tolist()))
    want = sorted(zip(*(idx[m].tolist() for m in range(len(dims))), val.tolist()))
    assert got == want
    return f


@pytest.mark.parametrize("T", [1, 3, 32])
def test_invariants_random(T):
    for order, dims in ((3, (7, 5, 9)), (4, (4, 6, 3, 5)), (2, (11, 17))):
        idx, val = gen.coo(dims, 150, None, 11 + order)
        for mode in range(order):
            for op in (oracle.OP_MTTKRP, oracle.OP_TTM):
                _check_invariants(dims, idx, val, op, mode, T)


def test_bruteforce_permutations():
    """nnz <= 6: the sorted permutation is the unique ordering that is increasing under the
    Table I key; enumerate all orderings and compare."""
    dims = (3, 3, 4)
    idx, val = gen.coo(dims, 6, None, 5)
    for mode in range(3):
        for op in (oracle.OP_MTTKRP, oracle.OP_TTM):
            im, pm = oracle.mode_spec(dims, op, mode)
            f = oracle.build_fcoo(dims, idx, val, op, mode, 2)
            sorted_orders = []
            for perm in itertools.permutations(range(6)):
                ks = [tuple(int(idx[m][q]) for m in im + pm) for q in perm]
                if all(ks[a] < ks[a + 1] for a in range(5)):
                    sorted_orders.append(perm)
            assert len(sorted_orders) == 1
            assert tuple(int(x) for x in f.perm) == sorted_orders[0]


def test_errors():
    dims = (4, 4, 4)
    idx = np.array([[0, 1], [0, 1], [0, 1]], np.uint32)
    val = np.ones(2, np.float32)
    dup = np.array([[0, 0], [1, 1], [2, 2]], np.uint32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_fcoo(dims, dup, val, oracle.OP_MTTKRP, 0, 4)
    assert e.value.code == oracle.ERR_DUPLICATE
    bad = idx.copy()
    bad[2, 1] = 4
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_fcoo(dims, bad, val, oracle.OP_MTTKRP, 0, 4)
    assert e.value.code == oracle.ERR_INDEX_RANGE
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_fcoo(dims, idx[:, :0], val[:0], oracle.OP_MTTKRP, 0, 4)
    assert e.value.code == oracle.ERR_EMPTY
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, 3, 4)
    assert e.value.code == oracle.ERR_MODE


def test_toggle_reading_equivalence():
    """Q1: a toggle encoding (bit flips at every new segment) marks the same
    boundaries as the head-marker bf: head[p] = tog[p] xor tog[p-1], head[0] = 1."""
    dims = (9, 8, 7)
    idx, val = gen.coo(dims, 200, None, 3)
    f = oracle.build_fcoo(dims, idx, val, oracle.OP_TTM, 1, 8)
    heads = f.bf_bits().astype(np.int64)
    tog = np.cumsum(heads) & 1
    back = np.concatenate([[1], tog[1:] ^ tog[:-1]])
    assert np.array_equal(back, heads)


def test_product_desc_option_invariants():
    """FCOO_BUILD_PRODUCT_DESC: same index modes and segments, product modes by descending extent."""
    dims = (7, 5, 9, 4)
    idx, val = gen.coo(dims, 300, None, 23)
    assert oracle.mode_spec(dims, oracle.OP_MTTKRP, 0, desc=True)[1] == [2, 1, 3]
    for mode in range(4):
        a = oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, mode, 32)
        b = oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, mode, 32, desc=True)
        assert a.nsegs == b.nsegs and np.array_equal(a.bf, b.bf) and np.array_equal(a.seg_coord, b.seg_coord)
        keys = np.stack([idx[m][b.perm] for m in b.index_modes + b.product_modes]).astype(np.int64)
        for p in range(1, val.shape[0]):
            assert tuple(keys[:, p - 1]) < tuple(keys[:, p])
