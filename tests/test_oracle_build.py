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


# ---------------------------------------------------------------------------------------------
# Blocked F-COO (orc_build_blocked; DESIGN.md §5 "blocked layout", reading Q22): the F-COO of
# each sub-tensor X_b = {q : i_outer(q) // BR == b}, concatenated, each padded to a multiple of T.
# Pinned against the (separately pinned) F-COO definition of each X_b, the single-block special
# case, brute-force orderings, and the dense definition of Eq.(5) evaluated from the stream.

def _blocked_cases():
    yield (3, (23, 17, 29), 400, 0, 8, 32)
    yield (3, (23, 17, 29), 400, 1, 5, 64)
    yield (3, (23, 17, 29), 400, 2, 4, 32)
    yield (4, (9, 6, 11, 7), 500, 0, 2, 32)
    yield (4, (9, 6, 11, 7), 500, 3, 3, 96)
    yield (2, (31, 40), 300, 0, 7, 32)
    yield (2, (31, 40), 300, 1, 16, 64)


@pytest.mark.parametrize("case", list(_blocked_cases()))
def test_blocked_blocks_are_fcoo_of_subtensors(case):
    order, dims, nnz, mode, BR, T = case
    idx, val = gen.coo(dims, nnz, None, 40 + order + mode)
    f = oracle.build_fcoo_blocked(dims, idx, val, mode, T, BR)
    outer, last = f.product_modes[0], f.product_modes[-1]
    assert f.nblocks == (dims[outer] + BR - 1) // BR
    assert f.blk_start[0] == 0 and f.blk_start[-1] == f.nstream and f.nstream % T == 0
    bits = f.bf_bits()
    for b in range(f.nblocks):
        s0, e0, s1 = int(f.blk_start[b]), int(f.blk_end[b]), int(f.blk_start[b + 1])
        sel = np.nonzero(idx[outer] // BR == b)[0]
        assert e0 - s0 == sel.size and s1 - s0 == -(-sel.size // T) * T
        # padding: empty positions
        assert np.all(f.perm[e0:s1] == 0xFFFFFFFF) and np.all(f.val[e0:s1] == 0) and np.all(f.pk[e0:s1] == 0)
        assert not bits[e0:s1].any() and np.all(f.pidx[:, e0:s1] == 0)
        if sel.size == 0:
            continue
        # the real positions are the (unblocked, pinned) F-COO of X_b, tile length irrelevant
        sub = oracle.build_fcoo(dims, idx[:, sel], val[sel], oracle.OP_MTTKRP, mode, T)
        assert np.array_equal(f.perm[s0:e0], sel[sub.perm])
        assert np.array_equal(bits[s0:e0], sub.bf_bits())
        assert np.array_equal(f.pidx[:, s0:e0], sub.pidx)
        assert np.array_equal(f.val[s0:e0].view(np.uint32), sub.val.view(np.uint32))
        # packed word: (outer - b*BR) << IB | last  (order 2: the local outer index alone)
        loc = idx[outer][f.perm[s0:e0]].astype(np.int64) - b * BR
        assert np.all((loc >= 0) & (loc < BR))
        want = (loc << f.IB) | idx[last][f.perm[s0:e0]] if order > 2 else loc
        assert np.array_equal(f.pk[s0:e0].astype(np.int64), want)
    # tile flags and segment tables follow from bf exactly as in the unblocked build
    ntiles = f.nstream // T
    for t in range(ntiles):
        assert ((int(f.sf[t >> 5]) >> (t & 31)) & 1) == bits[t * T]
        assert f.seg_base[t] == bits[: t * T].sum()
    hp = np.nonzero(bits)[0]
    assert hp.size == f.nsegs
    assert np.array_equal(f.seg_coord[:, 0], idx[mode][f.perm[hp]])


def test_blocked_single_block_equals_fcoo():
    """BR >= I_outer and T | nnz: one block, no padding -> exactly the F-COO build."""
    dims = (13, 11, 17)
    idx, val = gen.coo(dims, 256, None, 77)
    for mode in range(3):
        f = oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, mode, 32)
        g = oracle.build_fcoo_blocked(dims, idx, val, mode, 32, 64)
        assert g.nblocks == 1 and g.nstream == 256
        for a in ("perm", "bf", "sf", "seg_base", "seg_coord", "pidx"):
            assert np.array_equal(getattr(f, a), getattr(g, a)), a
        assert np.array_equal(f.val.view(np.uint32), g.val.view(np.uint32))


def test_blocked_bruteforce_orderings():
    """nnz <= 6: the real positions are the unique ordering increasing under (block, key)."""
    dims = (3, 5, 4)
    idx, val = gen.coo(dims, 6, None, 9)
    for mode in range(3):
        im, pm = oracle.mode_spec(dims, oracle.OP_MTTKRP, mode)
        BR = 2
        f = oracle.build_fcoo_blocked(dims, idx, val, mode, 2, BR)
        real = [int(p) for p in f.perm if p != 0xFFFFFFFF]
        orders = []
        for perm in itertools.permutations(range(6)):
            ks = [(int(idx[pm[0]][q]) // BR,) + tuple(int(idx[m][q]) for m in im + pm) for q in perm]
            if all(ks[a] < ks[a + 1] for a in range(5)):
                orders.append(perm)
        assert len(orders) == 1 and tuple(real) == orders[0]


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_blocked_stream_mttkrp_matches_dense(mode):
    """Eq.(5) evaluated by walking the blocked stream (segments -> rows, summed over blocks) equals
    the dense unfolding x Khatri-Rao definition (tests/dense_defs.py)."""
    import dense_defs
    dims = (6, 7, 5)
    R = 3
    idx, val = gen.coo(dims, 90, None, 31)
    fs = [np.asarray(f, np.float64) for f in gen.factors(dims, R, 4, signed=True)]
    f = oracle.build_fcoo_blocked(dims, idx, val, mode, 8, 2)
    M = np.zeros((dims[mode], R))
    bits = f.bf_bits()
    s = -1
    for p in range(f.nstream):
        if f.perm[p] == 0xFFFFFFFF:
            continue
        if bits[p]:
            s += 1
        row = int(f.seg_coord[s, 0])
        h = float(f.val[p]) * np.ones(R)
        for a, m in enumerate(f.product_modes):
            h = h * fs[m][int(f.pidx[a, p])]
        M[row] += h
    X = dense_defs.dense_from_coo(dims, idx, val)
    ref = dense_defs.mttkrp_dense(X, fs, mode)
    assert np.allclose(M, ref, rtol=1e-12, atol=1e-12)


def test_blocked_errors():
    dims = (4, 4, 4)
    dup = np.array([[0, 0], [1, 1], [2, 2]], np.uint32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_fcoo_blocked(dims, dup, np.ones(2, np.float32), 0, 4, 2)
    assert e.value.code == oracle.ERR_DUPLICATE
    # the packed word needs ceil(log2 BR) + ceil(log2 I_last) <= 32 bits
    big = (4, 3, 1 << 30)
    idx = np.array([[0, 1], [0, 1], [5, 7]], np.uint32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_fcoo_blocked(big, idx, np.ones(2, np.float32), 0, 4, 8)
    assert e.value.code == oracle.ERR_ARG


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_blocked_ttm_stream(mode):
    """Blocked F-COO for SpTTM (op = TTM): the product mode n is blocked; each blocked segment maps
    (seg_row) to the fibre with its index tuple in the plain F-COO's fibre table, and Eq.(3)
    evaluated from the blocked stream (each segment added into its fibre's row) equals the dense
    X x_n U definition (tests/dense_defs.py)."""
    import dense_defs
    dims = (7, 9, 5)
    R = 3
    idx, val = gen.coo(dims, 150, None, 37)
    U = gen.uniform((dims[mode], R), 38, mode, signed=True).astype(np.float64)
    f = oracle.build_fcoo_blocked(dims, idx, val, mode, 8, 2, op=oracle.OP_TTM)
    g = oracle.build_fcoo(dims, idx, val, oracle.OP_TTM, mode, 8)
    assert f.product_modes == [mode] and f.nfib == g.nsegs
    assert np.array_equal(g.seg_coord[f.seg_row], f.seg_coord)
    assert np.all(f.pk[f.perm != 0xFFFFFFFF] == idx[mode][f.perm[f.perm != 0xFFFFFFFF]] % 2)
    Y = np.zeros((f.nfib, R))
    bits = f.bf_bits()
    s = -1
    for p in range(f.nstream):
        if f.perm[p] == 0xFFFFFFFF:
            continue
        if bits[p]:
            s += 1
        Y[f.seg_row[s]] += float(f.val[p]) * U[int(f.pidx[0, p])]
    X = dense_defs.dense_from_coo(dims, idx, val)
    ref = dense_defs.ttm_dense(X, U, mode)
    got = np.zeros_like(ref)
    for r, c in enumerate(g.seg_coord):  # ttm_dense: the other modes in order, then the R axis
        got[tuple(int(x) for x in c)] = Y[r]
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)
