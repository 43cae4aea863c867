"""GPU: the device F-COO build is bit-exact against the oracle build (SURVEY §8(c) c1 acceptance),
through the C ABI (fcoo_build + fcoo_export)."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_09905_b200 as F
    return F


def _compare(F, dims, idx, val, op, mode, T, desc=False):
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, op=op, tile_nnz=T, keep_perm=True, product_desc=desc)
    got = F.fcoo_export(h, perm=True)
    ref = oracle.build_fcoo(dims, idx, val, op, mode, T, desc=desc)
    assert h.info.nsegs == ref.nsegs
    assert h.info.idx_modes == ref.index_modes and h.info.prod_modes == ref.product_modes
    assert np.array_equal(got["perm"], ref.perm)
    assert got["bf"].tobytes() == ref.bf.tobytes()
    assert got["sf"].tobytes() == ref.sf.tobytes()
    assert got["seg_base"].tobytes() == ref.seg_base.tobytes()
    assert got["seg_coord"].tobytes() == ref.seg_coord.tobytes()
    assert got["pidx"].tobytes() == ref.pidx.tobytes()
    assert got["val"].tobytes() == ref.val.tobytes()
    assert h.info.storage_bytes == oracle.storage_bytes(val.shape[0], len(ref.product_modes), T)
    h.destroy()


def test_build_tiny_all_modes(F):
    w = gen.WORKLOADS["tiny"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        for op in (F.OP_MTTKRP, F.OP_TTM):
            _compare(F, w.dims, idx, val, op, mode, 32)


@pytest.mark.parametrize("T", [32, 64, 256, 1024])
def test_build_random(F, T):
    for dims, alpha in (((300, 200, 500), (0.5, 0.5, 0.5)), ((40, 50, 30, 20), (0.8, 0.0, 0.5, 0.3)),
                        ((3000, 7), (0.0, 0.0))):
        idx, val = gen.coo(dims, 20000, alpha, 17)
        for mode in range(len(dims)):
            for op in (F.OP_MTTKRP, F.OP_TTM):
                _compare(F, dims, idx, val, op, mode, T)


def test_build_product_desc_option(F):
    for dims in ((300, 200, 500), (40, 50, 30, 20)):
        idx, val = gen.coo(dims, 20000, None, 19)
        for mode in range(len(dims)):
            _compare(F, dims, idx, val, F.OP_MTTKRP, mode, 64, desc=True)


def test_build_nell2_subset(F):
    w = gen.WORKLOADS["nell2"]
    idx, val = gen.coo(w.dims, 2_000_000, w.alpha, w.seed)
    for mode in range(3):
        _compare(F, w.dims, idx, val, F.OP_MTTKRP, mode, 256)


def test_build_edge_cases(F):
    # singleton tensor; all nonzeros in one slice (one giant segment); all singleton segments
    _compare(F, (5, 6, 7), np.array([[3], [4], [5]], np.uint32), np.array([2.5], np.float32), F.OP_MTTKRP, 1, 32)
    n = 5000
    one = np.stack([np.zeros(n, np.uint32), (np.arange(n) % 100).astype(np.uint32),
                    (np.arange(n) // 100).astype(np.uint32)])
    v = gen.uniform((n,), 3, 0) + 0.5
    _compare(F, (1, 100, 50), one, v, F.OP_MTTKRP, 0, 64)
    single = np.stack([np.arange(n, dtype=np.uint32), (np.arange(n) * 7 % 13).astype(np.uint32),
                       np.zeros(n, np.uint32)])
    _compare(F, (n, 13, 1), single, v, F.OP_MTTKRP, 0, 32)
    _compare(F, (n, 13, 1), single, v, F.OP_TTM, 2, 32)


# FROSTT nell-1 extents (Table IV P:L414 "2.9M x 2.1M x 25.5M"): 22 + 22 + 25 = 69 key bits, so the
# build takes the 128-bit key path
NELL1_DIMS = (2902330, 2143368, 25495389)


def test_build_wide_keys_nell1_shape(F):
    idx, val = gen.coo(NELL1_DIMS, 300_000, (0.5, 0.5, 0.5), 23)
    for mode in range(3):
        for op in (F.OP_MTTKRP, F.OP_TTM):
            _compare(F, NELL1_DIMS, idx, val, op, mode, 256)


def test_build_wide_keys_boundaries(F):
    # 64 bits exactly (last 64-bit case), 65 bits (first 128-bit case), 128 bits exactly
    for dims in (((1 << 32) - 1, (1 << 32) - 1), ((1 << 32) - 1, (1 << 32) - 1, 2),
                 ((1 << 32) - 1,) * 4):
        n = 3000
        # row 0 is q * prime mod (2^32 - 1): distinct, so no duplicate coordinates
        idx = np.stack([(np.arange(n, dtype=np.uint64) * np.uint64(2654435761 + 2 * m) % np.uint64(dims[m]))
                        .astype(np.uint32) for m in range(len(dims))])
        val = (gen.uniform((n,), 41, 0) + 0.5).astype(np.float32)
        for mode in range(len(dims)):
            _compare(F, dims, idx, val, F.OP_MTTKRP, mode, 64)
            _compare(F, dims, idx, val, F.OP_TTM, mode, 32)


def test_build_errors(F):
    dims = (10, 10, 10)
    idx = np.array([[1, 2, 1], [1, 2, 1], [1, 2, 1]], np.uint32)  # duplicate (1,1,1)
    val = np.ones(3, np.float32)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_build(F.Coo.from_numpy(dims, idx, val), 0)
    assert e.value.code == 5  # FCOO_ERR_DUPLICATE
    bad = np.array([[1, 2], [1, 10], [1, 2]], np.uint32)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_build(F.Coo.from_numpy(dims, bad, val[:2]), 0)
    assert e.value.code == 4  # FCOO_ERR_INDEX_RANGE
    big = (1 << 30,) * 5  # 150 key bits > 128
    idx5 = np.array([[1, 2]] * 5, np.uint32)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_build(F.Coo.from_numpy(big, idx5, val[:2]), 0)
    assert e.value.code == 7  # FCOO_ERR_KEY_BITS


def test_tns_file_to_device_build(F, tmp_path):
    """Real-dataset path: FROSTT text -> native reader -> device build, with
    nell-1 extents given as the dims override (69-bit keys)."""
    idx, val = gen.coo(NELL1_DIMS, 50_000, (0.5, 0.5, 0.5), 29)
    path = str(tmp_path / "nell1_sample.tns")
    F.write_tns(path, idx, val)
    dims, idx2, val2 = F.read_tns(path, dims=NELL1_DIMS)
    assert dims == NELL1_DIMS and np.array_equal(idx2, idx) and np.array_equal(val2, val)
    for mode in range(3):
        _compare(F, dims, idx2, val2, F.OP_MTTKRP, mode, 128)
