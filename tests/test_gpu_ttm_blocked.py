"""GPU: SpTTM (Eq.(3)) on a BLOCKED F-COO handle (FCOO_BUILD_BLOCKED with op TTM,
DESIGN.md §5 / §6.4, reading Q22) through the C ABI.

- the device build is byte-exact against the oracle's orc_build_blocked_ex(op = TTM): perm, bf,
  sf, segment tables, packed words (the local index i_n - b*BR), block tables, and the fibre map
  seg_row (segment -> output row) with the fibre table (= the plain F-COO's segment table);
- the blocked SpTTM kernel (U's block of BR rows in shared memory, every (block, fibre) segment
  red.add-ed into its fibre's row) matches the fp64 oracle element by element within the
  normalised 1e-4 tolerance, across ranks, orders 3-4, tiles, block sizes, tile-aligned shards and
  the full-size brainq-shaped configuration (BASELINE configs[3]) at the automatic tile.
"""
import numpy as np
import pytest

import gen
import oracle
from parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_09905_b200 as F
    return F


def _compare_build(F, dims, idx, val, mode, T, BR):
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, op=F.OP_TTM, tile_nnz=T, keep_perm=True, blocked=True, block_rows=BR)
    got = F.fcoo_export(h, perm=True)
    ref = oracle.build_fcoo_blocked(dims, idx, val, mode, T, BR, op=oracle.OP_TTM)
    plain = oracle.build_fcoo(dims, idx, val, oracle.OP_TTM, mode, T)
    i = h.info
    assert i.blocked and i.nblocks == ref.nblocks and i.nstream == ref.nstream and i.nsegs == ref.nsegs
    assert i.nfib == ref.nfib == plain.nsegs and i.prod_modes == [mode]
    assert np.array_equal(got["perm"], ref.perm)
    assert got["bf"].tobytes() == ref.bf.tobytes()
    assert got["sf"].tobytes() == ref.sf.tobytes()
    assert got["seg_base"].tobytes() == ref.seg_base.tobytes()
    assert got["seg_coord"].tobytes() == ref.seg_coord.tobytes()
    assert got["val"].tobytes() == ref.val.tobytes()
    assert got["pk"][0].tobytes() == ref.pk.tobytes()
    assert got["pidx"].tobytes() == ref.pidx.tobytes()
    assert np.array_equal(got["blk_start"], ref.blk_start) and np.array_equal(got["blk_end"], ref.blk_end)
    assert got["seg_row"].tobytes() == ref.seg_row.tobytes()
    assert got["fib_coord"].tobytes() == plain.seg_coord.tobytes()
    h.destroy()


@pytest.mark.parametrize("T", [32, 256])
def test_blocked_ttm_build(F, T):
    for dims, alpha, BR, nnz in (((60, 700, 9), None, 64, 20000), ((30, 40, 20, 10), (0.5, 0.5, 0.5, 0.5), 32, 15000),
                                 ((5, 3000, 4), (0.0, 0.9, 0.0), 256, 12000)):
        idx, val = gen.coo(dims, nnz, alpha, 23)
        for mode in range(len(dims)):
            _compare_build(F, dims, idx, val, mode, T, BR)


def _check(F, dims, idx, val, mode, R, T=256, BR=0, shards=1, signed=True):
    import torch
    U = gen.uniform((dims[mode], R), 61, mode, signed=signed)
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, op=F.OP_TTM, tile_nnz=T, blocked=True, block_rows=BR)
    nfib = h.info.nfib
    out = torch.full((nfib, R), float("nan"), device="cuda")
    Ut = torch.from_numpy(U).cuda()
    if shards == 1:
        F.fcoo_ttm(h, Ut, R, out)
    else:
        acc = torch.zeros_like(out)
        for g in range(shards):
            F.fcoo_set_shard(h, g, shards)
            F.fcoo_ttm(h, Ut, R, out)
            acc += out
        out = acc
    torch.cuda.synchronize()
    ex = F.fcoo_export(h)
    coords, Y, D = oracle.ttm(dims, idx, val, mode, U)
    assert np.array_equal(ex["fib_coord"], coords)
    got = out.cpu().numpy()
    h.destroy()
    return assert_parity(got, Y, D, what=f"blocked ttm dims={dims} mode={mode} R={R} T={T} BR={BR}")


@pytest.mark.parametrize("R", [1, 4, 8, 16, 32, 64, 100])
def test_blocked_ttm_ranks(F, R):
    """float4 lanes (R = 8..64, U block in shared memory), scalar lanes (R = 1, 4 -> G = 1, 100)."""
    dims = (60, 3000, 9)
    idx, val = gen.coo(dims, 40000, (0.3, 0.0, 0.6), 71)
    for mode in range(3):
        _check(F, dims, idx, val, mode, R, T=64, BR=128)


def test_blocked_ttm_order4_tiles_shards(F):
    dims = (30, 40, 20, 10)
    idx, val = gen.coo(dims, 30000, (0.5, 0.5, 0.5, 0.5), 73)
    for mode in range(4):
        _check(F, dims, idx, val, mode, 16, T=32, BR=32)
        _check(F, dims, idx, val, mode, 16, T=128, BR=64, shards=3)


def test_blocked_ttm_long_fibre(F):
    """One fibre (mode 1 of a 1 x N x 1 tensor) spanning every block and every tile."""
    n = 30000
    v = gen.uniform((n,), 5, 0) + 0.5
    one = np.stack([np.zeros(n, np.uint32), np.arange(n, dtype=np.uint32), np.zeros(n, np.uint32)])
    _check(F, (1, n, 1), one, v, 1, 16, T=32, BR=1024, signed=False)


def test_brainq_blocked_full_size(F):
    """BASELINE configs[3] at full size (60 x 70K x 9, 11M nnz), R=16, every mode on blocked
    handles at the automatic tile and block size (the launch configuration ops_bench times)."""
    w = gen.WORKLOADS["brainq"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        _check(F, w.dims, idx, val, mode, 16, T=0, BR=0)


def test_blocked_ttm_edge_shapes(F):
    """Order 5; R = 128 (32-lane float4 groups) and R = 100 (scalar lanes); block rows that do not
    divide I_n; an empty block (no nonzero has i_n in [64, 128)); a single fibre."""
    dims = (6, 5, 4, 7, 3)
    idx, val = gen.coo(dims, 2000, None, 107)
    for mode in range(5):
        _check(F, dims, idx, val, mode, 16, T=32, BR=32)
    dims = (40, 300, 30)
    idx, val = gen.coo(dims, 20000, (0.4, 0.2, 0.3), 109)
    for R in (128, 100):
        _check(F, dims, idx, val, 1, R, T=64, BR=96)
    keep = (idx[1] < 64) | (idx[1] >= 128)
    _check(F, dims, idx[:, keep].copy(), val[keep].copy(), 1, 16, T=32, BR=64)
    n = 5000
    one = np.stack([np.full(n, 3, np.uint32), np.arange(n, dtype=np.uint32) % 300, np.full(n, 7, np.uint32)])
    one = one[:, np.unique(one[1], return_index=True)[1]].copy()
    _check(F, dims, one, gen.uniform((one.shape[1],), 7, 0) + 0.5, 1, 32, T=32, BR=64, signed=False)
