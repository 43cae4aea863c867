"""GPU: the blocked F-COO (FCOO_BUILD_BLOCKED, reading Q22) through the C ABI.

- the device build is byte-exact against the oracle's orc_build_blocked (perm, bf, sf, segment
  tables, decoded product indices, values, packed words, block tables), including the full-size
  nell-2-shaped tensor at the automatic tile that bench.py times;
- SpMTTKRP on blocked handles matches the fp64 oracle element by element (normalised by the
  per-element sum of |contributions|, tolerance 1e-4) across ranks (float4 lanes with the shared-
  memory block at 256 and 512 threads, scalar lanes with global outer rows), orders 2..5, tiles,
  block sizes, shards and the full-size configuration.
"""
import concurrent.futures as cf

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


def _compare_build(F, dims, idx, val, mode, T, BR, coo=None, ref=None):
    coo = coo or F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, tile_nnz=T, keep_perm=True, blocked=True, block_rows=BR)
    got = F.fcoo_export(h, perm=True)
    ref = ref or oracle.build_fcoo_blocked(dims, idx, val, mode, T, BR)
    i = h.info
    assert i.blocked and i.block_rows == BR and i.nblocks == ref.nblocks and i.nstream == ref.nstream
    assert i.nsegs == ref.nsegs and i.prod_modes == ref.product_modes and i.pk_shift == ref.IB
    assert np.array_equal(got["perm"], ref.perm)
    assert got["bf"].tobytes() == ref.bf.tobytes()
    assert got["sf"].tobytes() == ref.sf.tobytes()
    assert got["seg_base"].tobytes() == ref.seg_base.tobytes()
    assert got["seg_coord"].tobytes() == ref.seg_coord.tobytes()
    assert got["pidx"].tobytes() == ref.pidx.tobytes()
    assert got["val"].tobytes() == ref.val.tobytes()
    assert got["pk"][0].tobytes() == ref.pk.tobytes()
    for a in range(1, len(ref.product_modes) - 1):  # middle product modes: stored as global indices
        assert np.array_equal(got["pk"][a], ref.pidx[a])
    assert np.array_equal(got["blk_start"], ref.blk_start) and np.array_equal(got["blk_end"], ref.blk_end)
    h.destroy()


@pytest.mark.parametrize("T", [32, 64, 256, 1024])
def test_blocked_build_random(F, T):
    cases = (((300, 200, 500), (0.5, 0.5, 0.5), 40), ((40, 50, 30, 20), (0.8, 0.0, 0.5, 0.3), 32),
             ((3000, 70), (0.0, 0.0), 64), ((12, 10, 8, 6, 5), None, 32))
    for dims, alpha, BR in cases:
        nnz = min(20000, int(np.prod(dims) * 0.3))
        idx, val = gen.coo(dims, nnz, alpha, 17)
        for mode in range(len(dims)):
            _compare_build(F, dims, idx, val, mode, T, BR)


def test_blocked_build_tiny_and_single_block(F):
    w = gen.WORKLOADS["tiny"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        _compare_build(F, w.dims, idx, val, mode, 32, 32)
        _compare_build(F, w.dims, idx, val, mode, 64, 65536)  # one block


def test_blocked_build_errors(F):
    w = gen.WORKLOADS["tiny"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    coo = F.Coo.from_numpy(w.dims, idx, val)
    for kw, code in ((dict(deterministic=True), F.ERR_ARG),
                     (dict(product_desc=True), F.ERR_ARG), (dict(block_rows=16), F.ERR_ARG),
                     (dict(block_rows=70000), F.ERR_ARG)):
        with pytest.raises(F.FcooError) as e:
            F.fcoo_build(coo, 0, blocked=True, **kw)
        assert e.value.code == code, kw
    dims6 = (3, 3, 3, 3, 3, 3)
    i6, v6 = gen.coo(dims6, 100, None, 3)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_build(F.Coo.from_numpy(dims6, i6, v6), 0, blocked=True)
    assert e.value.code == F.ERR_ARG
    # the packed word must fit 32 bits: ceil(log2 BR) + ceil(log2 I_last)
    big = (4, 3, 1 << 30)
    ib = np.array([[0, 1], [0, 1], [5, 7]], np.uint32)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_build(F.Coo.from_numpy(big, ib, np.ones(2, np.float32)), 0, blocked=True, block_rows=8 * 1024)
    assert e.value.code == F.ERR_ARG
    # duplicates are detected after the sort (second host sync)
    dup = np.concatenate([idx, idx[:, :1]], axis=1)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_build(F.Coo.from_numpy(w.dims, dup, np.concatenate([val, val[:1]])), 1, blocked=True)
    assert e.value.code == F.ERR_DUPLICATE
    h = F.fcoo_build(coo, 0, blocked=True)
    out = __import__("torch").empty((w.dims[0], 8 * 8), device="cuda")
    fs = [__import__("torch").ones((d, 8), device="cuda") for d in w.dims]
    with pytest.raises(F.FcooError) as e:  # SpTTMc needs the unblocked layout
        F.fcoo_ttmc(h, fs, out)
    assert e.value.code == F.ERR_SHAPE
    h.destroy()


def _run(F, dims, idx, val, mode, fs_np, R, T, BR, shards=1):
    import torch
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, tile_nnz=T, blocked=True, block_rows=BR)
    fs = [torch.from_numpy(f).cuda() for f in fs_np]
    out = torch.full((dims[mode], R), float("nan"), device="cuda")
    if shards == 1:
        F.fcoo_mttkrp(h, fs, R, out)
    else:  # fake multi-rank: tile-aligned shards one after another, partials summed on the device
        acc = torch.zeros_like(out)
        for g in range(shards):
            F.fcoo_set_shard(h, g, shards)
            F.fcoo_mttkrp(h, fs, R, out)
            acc += out
        out = acc
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    h.destroy()
    return res


def _check(F, dims, idx, val, mode, R, T=64, BR=64, signed=True, shards=1, seed=5):
    fs = gen.factors(dims, R, seed, signed=signed)
    got = _run(F, dims, idx, val, mode, fs, R, T, BR, shards)
    M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
    return assert_parity(got, M, D, what=f"blocked dims={dims} mode={mode} R={R} T={T} BR={BR} shards={shards}")


def test_blocked_mttkrp_tiny(F):
    w = gen.WORKLOADS["tiny"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        _check(F, w.dims, idx, val, mode, 8, T=32, BR=32)
        _check(F, w.dims, idx, val, mode, 8, T=256, BR=4096, signed=False)


# R: float4 lanes G = 2..32 (8..128), block in shared memory at 256 threads (R <= 32 with BR 512
# and every R with BR 64) or 512 threads (R = 64, BR 512); scalar lanes (1, 3, 100, 200, 256)
# and float4 ranks whose block does not fit (R = 128, BR 512) read the outer rows from global memory
@pytest.mark.parametrize("R", [1, 3, 8, 16, 32, 48, 64, 100, 128, 256])
def test_blocked_ranks(F, R):
    dims = (900, 700, 1500)
    idx, val = gen.coo(dims, 40000, (0.5, 0.5, 0.5), 23)
    for mode in range(3):
        for BR in (64, 512):
            _check(F, dims, idx, val, mode, R, T=64, BR=BR)


@pytest.mark.parametrize("dims", [(40, 50, 30, 20), (12, 10, 8, 6, 5), (3000, 700), (2000, 60)])
def test_blocked_orders(F, dims):
    nnz = min(20000, int(np.prod(dims) * 0.3))
    idx, val = gen.coo(dims, nnz, None, 29)
    for mode in range(len(dims)):
        for R in (16, 5):
            _check(F, dims, idx, val, mode, R, T=32, BR=32)


@pytest.mark.parametrize("T", [32, 96, 256, 2048])
def test_blocked_tiles_and_ragged_blocks(F, T):
    dims = (700, 1100, 900)
    idx, val = gen.coo(dims, 22345, (0.7, 0.3, 0.5), 31)
    for mode in range(3):
        _check(F, dims, idx, val, mode, 32, T=T, BR=100)


def test_blocked_adversarial_segments(F):
    n = 20000
    v = gen.uniform((n,), 3, 0) + 0.5
    # one giant slice spanning many tiles of every block
    giant = np.stack([np.zeros(n, np.uint32), (np.arange(n) % 200).astype(np.uint32),
                      (np.arange(n) // 200).astype(np.uint32)])
    _check(F, (3, 200, 100), giant, v, 0, 32, T=32, BR=32, signed=False)
    # singleton segments and empty rows
    single = np.stack([(np.arange(n) * 2).astype(np.uint32), (np.arange(n) % 130).astype(np.uint32),
                       (np.arange(n) % 50).astype(np.uint32)])
    _check(F, (2 * n + 5, 130, 50), single, v, 0, 32, T=32, BR=32)
    # empty blocks: outer indices only in a few scattered blocks
    sparse = np.stack([(np.arange(n) % 97).astype(np.uint32), ((np.arange(n) % 5) * 1000).astype(np.uint32),
                       (np.arange(n) // 97).astype(np.uint32)])
    _check(F, (97, 5000, n // 97 + 1), sparse, v, 0, 16, T=64, BR=64)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_blocked_fake_multirank_shards(F, shards):
    dims = (100, 900, 800)
    idx, val = gen.coo(dims, 50000, (1.0, 0.5, 0.5), 37)
    for mode in range(3):
        _check(F, dims, idx, val, mode, 32, T=64, BR=128, shards=shards)


# ---- full size: BASELINE configs[1] (nell-2-shaped, 76.9M nnz), the bench's exact build ----

@pytest.fixture(scope="module")
def nell2():
    w, idx, val = gen.workload("nell2")
    return w, idx, val


def test_blocked_build_nell2_full_size_all_modes(F, nell2):
    """Byte-exact against the oracle at full size, automatic tile, default block rows (the layout
    bench.py times), every mode; the three oracle builds run in parallel host threads."""
    w, idx, val = nell2
    coo = F.Coo.from_numpy(w.dims, idx, val)
    h0 = F.fcoo_build(coo, 0, blocked=True)
    T, BR = h0.info.tile_nnz, h0.info.block_rows
    h0.destroy()
    with cf.ThreadPoolExecutor(3) as ex:
        refs = list(ex.map(lambda m: oracle.build_fcoo_blocked(w.dims, idx, val, m, T, BR), range(3)))
    for mode in range(3):
        _compare_build(F, w.dims, idx, val, mode, T, BR, coo=coo, ref=refs[mode])
        refs[mode] = None


def test_build_nell2_full_size_all_modes_unblocked(F, nell2):
    """The unblocked F-COO at full size and the automatic tile, byte-exact, every mode."""
    w, idx, val = nell2
    coo = F.Coo.from_numpy(w.dims, idx, val)
    T = F.fcoo_build(coo, 0).info.tile_nnz
    with cf.ThreadPoolExecutor(3) as ex:
        refs = list(ex.map(lambda m: oracle.build_fcoo(w.dims, idx, val, oracle.OP_MTTKRP, m, T), range(3)))
    for mode in range(3):
        h = F.fcoo_build(coo, mode, keep_perm=True)
        got = F.fcoo_export(h, perm=True)
        ref = refs[mode]
        assert h.info.nsegs == ref.nsegs
        for k in ("perm", "bf", "sf", "seg_base", "seg_coord", "pidx", "val"):
            assert got[k].tobytes() == getattr(ref, k).tobytes(), k
        h.destroy()
        refs[mode] = None


@pytest.mark.parametrize("R", [16, 32, 64])
def test_blocked_mttkrp_nell2_full_size(F, nell2, R):
    """Every output element at full size against the OpenMP fp64 oracle, R = 16/32/64."""
    import os
    w, idx, val = nell2
    fs = gen.factors(w.dims, R, 7, signed=True)
    coo = F.Coo.from_numpy(w.dims, idx, val)
    import torch
    ft = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        h = F.fcoo_build(coo, mode, blocked=True)
        out = torch.full((w.dims[mode], R), float("nan"), device="cuda")
        F.fcoo_mttkrp(h, ft, R, out)
        torch.cuda.synchronize()
        M, D = oracle.mttkrp(w.dims, idx, val, mode, fs, nthreads=os.cpu_count() or 8)
        assert_parity(out.cpu().numpy(), M, D, what=f"nell2 blocked mode={mode} R={R}")
        h.destroy()
