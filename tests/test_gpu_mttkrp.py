"""GPU parity of fcoo_mttkrp (through the C ABI) against the fp64 oracle, element by element,
normalised by the per-element sum of |contributions| (tolerance 1e-4, north_star)."""
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


def _run(F, dims, idx, val, mode, factors_np, R, T=256, shards=1):
    import torch
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, tile_nnz=T)
    fs = [torch.from_numpy(f).cuda() for f in factors_np]
    out = torch.full((dims[mode], R), float("nan"), device="cuda")
    if shards == 1:
        F.fcoo_mttkrp(h, fs, R, out)
    else:  # fake multi-rank: shards run one after another, partials summed on device
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


def _check(F, dims, idx, val, mode, R, T=256, signed=False, shards=1, seed=5):
    fs = gen.factors(dims, R, seed, signed=signed)
    got = _run(F, dims, idx, val, mode, fs, R, T, shards)
    M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
    return assert_parity(got, M, D, what=f"dims={dims} mode={mode} R={R} T={T} shards={shards}")


def test_tiny_config_all_modes(F):
    """BASELINE configs[0]: 50x40x30, 1000 nnz, R=8, all modes."""
    w = gen.WORKLOADS["tiny"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        _check(F, w.dims, idx, val, mode, 8, T=32)
        _check(F, w.dims, idx, val, mode, 8, T=256, signed=True)


@pytest.mark.parametrize("R", [1, 3, 4, 8, 16, 32, 64, 100, 128, 200, 256])
def test_ranks(F, R):
    dims = (300, 200, 500)
    idx, val = gen.coo(dims, 30000, (0.5, 0.5, 0.5), 23)
    for mode in range(3):
        _check(F, dims, idx, val, mode, R, T=64, signed=True)


@pytest.mark.parametrize("dims", [(40, 50, 30, 20), (12, 10, 8, 6, 5), (3000, 7), (9, 8, 7, 6, 5, 4, 3)])
def test_orders(F, dims):
    nnz = min(20000, int(np.prod(dims) * 0.3))
    idx, val = gen.coo(dims, nnz, None, 29)
    for mode in range(len(dims)):
        for R in (16, 5):
            _check(F, dims, idx, val, mode, R, T=32, signed=True)


@pytest.mark.parametrize("T", [32, 96, 256, 1024, 4096])
def test_tile_sizes_and_ragged_tail(F, T):
    dims = (700, 500, 900)
    idx, val = gen.coo(dims, 12345, (0.7, 0.3, 0.5), 31)
    for mode in range(3):
        _check(F, dims, idx, val, mode, 32, T=T)


def test_adversarial_segments(F):
    n = 20000
    v = gen.uniform((n,), 3, 0) + 0.5
    # one giant segment spanning many tiles
    giant = np.stack([np.zeros(n, np.uint32), (np.arange(n) % 200).astype(np.uint32),
                      (np.arange(n) // 200).astype(np.uint32)])
    _check(F, (3, 200, 100), giant, v, 0, 32, T=32)
    # all singleton segments (every nonzero its own row), plus empty rows
    single = np.stack([(np.arange(n) * 2).astype(np.uint32), (np.arange(n) % 13).astype(np.uint32),
                       (np.arange(n) % 5).astype(np.uint32)])
    _check(F, (2 * n + 5, 13, 5), single, v, 0, 32, T=32)
    # segment heads exactly on tile boundaries: every slice has exactly 64 nonzeros, T = 64
    blk = np.stack([(np.arange(n) // 64).astype(np.uint32), (np.arange(n) % 64).astype(np.uint32),
                    np.zeros(n, np.uint32)])
    _check(F, (n // 64 + 1, 64, 1), blk, v, 0, 16, T=64)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_fake_multirank_shards(F, shards):
    """Shard-boundary logic without NCCL: tile-aligned shards summed equal the whole."""
    dims = (100, 900, 800)
    idx, val = gen.coo(dims, 50000, (1.0, 0.5, 0.5), 37)
    for mode in range(3):
        _check(F, dims, idx, val, mode, 32, T=64, shards=shards)


def test_build_sharded_single_rank_comm(F):
    """fcoo_build_sharded with a 1-rank communicator: shard 0 of 1 is the whole
    tensor, no collective runs, and the result equals the oracle; the handle reports the shard."""
    import torch
    dims = (300, 200, 100)
    idx, val = gen.coo(dims, 20000, (0.5, 0.5, 0.5), 41)
    R = 16
    fs = gen.factors(dims, R, 3, signed=True)
    comm = F.fcoo_comm_init(0, 1, F.fcoo_comm_unique_id())
    coo = F.Coo.from_numpy(dims, idx, val)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        h = F.fcoo_build_sharded(coo, mode, comm, tile_nnz=64)
        assert (h.info.shard, h.info.nshards, h.info.tile_begin, h.info.tile_end) == (0, 1, 0, h.info.ntiles)
        out = torch.full((dims[mode], R), float("nan"), device="cuda")
        F.fcoo_mttkrp(h, ft, R, out)
        torch.cuda.synchronize()
        M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
        assert_parity(out.cpu().numpy(), M, D, what=f"build_sharded mode={mode}")
        h.destroy()
    comm.destroy()


def test_owned_rows_bitwise_repeatable(F):
    """Stores + boundary-only atomics: a row whose segment starts and ends inside
    one tile is written by one plain store of one lane-group's fixed-order sum, so it is bitwise
    identical across calls; only rows of tile-crossing segments (red.add, arrival order) may differ
    in the last bits.  Both runs also match the oracle."""
    import torch
    dims = (2000, 300, 400)
    idx, val = gen.coo(dims, 60000, None, 41)
    fs = gen.factors(dims, 32, 42)
    T = 64
    a = _run(F, dims, idx, val, 0, fs, 32, T)
    b = _run(F, dims, idx, val, 0, fs, 32, T)
    M, D = oracle.mttkrp(dims, idx, val, 0, fs)
    assert_parity(a, M, D)
    assert_parity(b, M, D)
    # rows owned by one tile, from the exported flags: segment s = [head_s, head_{s+1})
    h = F.fcoo_build(F.Coo.from_numpy(dims, idx, val), 0, tile_nnz=T)
    ex = F.fcoo_export(h)
    nnz = val.shape[0]
    heads = np.nonzero(np.unpackbits(ex["bf"], bitorder="little")[:nnz])[0]
    ends = np.append(heads[1:], nnz) - 1
    owned = ex["seg_coord"][:, 0][(heads // T) == (ends // T)]
    h.destroy()
    assert owned.size > 100
    assert np.array_equal(a[owned].view(np.uint32), b[owned].view(np.uint32))


def test_nell2_shaped_full_size(F):
    """BASELINE configs[1] at full size (76.9M nnz), R=32, every mode, launch configuration of
    bench.py (T=2048), compared element by element with the multi-threaded oracle."""
    w = gen.WORKLOADS["nell2"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    import os
    for mode in range(3):
        fs = gen.factors(w.dims, 32, 7)
        got = _run(F, w.dims, idx, val, mode, fs, 32, 2048)
        M, D = oracle.mttkrp(w.dims, idx, val, mode, fs, nthreads=os.cpu_count() or 8)
        assert_parity(got, M, D, what=f"nell2 mode {mode}")


def test_netflix_stress_giant_slice(F):
    """Reading Q16 at scale: heavy power law (alpha 1.0/1.0/0.5), 100M nonzeros, the largest slice
    holds millions of nonzeros spread over thousands of tiles (boundary red.add on one row);
    every mode, R=32, parity per element against the multi-threaded oracle."""
    import os
    w = gen.WORKLOADS["netflix_stress"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    biggest = int(np.bincount(idx[0]).max())
    assert biggest > 1_000_000
    for mode in range(3):
        fs = gen.factors(w.dims, 32, 8)
        got = _run(F, w.dims, idx, val, mode, fs, 32, 0)
        M, D = oracle.mttkrp(w.dims, idx, val, mode, fs, nthreads=os.cpu_count() or 8)
        assert_parity(got, M, D, what=f"netflix stress mode {mode}")


def test_order4_full_size(F):
    """BASELINE configs[4] shape at full size (500K x 20K x 2K x 1K, 150M nnz), R=32, every mode,
    automatic tile, element by element against the multi-threaded oracle."""
    import os
    w = gen.WORKLOADS["order4"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(4):
        fs = gen.factors(w.dims, 32, 9)
        got = _run(F, w.dims, idx, val, mode, fs, 32, 0)
        M, D = oracle.mttkrp(w.dims, idx, val, mode, fs, nthreads=os.cpu_count() or 8)
        assert_parity(got, M, D, what=f"order4 mode {mode}")


def test_nell1_full_size_wide_keys(F):
    """Table IV nell-1 extents at full size (143.6M nnz, 69-bit build keys -> the 128-bit sort
    path), every mode, R=8 (keeps the fp64 oracle output for the 25.5M-row mode in host memory)."""
    import os
    w = gen.WORKLOADS["nell1"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        fs = gen.factors(w.dims, 8, 10)
        got = _run(F, w.dims, idx, val, mode, fs, 8, 0)
        M, D = oracle.mttkrp(w.dims, idx, val, mode, fs, nthreads=os.cpu_count() or 8)
        assert_parity(got, M, D, what=f"nell1 mode {mode}")


@pytest.mark.parametrize("T", [32, 64, 256, 2048])
def test_deterministic_flag_bitwise_and_parity(F, T):
    """FCOO_BUILD_DETERMINISTIC: tile partials of shared segments combined in tile
    order instead of red.add — repeated calls are bitwise identical (also with shards, whose
    partial rows are then summed on the host in rank order), and the result matches the oracle.
    Heavy power law so single slices span many tiles."""
    import torch
    dims = (60, 700, 500)
    idx, val = gen.coo(dims, 120000, (1.2, 0.5, 0.5), 49)
    R = 32
    fs = gen.factors(dims, R, 8, signed=True)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    coo = F.Coo.from_numpy(dims, idx, val)
    for mode in range(3):
        h = F.fcoo_build(coo, mode, tile_nnz=T, deterministic=True)
        outs = []
        for _ in range(3):
            o = torch.full((dims[mode], R), float("nan"), device="cuda")
            F.fcoo_mttkrp(h, ft, R, o)
            outs.append(o)
        torch.cuda.synchronize()
        assert all(torch.equal(outs[0], o) for o in outs[1:])
        M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
        assert_parity(outs[0].cpu().numpy(), M, D, what=f"deterministic T={T} mode={mode}")
        parts = []
        for g in range(3):
            F.fcoo_set_shard(h, g, 3)
            o = torch.full((dims[mode], R), float("nan"), device="cuda")
            F.fcoo_mttkrp(h, ft, R, o)
            parts.append(o.double())
        torch.cuda.synchronize()
        assert_parity((parts[0] + parts[1] + parts[2]).cpu().numpy(), M, D, what=f"deterministic shards T={T}")
        h.destroy()


@pytest.mark.parametrize("R", [8, 16, 5])
def test_deterministic_flag_other_paths(F, R):
    """The unstaged engine (R < 16, scalar R) and SpTTM on deterministic handles."""
    import torch
    dims = (80, 600, 400)
    idx, val = gen.coo(dims, 50000, (1.0, 0.5, 0.5), 50)
    fs = gen.factors(dims, R, 9, signed=True)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, 0, tile_nnz=64, deterministic=True)
    a = torch.empty((dims[0], R), device="cuda")
    b = torch.empty((dims[0], R), device="cuda")
    F.fcoo_mttkrp(h, ft, R, a)
    F.fcoo_mttkrp(h, ft, R, b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    M, D = oracle.mttkrp(dims, idx, val, 0, fs, nthreads=8)
    assert_parity(a.cpu().numpy(), M, D, what=f"deterministic unstaged R={R}")
    h.destroy()
    t = F.fcoo_build(coo, 1, op=F.OP_TTM, tile_nnz=64, deterministic=True)
    y1 = torch.empty((t.info.nsegs, R), device="cuda")
    y2 = torch.empty((t.info.nsegs, R), device="cuda")
    F.fcoo_ttm(t, ft[1], R, y1)
    F.fcoo_ttm(t, ft[1], R, y2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    coords, Y, Dy = oracle.ttm(dims, idx, val, 1, fs[1])
    assert_parity(y1.cpu().numpy(), Y, Dy, what=f"deterministic ttm R={R}")
    t.destroy()
