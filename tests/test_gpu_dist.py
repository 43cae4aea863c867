"""GPU: the row-partitioned path through the C ABI (include/fcoo.h fcoo_slice_histogram,
fcoo_bucket_rows, fcoo_set_row_shard, fcoo_build_distributed; SURVEY §8(e) owned-rows combine,
§8(f)-4 distributed build).

- the slice histogram and the destination bucketing are exact (integer work: bit-exact against
  numpy's bincount and stable argsort);
- fake ranks on one GPU: every step of fcoo_build_distributed except the NCCL transport (whose
  receive order — source rank, then the source's bucket order — is reproduced by concatenation);
  each rank's F-COO is byte-exact against the oracle build of the nonzeros of its rows, its SpMTTKRP
  output is 0 outside its rows and matches the oracle inside (normalised 1e-4), and the owned row
  ranges assembled give the full result — plain and blocked layouts, every mode, with an empty rank;
- a 1-rank NCCL communicator runs fcoo_build_distributed end to end (histogram all-reduce, count
  all-gather, own-bucket copy, build) and equals fcoo_build; an empty local chunk gives an empty handle
  whose output is all zero.  The N-rank run is in test_gpu_multirank.py (skips on one GPU).
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


def test_histogram_and_bucket_exact(F):
    dims = (500, 70, 300)
    idx, val = gen.coo(dims, 40000, (1.1, 0.3, 0.6), 91)
    coo = F.Coo.from_numpy(dims, idx, val)
    for mode in range(3):
        h = F.fcoo_slice_histogram(coo, mode).cpu().numpy().view(np.uint32)
        assert np.array_equal(h, np.bincount(idx[mode], minlength=dims[mode]))
        for n in (1, 3, 8):
            bounds = F.fcoo_row_partition(h, n)
            got, counts = F.fcoo_bucket_rows(coo, mode, bounds)
            dest = np.searchsorted(bounds, idx[mode], side="right") - 1
            order = np.argsort(dest, kind="stable")
            assert np.array_equal(counts, np.bincount(dest, minlength=n))
            assert np.array_equal(got.idx.cpu().numpy().view(np.uint32), idx[:, order])
            assert got.val.cpu().numpy().tobytes() == val[order].tobytes()


def _fake_ranks(F, dims, idx, val, mode, nranks, blocked, R=16, T=64):
    """fcoo_build_distributed's steps for nranks ranks on one GPU (chunks = draw-order slices)."""
    import torch
    nnz = val.shape[0]
    chunks = [F.Coo.from_numpy(dims, idx[:, nnz * r // nranks: nnz * (r + 1) // nranks].copy(),
                               val[nnz * r // nranks: nnz * (r + 1) // nranks].copy()) for r in range(nranks)]
    h = sum(F.fcoo_slice_histogram(c, mode).cpu().numpy().view(np.uint32).astype(np.int64) for c in chunks)
    bounds = F.fcoo_row_partition(h.astype(np.uint32), nranks)
    buckets = [F.fcoo_bucket_rows(c, mode, bounds) for c in chunks]
    fs = gen.factors(dims, R, 93, signed=True)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    M, D = oracle.mttkrp(dims, idx, val, mode, fs)
    total = np.zeros_like(M)
    empty_ranks = 0
    for k in range(nranks):
        parts_i, parts_v = [], []
        for b, counts in buckets:  # receive order: source rank, then the source's bucket order
            off = int(counts[:k].sum())
            parts_i.append(b.idx[:, off:off + int(counts[k])])
            parts_v.append(b.val[off:off + int(counts[k])])
        ri, rv = torch.cat(parts_i, dim=1).contiguous(), torch.cat(parts_v).contiguous()
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        sel = (idx[mode] >= lo) & (idx[mode] < hi)
        assert rv.shape[0] == int(sel.sum())
        if rv.shape[0] == 0:
            empty_ranks += 1
            continue
        mine = F.Coo(dims, ri, rv)
        hk = F.fcoo_build(mine, mode, tile_nnz=T, blocked=blocked, block_rows=32 if blocked else 0)
        # byte-exact against the oracle build of the rows' nonzeros (the build is a function of the set)
        ex = F.fcoo_export(hk)
        if blocked:
            ref = oracle.build_fcoo_blocked(dims, idx[:, sel].copy(), val[sel].copy(), mode, T, 32)
        else:
            ref = oracle.build_fcoo(dims, idx[:, sel].copy(), val[sel].copy(), oracle.OP_MTTKRP, mode, T)
        assert ex["bf"].tobytes() == ref.bf.tobytes() and ex["pidx"].tobytes() == ref.pidx.tobytes()
        assert ex["val"].tobytes() == ref.val.tobytes() and ex["seg_coord"].tobytes() == ref.seg_coord.tobytes()
        F.fcoo_set_row_shard(hk, k, bounds)
        assert hk.info.row_sharded == (nranks > 1) and (hk.info.row_begin, hk.info.row_end) == ((lo, hi) if nranks > 1
                                                                                               else (0, dims[mode]))
        out = torch.full((dims[mode], R), float("nan"), device="cuda")
        F.fcoo_mttkrp(hk, ft, R, out)
        got = out.cpu().numpy().astype(np.float64)
        assert np.all(got[:lo] == 0) and np.all(got[hi:] == 0), "rows outside the shard must be 0"
        total += got
        hk.destroy()
    assert_parity(total.astype(np.float32), M, D, what=f"row shards mode={mode} n={nranks} blocked={blocked}")
    return empty_ranks


@pytest.mark.parametrize("blocked", [False, True])
def test_fake_ranks_every_mode(F, blocked):
    dims = (120, 900, 300)
    idx, val = gen.coo(dims, 60000, (0.9, 0.5, 0.5), 95)
    for mode in range(3):
        for n in (2, 5):
            _fake_ranks(F, dims, idx, val, mode, n, blocked)


def test_fake_ranks_heavy_slice_leaves_rank_empty(F):
    """One slice holding most nonzeros: ranks after it own no rows (fcoo_row_partition), the others
    still assemble the exact result."""
    dims = (40, 200, 100)
    idx, val = gen.coo(dims, 20000, (3.0, 0.5, 0.5), 97)
    assert np.bincount(idx[0]).max() > 20000 / 4
    assert _fake_ranks(F, dims, idx, val, 0, 4, False) >= 1


def test_set_row_shard_checks(F):
    dims = (50, 40, 30)
    idx, val = gen.coo(dims, 3000, None, 99)
    sel = idx[0] < 20
    h = F.fcoo_build(F.Coo.from_numpy(dims, idx[:, sel].copy(), val[sel].copy()), 0, tile_nnz=32)
    with pytest.raises(F.FcooError) as e:  # rows 0..19 are not inside [25, 50)
        F.fcoo_set_row_shard(h, 1, np.array([0, 25, 50]))
    assert e.value.code == F.ERR_ARG
    with pytest.raises(F.FcooError):  # bounds must end at I_n
        F.fcoo_set_row_shard(h, 0, np.array([0, 25, 49]))
    F.fcoo_set_row_shard(h, 0, np.array([0, 25, 50]))
    with pytest.raises(F.FcooError):  # no tile shards on a row shard
        F.fcoo_set_shard(h, 0, 2)
    t = F.fcoo_build(F.Coo.from_numpy(dims, idx, val), 0, op=F.OP_TTM, tile_nnz=32)
    with pytest.raises(F.FcooError) as e:
        F.fcoo_set_row_shard(t, 0, np.array([0, 50]))
    assert e.value.code == F.ERR_SHAPE


def _one_rank_comm(F):
    return F.fcoo_comm_init(0, 1, F.fcoo_comm_unique_id())


@pytest.mark.parametrize("blocked", [False, True])
def test_distributed_build_one_rank_nccl(F, blocked):
    import torch
    dims = (300, 200, 500)
    idx, val = gen.coo(dims, 50000, (0.8, 0.5, 0.5), 101)
    coo = F.Coo.from_numpy(dims, idx, val)
    comm = _one_rank_comm(F)
    R = 32
    fs = gen.factors(dims, R, 103, signed=True)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    try:
        for mode in range(3):
            hd = F.fcoo_build_distributed(coo, mode, comm, tile_nnz=128, blocked=blocked)
            hp = F.fcoo_build(coo, mode, tile_nnz=128, blocked=blocked)
            a, b = F.fcoo_export(hd), F.fcoo_export(hp)
            for k in ("bf", "sf", "seg_base", "seg_coord", "pidx", "val"):
                assert a[k].tobytes() == b[k].tobytes(), k
            out = torch.empty((dims[mode], R), device="cuda")
            F.fcoo_mttkrp(hd, ft, R, out)
            torch.cuda.synchronize()
            M, D = oracle.mttkrp(dims, idx, val, mode, fs)
            assert_parity(out.cpu().numpy(), M, D, what=f"distributed 1-rank mode={mode}")
            hd.destroy()
            hp.destroy()
        # an empty local chunk: an empty handle, all-zero output
        empty = F.Coo(dims, torch.zeros((3, 0), dtype=torch.int32, device="cuda"),
                      torch.zeros(0, dtype=torch.float32, device="cuda"))
        he = F.fcoo_build_distributed(empty, 1, comm)
        assert he.info.nnz == 0
        out = torch.full((dims[1], R), float("nan"), device="cuda")
        F.fcoo_mttkrp(he, ft, R, out)
        assert torch.all(out == 0)
        he.destroy()
    finally:
        comm.destroy()


def test_distributed_build_rejects_keep_perm(F):
    """A permutation would index the rank's received nonzeros, not its chunk: ARG (include/fcoo.h)."""
    import ctypes

    from paper_1705_09905_b200 import fcoo as FB
    dims = (30, 20, 10)
    idx, val = gen.coo(dims, 500, None, 105)
    coo = F.Coo.from_numpy(dims, idx, val)
    comm = _one_rank_comm(F)
    try:
        opts = FB._BuildOpts(F.OP_MTTKRP, 0, FB.BUILD_KEEP_PERM, 0)
        out = ctypes.c_void_p()
        rc = F.load_library().fcoo_build_distributed(ctypes.byref(coo.c), 0, ctypes.byref(opts), comm.h, None, None,
                                                     ctypes.byref(out))
        assert rc == F.ERR_ARG and not out.value
    finally:
        comm.destroy()


def test_fake_ranks_order4_blocked(F):
    """The row-partitioned steps on a 4-order tensor (blocked handles with 3 packed words per
    nonzero), every mode, 3 fake ranks."""
    dims = (40, 30, 20, 50)
    idx, val = gen.coo(dims, 30000, (0.7, 0.3, 0.5, 0.2), 111)
    for mode in range(4):
        _fake_ranks(F, dims, idx, val, mode, 3, True)


def test_distributed_build_index_error(F):
    """A coordinate beyond its extent is reported (INDEX_RANGE) before any exchange; with N ranks the
    status is agreed across ranks before each collective step (include/fcoo.h)."""
    dims = (30, 20, 10)
    idx, val = gen.coo(dims, 500, None, 113)
    idx = idx.copy()
    idx[0, 7] = 30  # out of range in the distributed mode
    coo = F.Coo.from_numpy(dims, idx, val)
    comm = _one_rank_comm(F)
    try:
        with pytest.raises(F.FcooError) as e:
            F.fcoo_build_distributed(coo, 0, comm)
        assert e.value.code == F.ERR_INDEX_RANGE
    finally:
        comm.destroy()
