"""World-size-2 CPU (gloo) tests of the multi-GPU host logic: the NCCL unique id
is broadcast through torch.distributed; tile-aligned shard ranges (fcoo_shard_range, the library's
own arithmetic) partition the sorted nonzero stream; per-rank partial MTTKRP / TTM results
summed by an all-reduce equal the single-process result.  Partials are computed by the oracle
(no GPU here); the combine is the same sum the NCCL all-reduce performs on the GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T):
    import sys
    sys.path.insert(0, ROOT)
    import gen
    import oracle
    import paper_1705_09905_b200 as P
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # 1. unique-id broadcast as comm_from_process_group does it
        obj = [P.fcoo_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
        assert isinstance(uid, bytes) and len(uid) == 128
        got = [None] * world
        dist.all_gather_object(got, uid)
        assert all(g == uid for g in got)

        # 2. sharded MTTKRP: tile-aligned ranges of the mode-n sorted stream, partials all-reduced
        dims = (40, 300, 200)
        idx, val = gen.coo(dims, 20000, (1.0, 0.5, 0.5), 77)
        fs = gen.factors(dims, 8, 78, signed=True)
        for mode in range(3):
            f = oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, mode, T)
            ntiles = (val.shape[0] + T - 1) // T
            b, e = P.fcoo_shard_range(ntiles, rank, world)
            lo, hi = b * T, min(e * T, val.shape[0])
            sel = f.perm[lo:hi]
            part, _ = oracle.mttkrp(dims, idx[:, sel].copy(), val[sel].copy(), mode, fs)
            t = torch.from_numpy(part)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            full, D = oracle.mttkrp(dims, idx, val, mode, fs)
            err = np.abs(t.numpy() - full) / np.where(D > 0, D, 1)
            assert err.max() <= 1e-12, (mode, err.max())
            # the shards cover the stream exactly once
            cov = torch.tensor([hi - lo], dtype=torch.int64)
            dist.all_reduce(cov)
            assert int(cov) == val.shape[0]

        # 3. sharded SpTTM: fibre (segment) rows summed across ranks
        U = gen.uniform((dims[1], 4), 79, 0, signed=True)
        f = oracle.build_fcoo(dims, idx, val, oracle.OP_TTM, 1, T)
        coords, Y, D = oracle.ttm(dims, idx, val, 1, U)
        ntiles = (val.shape[0] + T - 1) // T
        b, e = P.fcoo_shard_range(ntiles, rank, world)
        lo, hi = b * T, min(e * T, val.shape[0])
        sel = f.perm[lo:hi]
        c2, Y2, _ = oracle.ttm(dims, idx[:, sel].copy(), val[sel].copy(), 1, U)
        full = np.zeros_like(Y)
        pos = {tuple(c): k for k, c in enumerate(coords.tolist())}
        for k, c in enumerate(c2.tolist()):
            full[pos[tuple(c)]] += Y2[k]
        t = torch.from_numpy(full)
        dist.all_reduce(t)
        assert np.allclose(t.numpy(), Y, rtol=1e-12, atol=1e-14)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T", [32, 256])
def test_two_rank_gloo_shard_and_combine(T):
    mp.spawn(_worker, args=(2, _free_port(), T), nprocs=2, join=True)


def test_shard_ranges_partition():
    import paper_1705_09905_b200 as P
    for ntiles in (0, 1, 7, 100, 37541):
        for world in (1, 2, 3, 8):
            ranges = [P.fcoo_shard_range(ntiles, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == ntiles
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1 and b0 <= e0
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(P.FcooError):
        P.fcoo_shard_range(10, 2, 2)
