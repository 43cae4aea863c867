"""CPU tests of the row-partitioned multi-GPU path (SURVEY §8(e) owned-rows alternative, §8(f)-4
distributed build; include/fcoo.h fcoo_row_partition / fcoo_build_distributed):

- fcoo_row_partition (the library's host arithmetic) against its stated definition and the balance
  it guarantees;
- a world-size-2 gloo run of the whole scheme with the oracle doing the per-rank compute: each rank
  starts from its own chunk of the nonzeros, the slice histograms are all-reduced, the library picks
  the row bounds, the chunks are bucketed by destination and exchanged (all-to-all), each rank
  computes the MTTKRP of the rows it owns, and an all-gather of the owned row ranges reproduces the
  single-process result for every mode — no row is partial on two ranks (slices never cross).
"""
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


def _check_partition(h, nranks, bounds):
    h = np.asarray(h, np.int64)
    I, nnz = h.shape[0], int(h.sum())
    pre = np.concatenate([[0], np.cumsum(h)])
    assert bounds[0] == 0 and bounds[-1] == I and np.all(np.diff(bounds) >= 0)
    for k in range(1, nranks):
        target = -(-k * nnz // nranks)  # ceil(k nnz / nranks)
        b = int(bounds[k])
        assert pre[b] >= target or b == I
        assert b == 0 or pre[b - 1] < target  # the smallest such row
    loads = [int(pre[bounds[k + 1]] - pre[bounds[k]]) for k in range(nranks)]
    assert sum(loads) == nnz
    assert max(loads) <= -(-nnz // nranks) + int(h.max())  # balanced up to one slice


def test_row_partition_definition():
    import gen
    import paper_1705_09905_b200 as P
    rng = np.random.default_rng(5)
    cases = [np.array([5, 0, 3, 10, 1, 1, 0, 4]), np.zeros(7, np.int64), np.ones(1000, np.int64),
             rng.zipf(1.5, 3000).clip(max=10 ** 6), np.bincount(gen.coo((500, 40, 30), 20000, (1.0, 0, 0), 3)[0][0],
                                                               minlength=500)]
    for h in cases:
        for n in (1, 2, 3, 7, 8, 64):
            _check_partition(h, n, P.fcoo_row_partition(h, n))
    # one slice heavier than nnz / nranks: ranks after it may own no rows
    assert list(P.fcoo_row_partition(np.array([1, 100, 1, 1]), 4)) == [0, 2, 2, 2, 4]
    with pytest.raises(P.FcooError):
        P.fcoo_row_partition(np.array([], np.uint32), 2)


def _worker(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    import gen
    import oracle
    import paper_1705_09905_b200 as P
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        dims = (60, 300, 200)
        idx, val = gen.coo(dims, 20000, (1.2, 0.5, 0.5), 81)
        fs = gen.factors(dims, 8, 82, signed=True)
        nnz = val.shape[0]
        lo, hi = nnz * rank // world, nnz * (rank + 1) // world  # this rank's input chunk
        my_idx, my_val = idx[:, lo:hi], val[lo:hi]
        for mode in range(3):
            # 1. global slice histogram (the NCCL all-reduce of fcoo_build_distributed)
            h = torch.from_numpy(np.bincount(my_idx[mode], minlength=dims[mode]).astype(np.int64))
            dist.all_reduce(h)
            bounds = P.fcoo_row_partition(h.numpy().astype(np.uint32), world)
            # 2. bucket by destination (stable) and exchange (the grouped ncclSend/ncclRecv)
            dest = np.searchsorted(bounds, my_idx[mode], side="right") - 1
            order = np.argsort(dest, kind="stable")
            counts = np.bincount(dest, minlength=world)
            send = torch.from_numpy(np.concatenate([my_idx[:, order].astype(np.int64),
                                                    my_val[order].view(np.int32)[None].astype(np.int64)]).T.copy())
            cnt_all = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(cnt_all, torch.from_numpy(counts.astype(np.int64)))
            recv_counts = [int(c[rank]) for c in cnt_all]
            recv = torch.zeros((sum(recv_counts), 4), dtype=torch.int64)
            dist.all_to_all_single(recv, send, recv_counts, [int(c) for c in counts])
            r_idx = recv[:, :3].T.numpy().astype(np.uint32).copy()
            r_val = recv[:, 3].numpy().astype(np.int32).view(np.float32).copy()
            # every received nonzero lies in this rank's rows
            assert np.all((r_idx[mode] >= bounds[rank]) & (r_idx[mode] < bounds[rank + 1]))
            # 3. owned rows complete: the local MTTKRP restricted to [b_r, b_{r+1}) is the final answer
            full, D = oracle.mttkrp(dims, idx, val, mode, fs)
            own = np.zeros_like(full)
            if r_val.shape[0]:
                part, _ = oracle.mttkrp(dims, r_idx, r_val, mode, fs)
                assert np.all(part[: bounds[rank]] == 0) and np.all(part[bounds[rank + 1]:] == 0)
                own = part
            # 4. owned-rows gather (the in-place broadcasts): every rank ends with the full output
            rows = [torch.zeros((int(bounds[k + 1] - bounds[k]), 8), dtype=torch.float64) for k in range(world)]
            _gather_owned(rows, own, bounds, rank, world)
            got = np.concatenate([r.numpy() for r in rows])
            err = np.abs(got - full) / np.where(D > 0, D, 1)
            assert err.max() <= 1e-12, (mode, err.max())
            cov = torch.tensor([r_val.shape[0]], dtype=torch.int64)
            dist.all_reduce(cov)
            assert int(cov) == nnz
    finally:
        dist.destroy_process_group()


def _gather_owned(rows, own, bounds, rank, world):
    # one broadcast per owner of its row range, as comm_gather_rows does with an NCCL group
    for k in range(world):
        if rows[k].shape[0] == 0:
            continue
        if k == rank:
            rows[k].copy_(torch.from_numpy(own[bounds[k]:bounds[k + 1]].copy()))
        dist.broadcast(rows[k], src=k)


def test_two_rank_gloo_distributed_rows():
    mp.spawn(_worker, args=(2, _free_port()), nprocs=2, join=True)
