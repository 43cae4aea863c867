"""Multi-rank NCCL path on the GPUs of one node: one process per visible
GPU (torch.multiprocessing), the library's communicator built over torch.distributed, and every
rank checked against the fp64 oracle:
  - fcoo_build_sharded + fcoo_mttkrp on every mode, plain and blocked layouts: each rank processes
    its tile-aligned nnz shard, the partial outputs are summed by the library's NCCL all-reduce
    (comm_allreduce) and every rank holds the full result;
  - fcoo_build_distributed from per-rank chunks + fcoo_mttkrp with the owned-rows all-gather
    (row-partitioned handles, plain and blocked): every rank holds the full result;
  - cp_als with the comm (sharded MTTKRP, fp64 all-reduce of the last mode, replicated R x R work),
    and cp_als(dist=True) from per-rank chunks on row shards (owned-rows gathers, fp64 last mode
    gathered, |X|^2 summed over ranks): the fit trace matches the oracle and the factors are
    identical on every rank.
Skips on a box with fewer than two GPUs (this round's boxes have one; the test lights up on an
8 x B200 node)."""
import os

import numpy as np
import pytest

import gen
import oracle
from parity import assert_parity

pytestmark = pytest.mark.gpu


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    try:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
        import paper_1705_09905_b200 as F
        comm = F.comm_from_process_group()
        dims = (900, 700, 1500)
        idx, val = gen.coo(dims, 200000, (0.8, 0.5, 0.5), 123)
        coo = F.Coo.from_numpy(dims, idx, val)
        R = 32
        fs = gen.factors(dims, R, 124, signed=True)
        ft = [torch.from_numpy(f).cuda() for f in fs]
        for blocked in (False, True):
            for mode in range(3):
                h = F.fcoo_build_sharded(coo, mode, comm, tile_nnz=64, blocked=blocked)
                assert h.info.nshards == world and h.info.shard == rank
                out = torch.full((dims[mode], R), float("nan"), device="cuda")
                F.fcoo_mttkrp(h, ft, R, out)
                torch.cuda.synchronize()
                M, D = oracle.mttkrp(dims, idx, val, mode, fs)
                assert_parity(out.cpu().numpy(), M, D, what=f"rank {rank} blocked={blocked} mode {mode}")
                h.destroy()
        # distributed build (each rank passes its own draw-order chunk) + owned-rows all-gather
        nnz = val.shape[0]
        lo, hi = nnz * rank // world, nnz * (rank + 1) // world
        chunk = F.Coo.from_numpy(dims, idx[:, lo:hi].copy(), val[lo:hi].copy())
        for blocked in (False, True):
            for mode in range(3):
                h = F.fcoo_build_distributed(chunk, mode, comm, tile_nnz=64, blocked=blocked)
                assert h.info.row_sharded and h.info.row_rank == rank and h.info.row_nranks == world
                sel = (idx[mode] >= h.info.row_begin) & (idx[mode] < h.info.row_end)
                assert h.info.nnz == int(sel.sum())
                out = torch.full((dims[mode], R), float("nan"), device="cuda")
                F.fcoo_mttkrp(h, ft, R, out)
                torch.cuda.synchronize()
                M, D = oracle.mttkrp(dims, idx, val, mode, fs)
                assert_parity(out.cpu().numpy(), M, D, what=f"rank {rank} distributed blocked={blocked} mode {mode}")
                h.destroy()
        # sharded CP-ALS: fit trace vs the oracle, factors replicated bit for bit
        R2 = 8
        init = gen.factors(dims, R2, 125)
        fcp = [torch.from_numpy(f).cuda() for f in init]
        lam, trace = F.cp_als(coo, R2, 6, fcp, tile_nnz=64, comm=comm)
        torch.cuda.synchronize()
        _, _, t_o = oracle.cp_als(dims, idx, val, R2, 6, init)
        assert np.max(np.abs(np.asarray(trace) - t_o)) <= 1e-4, (trace, t_o)
        flat = torch.cat([f.flatten() for f in fcp] + [lam])
        gathered = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(gathered, flat)
        assert all(torch.equal(gathered[0], g) for g in gathered), "factors differ across ranks"
        # CP-ALS on row shards: each rank passes its chunk; same fit trace, replicated factors
        fcp2 = [torch.from_numpy(f).cuda() for f in init]
        lam2, trace2 = F.cp_als(chunk, R2, 6, fcp2, tile_nnz=64, comm=comm, dist=True)
        torch.cuda.synchronize()
        assert np.max(np.abs(np.asarray(trace2) - t_o)) <= 1e-4, (trace2, t_o)
        flat = torch.cat([f.flatten() for f in fcp2] + [lam2])
        gathered = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(gathered, flat)
        assert all(torch.equal(gathered[0], g) for g in gathered), "row-shard factors differ across ranks"
        comm.destroy()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (one NCCL rank per GPU)")
def test_multirank_sharded_mttkrp_and_cp():
    import socket

    import torch.multiprocessing as mp
    world = _ngpus()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results
