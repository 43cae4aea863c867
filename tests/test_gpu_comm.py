"""The NCCL path of the multi-GPU combine on one GPU: a 1-rank
torch.distributed NCCL group broadcasts the library's unique id (comm_from_process_group), the
library's own NCCL communicator all-reduces through fcoo_allreduce_sum, and a sharded build over
that communicator runs SpMTTKRP.  With one rank the all-reduce is the identity; the multi-rank
arithmetic of the same code is covered by the fake-shard GPU tests and the gloo CPU tests."""
import os
import socket

import numpy as np
import pytest

import gen
import oracle
from parity import assert_parity

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def pg():
    import torch
    import torch.distributed as dist
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_allreduce_through_library_communicator(pg):
    import torch
    import paper_1705_09905_b200 as P
    comm = P.comm_from_process_group()
    assert (comm.rank, comm.nranks) == (0, 1)
    x = torch.arange(1000, dtype=torch.float32, device="cuda") * 0.5 - 7.0
    ref = x.clone()
    P.fcoo_allreduce_sum(comm, x)
    torch.cuda.synchronize()
    assert torch.equal(x, ref)  # sum over one rank
    comm.destroy()


def test_sharded_build_over_nccl_comm(pg):
    import torch
    import paper_1705_09905_b200 as P
    comm = P.comm_from_process_group()
    dims = (500, 300, 200)
    idx, val = gen.coo(dims, 40000, (0.5, 0.5, 0.5), 43)
    R = 32
    fs = gen.factors(dims, R, 4, signed=True)
    coo = P.Coo.from_numpy(dims, idx, val)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        h = P.fcoo_build_sharded(coo, mode, comm)
        out = torch.full((dims[mode], R), float("nan"), device="cuda")
        P.fcoo_mttkrp(h, ft, R, out)
        torch.cuda.synchronize()
        M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
        assert_parity(out.cpu().numpy(), M, D, what=f"nccl comm mode={mode}")
        h.destroy()
    comm.destroy()


def test_cp_als_with_comm_matches_without(pg):
    """cp_als given the 1-rank communicator runs the same iteration as the comm-less call (the
    boundary red.add order of the MTTKRP is not fixed, so runs agree to rounding, not bitwise)."""
    import torch
    import paper_1705_09905_b200 as P
    comm = P.comm_from_process_group()
    dims = (60, 50, 40)
    idx, val = gen.coo(dims, 8000, (0.3, 0.3, 0.3), 44)
    R = 8
    init = gen.factors(dims, R, 12)
    coo = P.Coo.from_numpy(dims, idx, val)
    a = [torch.from_numpy(f).cuda() for f in init]
    b = [torch.from_numpy(f).cuda() for f in init]
    _, ta = P.cp_als(coo, R, 5, a)
    _, tb = P.cp_als(coo, R, 5, b, comm=comm)
    torch.cuda.synchronize()
    assert np.allclose(np.asarray(ta), np.asarray(tb), rtol=0, atol=1e-7)
    for x, y in zip(a, b):
        assert torch.allclose(x, y, rtol=0, atol=1e-4)
    comm.destroy()


def _mc_buffer(P, comm, numel):
    """A multicast-bound buffer, or skip: NVLS multicast objects need the NVSwitch fabric, and a
    box that exposes one GPU without it refuses cuMulticastCreate (tools/probe_mc.py)."""
    try:
        return P.McBuffer(comm, numel)
    except P.FcooError as e:
        if "cuMulticastCreate" in str(e):
            pytest.skip(f"NVLS multicast unavailable on this box: {e}")
        raise


@pytest.mark.parametrize("R", [16, 32, 64])
def test_fused_combine_multicast_epilogue(pg, R):
    """fcoo_mttkrp_mc: the epilogue writes through an NVLS multicast address
    (multimem.st for owned segments, multimem.red.add for shared ones); on a 1-rank comm the local
    copy must equal the oracle, as fcoo_mttkrp's output does."""
    import torch
    import paper_1705_09905_b200 as P
    comm = P.comm_from_process_group()
    dims = (700, 400, 300)
    idx, val = gen.coo(dims, 60000, (0.5, 0.5, 0.5), 45)
    fs = gen.factors(dims, R, 6, signed=True)
    coo = P.Coo.from_numpy(dims, idx, val)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    buf = _mc_buffer(P, comm, max(dims) * R)
    for mode in range(3):
        h = P.fcoo_build_sharded(coo, mode, comm, tile_nnz=64)
        got = P.fcoo_mttkrp_mc(h, ft, R, buf)
        torch.cuda.synchronize()
        M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
        assert_parity(got.cpu().numpy(), M, D, what=f"multicast mode={mode} R={R}")
        ref = torch.empty((dims[mode], R), device="cuda")
        P.fcoo_mttkrp(h, ft, R, ref)
        torch.cuda.synchronize()
        assert torch.allclose(got, ref, rtol=0, atol=1e-5)
        h.destroy()
    buf.free()
    comm.destroy()


@pytest.mark.parametrize("shards", [2, 3, 7])
def test_fused_combine_shard_boundaries(pg, shards):
    """Shards run one after another through the multicast epilogue (each call zeroes the buffer):
    summed on the host they equal the whole, so rows cut by a shard boundary are red.add-ed and
    rows a shard owns are stored exactly once."""
    import torch
    import paper_1705_09905_b200 as P
    comm = P.comm_from_process_group()
    dims = (150, 900, 800)
    idx, val = gen.coo(dims, 50000, (1.0, 0.5, 0.5), 46)
    R = 32
    fs = gen.factors(dims, R, 7, signed=True)
    coo = P.Coo.from_numpy(dims, idx, val)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    buf = _mc_buffer(P, comm, max(dims) * R)
    for mode in range(3):
        h = P.fcoo_build(coo, mode, tile_nnz=64)
        acc = torch.zeros((dims[mode], R), dtype=torch.float64, device="cuda")
        for g in range(shards):
            P.fcoo_set_shard(h, g, shards, comm)
            acc += P.fcoo_mttkrp_mc(h, ft, R, buf).double()
        torch.cuda.synchronize()
        M, D = oracle.mttkrp(dims, idx, val, mode, fs, nthreads=8)
        assert_parity(acc.cpu().numpy(), M, D, what=f"multicast shards={shards} mode={mode}")
        h.destroy()
    buf.free()
    comm.destroy()


def test_fused_combine_rejects_unsupported_rank(pg):
    import torch
    import paper_1705_09905_b200 as P
    comm = P.comm_from_process_group()
    dims = (50, 40, 30)
    idx, val = gen.coo(dims, 1000, None, 47)
    coo = P.Coo.from_numpy(dims, idx, val)
    ft = [torch.from_numpy(f).cuda() for f in gen.factors(dims, 8, 1)]
    buf = _mc_buffer(P, comm, 50 * 8)
    h = P.fcoo_build_sharded(coo, 0, comm)
    with pytest.raises(P.FcooError):
        P.fcoo_mttkrp_mc(h, ft, 8, buf)  # R = 8 runs the unstaged engine: no multicast epilogue
    h.destroy()
    buf.free()
    comm.destroy()
