"""GPU parity of fcoo_ttm (SpTTM, Eq.(3)) through the C ABI against the fp64 oracle: fibre
coordinates bit-exact, fibre values within the normalised 1e-4 tolerance."""
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


def _check(F, dims, idx, val, mode, R, T=256, signed=True, shards=1):
    import torch
    U = gen.uniform((dims[mode], R), 61, mode, signed=signed)
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, op=F.OP_TTM, tile_nnz=T)
    out = torch.full((h.info.nsegs, R), float("nan"), device="cuda")
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
    ex = F.fcoo_export(h)
    got = out.cpu().numpy()
    coords, Y, D = oracle.ttm(dims, idx, val, mode, U)
    assert np.array_equal(ex["seg_coord"], coords)
    h.destroy()
    return assert_parity(got, Y, D, what=f"ttm dims={dims} mode={mode} R={R}")


def test_hand_cases(F, golden):
    import torch
    for case in golden["ttm"]:
        idx = np.array(case["coords"], np.uint32).T.copy()
        coo = F.Coo.from_numpy(case["dims"], idx, np.array(case["vals"], np.float32))
        h = F.fcoo_build(coo, case["mode"], op=F.OP_TTM, tile_nnz=32)
        U = torch.tensor(case["U"], dtype=torch.float32, device="cuda")
        out = torch.empty((h.info.nsegs, U.shape[1]), device="cuda")
        F.fcoo_ttm(h, U, U.shape[1], out)
        assert out.cpu().numpy().tolist() == case["Y"], case["cite"]
        assert F.fcoo_export(h)["seg_coord"].tolist() == case["fibers"]


@pytest.mark.parametrize("R", [1, 4, 7, 16, 32, 64])
def test_ranks_all_modes(F, R):
    dims = (60, 700, 9)
    idx, val = gen.coo(dims, 40000, None, 71)
    for mode in range(3):
        _check(F, dims, idx, val, mode, R, T=64)


def test_order4_and_shards(F):
    dims = (30, 40, 20, 10)
    idx, val = gen.coo(dims, 30000, (0.5, 0.5, 0.5, 0.5), 73)
    for mode in range(4):
        _check(F, dims, idx, val, mode, 16, T=32)
        _check(F, dims, idx, val, mode, 16, T=32, shards=3)


@pytest.mark.parametrize("T", [0, 2048])
def test_brainq_shaped_full_size(F, T):
    """BASELINE configs[3]: brainq-shaped (60 x 70K x 9, 11M nnz), SpTTM every mode, R=16, at the
    automatic tile (T = 0: the one the timed path uses) and at T = 2048."""
    w = gen.WORKLOADS["brainq"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    for mode in range(3):
        _check(F, w.dims, idx, val, mode, 16, T=T)


@pytest.mark.parametrize("R", [8, 16, 32, 64, 128])
def test_lean_kernel_shapes(F, R):
    """The specialised SpTTM kernel (fcoo_ttm.cu) for every float4 shape R = 4G, with the factor in
    shared memory (mode 0/2: 60 and 9 rows) and gathered from global memory (mode 1); T = 32 so
    fibres cross many tiles, plus tile-aligned shards."""
    dims = (60, 3000, 9)
    idx, val = gen.coo(dims, 50000, (0.3, 0.0, 0.6), 79)
    for mode in range(3):
        _check(F, dims, idx, val, mode, R, T=32)
        _check(F, dims, idx, val, mode, R, T=64, shards=3)


def test_long_and_singleton_fibres(F):
    """One fibre spanning every tile (mode 1 of a 1 x N x 1 tensor) and all-singleton fibres."""
    n = 30000
    v = gen.uniform((n,), 5, 0) + 0.5
    one = np.stack([np.zeros(n, np.uint32), np.arange(n, dtype=np.uint32), np.zeros(n, np.uint32)])
    _check(F, (1, n, 1), one, v, 1, 16, T=32, signed=False)
    _check(F, (1, n, 1), one, v, 0, 16, T=64)
