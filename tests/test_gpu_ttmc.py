"""GPU SpTTMc (fcoo_ttmc, Eq.(4)) through the C ABI against the fp64 oracle, element by element
with the normalised 1e-4 tolerance; fast (shared outer index) and generic column layouts."""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from parity import assert_parity

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def F():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_09905_b200 as F
    return F


def _run(F, dims, idx, val, mode, fs, T=0, shards=1):
    import torch
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, tile_nnz=T)
    ft = [None if (m == mode or f is None) else torch.from_numpy(np.ascontiguousarray(f, np.float32)).cuda()
          for m, f in enumerate(fs)]
    W = int(np.prod([fs[m].shape[1] for m in range(3) if m != mode]))
    out = torch.full((dims[mode], W), float("nan"), device="cuda")
    if shards == 1:
        F.fcoo_ttmc(h, ft, out)
    else:
        acc = torch.zeros_like(out)
        for g in range(shards):
            F.fcoo_set_shard(h, g, shards)
            F.fcoo_ttmc(h, ft, out)
            acc += out
        out = acc
    torch.cuda.synchronize()
    h.destroy()
    return out.cpu().numpy()


def test_worked_case(F):
    for c in json.load(open(os.path.join(HERE, "golden", "ttmc_cases.json")))["cases"]:
        idx = np.array(c["coords"], np.uint32).T.copy()
        fs = [np.zeros((1, 1), np.float32) if f is None else np.array(f, np.float32) for f in c["factors"]]
        got = _run(F, c["dims"], idx, np.array(c["vals"], np.float32), c["mode"], fs, T=32)
        assert got.tolist() == c["Y"], c["cite"]


@pytest.mark.parametrize("ranks", [(16, 16), (8, 8), (4, 4), (32, 32), (3, 5), (16, 64), (64, 16), (1, 1), (2, 16),
                                   (8, 12), (2, 48), (32, 16), (8, 16), (8, 32), (16, 8), (64, 8)])
def test_ranks_all_modes(F, ranks):
    dims = (300, 200, 250)
    idx, val = gen.coo(dims, 30000, (0.5, 0.5, 0.5), 111)
    for mode in range(3):
        rk = [0, 0, 0]
        others = [m for m in range(3) if m != mode]
        rk[others[0]], rk[others[1]] = ranks
        rk[mode] = 1
        fs = [gen.uniform((d, max(1, r)), 112, m, signed=True) for m, (d, r) in enumerate(zip(dims, rk))]
        got = _run(F, dims, idx, val, mode, fs, T=64)
        Y, D = oracle.ttmc(dims, idx, val, mode, [None if m == mode else fs[m] for m in range(3)])
        assert_parity(got, Y, D, what=f"ttmc mode={mode} ranks={ranks}")


def test_shards_and_auto_tile(F):
    dims = (100, 900, 800)
    idx, val = gen.coo(dims, 60000, (1.0, 0.5, 0.5), 113)
    fs = gen.factors(dims, 16, 114, signed=True)
    for mode in range(3):
        Y, D = oracle.ttmc(dims, idx, val, mode, [None if m == mode else fs[m] for m in range(3)])
        assert_parity(_run(F, dims, idx, val, mode, fs), Y, D, what="auto tile")
        assert_parity(_run(F, dims, idx, val, mode, fs, T=64, shards=3), Y, D, what="3 shards")


def test_errors(F):
    import torch
    dims = (10, 9, 8, 7)
    idx, val = gen.coo(dims, 200, None, 115)
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, 0)
    fs = [None] + [torch.ones((d, 4), device="cuda") for d in dims[1:]]
    with pytest.raises(F.FcooError) as e:
        F.fcoo_ttmc(h, fs, torch.empty((10, 64), device="cuda"))
    assert e.value.code == 2  # FCOO_ERR_ORDER
    dims3 = (10, 9, 8)
    idx, val = gen.coo(dims3, 200, None, 116)
    coo = F.Coo.from_numpy(dims3, idx, val)
    ht = F.fcoo_build(coo, 0, op=F.OP_TTM)
    fs = [None, torch.ones((9, 4), device="cuda"), torch.ones((8, 4), device="cuda")]
    with pytest.raises(F.FcooError) as e:
        F.fcoo_ttmc(ht, fs, torch.empty((10, 16), device="cuda"))
    assert e.value.code == 9  # FCOO_ERR_SHAPE
    hm = F.fcoo_build(coo, 0)
    big = [None, torch.ones((9, 64), device="cuda"), torch.ones((8, 32), device="cuda")]
    with pytest.raises(F.FcooError) as e:
        F.fcoo_ttmc(hm, big, torch.empty((10, 2048), device="cuda"))
    assert e.value.code == 8  # FCOO_ERR_RANK


def test_long_segment_accumulation(F):
    """One slice holding 200K nonzeros (a single segment across ~100 tiles): the tensor-core path's
    3xTF32 products and per-chunk fp32 accumulation must stay within 1e-4 over a long chain; signed
    factors exercise cancellation."""
    n = 200_000
    dims = (2, 1000, 1000)
    q = np.arange(n, dtype=np.int64)
    idx = np.stack([np.zeros(n, np.int64), q // 1000 * 5 % 1000, q % 1000]).astype(np.uint32)
    idx = np.unique(idx, axis=1)
    val = (gen.uniform((idx.shape[1],), 131, 0) + 0.5).astype(np.float32)
    for ranks in ((32, 32), (16, 16)):
        fs = [gen.uniform((dims[0], 1), 132, 0, signed=True),
              gen.uniform((dims[1], ranks[0]), 132, 1, signed=True),
              gen.uniform((dims[2], ranks[1]), 132, 2, signed=True)]
        got = _run(F, dims, idx, val, 0, fs, T=2048)
        Y, D = oracle.ttmc(dims, idx, val, 0, [None, fs[1], fs[2]])
        assert_parity(got, Y, D, what=f"long segment ranks={ranks}")


def test_nell2_full_size_sampled_rows(F):
    """SURVEY §8(f)-3 at BASELINE configs[1]'s full size (76.9M nonzeros, every mode, R=16 and 32,
    automatic tile as tools/ops_bench.py times it): an output row of Eq.(4) depends only on its own
    slice's nonzeros, so the oracle computes 24 sampled rows per mode (the heaviest slices, the
    lightest, and random ones) from those nonzeros alone; compared element by element."""
    w = gen.WORKLOADS["nell2"]
    idx, val = gen.coo(w.dims, w.nnz, w.alpha, w.seed)
    rng = np.random.default_rng(5)
    for R in (16, 32):
        fs = gen.factors(w.dims, R, 7, signed=True)
        for mode in range(3):
            got = _run(F, w.dims, idx, val, mode, fs, T=0)
            counts = np.bincount(idx[mode], minlength=w.dims[mode])
            order = np.argsort(counts, kind="stable")
            rows = np.unique(np.concatenate([order[-8:], order[:8], rng.choice(w.dims[mode], 8, replace=False)]))
            sel = np.isin(idx[mode], rows)
            sub_idx, sub_val = np.ascontiguousarray(idx[:, sel]), np.ascontiguousarray(val[sel])
            fs_m = [None if m == mode else fs[m] for m in range(3)]
            Y, D = oracle.ttmc(w.dims, sub_idx, sub_val, mode, fs_m)
            assert_parity(got[rows], Y[rows], D[rows], what=f"nell2 ttmc R={R} mode={mode} sampled rows")
