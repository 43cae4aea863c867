"""GPU: the second flag level of an MTTKRP F-COO (FCOO_BUILD_FIBRE_FLAGS; Fig. 2: one
sorted stream carries the slice flags of SpMTTKRP on mode n AND the fibre flags of SpTTM on the last
product mode) through the C ABI.

- bf2 and the fibre table are byte-exact against their definition evaluated on the oracle's F-COO
  stream: a fibre head is a position whose (index tuple, product coordinates but the last) differs
  from the previous position's (the first position is a head);
- the rest of the handle is unchanged (bf, sf, product indices, values, segment tables);
- fcoo_ttm on such an MTTKRP handle computes SpTTM (Eq.(3)) on the last product mode and matches
  the fp64 oracle's SpTTM on that mode row by row (normalised 1e-4), also over tile-aligned shards;
- option and shape errors.
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


def _expected_level2(ref):
    """bf2 bits and the fibre table from the oracle's stream (definition of the second level)."""
    nnz = ref.val.shape[0]
    seg = np.cumsum(ref.bf_bits()[:nnz].astype(np.int64)) - 1          # segment of each position
    cols = [ref.seg_coord[seg, a] for a in range(ref.seg_coord.shape[1])]
    cols += [ref.pidx[a] for a in range(ref.pidx.shape[0] - 1)]          # product coords but the last
    key = np.stack(cols, axis=1)
    head = np.ones(nnz, bool)
    head[1:] = np.any(key[1:] != key[:-1], axis=1)
    return head, key[head]


def _check(F, dims, idx, val, mode, R, T, shards=1):
    import torch
    coo = F.Coo.from_numpy(dims, idx, val)
    h = F.fcoo_build(coo, mode, tile_nnz=T, fibre_flags=True)
    plain = F.fcoo_build(coo, mode, tile_nnz=T)
    i = h.info
    ref = oracle.build_fcoo(dims, idx, val, oracle.OP_MTTKRP, mode, i.tile_nnz)  # T = 0: the automatic tile
    assert i.fibre_flags and i.op == F.OP_MTTKRP
    ex, ex0 = F.fcoo_export(h), F.fcoo_export(plain)
    for k in ("bf", "sf", "seg_base", "seg_coord", "pidx", "val"):  # level 1 untouched
        assert ex[k].tobytes() == ex0[k].tobytes(), k
    head, fib = _expected_level2(ref)
    bits = np.unpackbits(ex["bf2"], bitorder="little")[: val.shape[0]].astype(bool)
    assert np.array_equal(bits, head)
    assert i.nfib == fib.shape[0] and np.array_equal(ex["fib_coord"], fib.astype(np.uint32))
    # SpTTM on the last product mode from the same stream
    m = i.prod_modes[-1]
    U = gen.uniform((dims[m], R), 63, m, signed=True)
    Ut = torch.from_numpy(U).cuda()
    out = torch.full((i.nfib, R), float("nan"), device="cuda")
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
    coords, Y, D = oracle.ttm(dims, idx, val, m, U)
    # the view's fibre columns are (mode n, prod_modes[:-1]); the oracle's are the other modes ascending
    view_modes = i.idx_modes + i.prod_modes[:-1]
    order = np.argsort(view_modes)
    pos = {tuple(c): r for r, c in enumerate(coords.tolist())}
    rows = np.array([pos[tuple(c)] for c in ex["fib_coord"][:, order].tolist()])
    got = out.cpu().numpy()
    h.destroy()
    plain.destroy()
    return assert_parity(got, Y[rows], D[rows], what=f"fibre-level ttm dims={dims} mode={mode} R={R} T={T}")


@pytest.mark.parametrize("R", [8, 16, 32, 64])
def test_fibre_level_order3(F, R):
    dims = (120, 90, 300)
    idx, val = gen.coo(dims, 40000, (0.6, 0.4, 0.5), 121)
    for mode in range(3):
        _check(F, dims, idx, val, mode, R, T=64)


def test_fibre_level_order4_and_shards(F):
    dims = (30, 40, 20, 10)
    idx, val = gen.coo(dims, 30000, (0.5, 0.5, 0.5, 0.5), 123)
    for mode in range(4):
        _check(F, dims, idx, val, mode, 16, T=32)
        _check(F, dims, idx, val, mode, 16, T=128, shards=3)


def test_fibre_level_nell2_subset(F):
    """A nell-2-shaped prefix (2M nonzeros) at the automatic tile: mode 0's last product mode is
    mode 2 (the largest), so the fibres are the (i, j) pairs of SpTTM on mode 2."""
    w = gen.WORKLOADS["nell2"]
    idx, val = gen.coo(w.dims, 2_000_000, w.alpha, w.seed)
    _check(F, w.dims, idx, val, 0, 16, T=0)


def test_fibre_level_errors(F):
    import torch
    dims = (20, 15, 10)
    idx, val = gen.coo(dims, 800, None, 125)
    coo = F.Coo.from_numpy(dims, idx, val)
    for kw in (dict(blocked=True), dict(deterministic=True), dict(op=F.OP_TTM)):
        with pytest.raises(F.FcooError) as e:
            F.fcoo_build(coo, 0, fibre_flags=True, **kw)
        assert e.value.code == F.ERR_ARG
    two = F.Coo.from_numpy((20, 15), idx[:2].copy(), val)
    with pytest.raises(F.FcooError):
        F.fcoo_build(two, 0, fibre_flags=True)
    h = F.fcoo_build(coo, 0)  # no second level: fcoo_ttm refuses an MTTKRP handle
    U = torch.zeros((dims[h.info.prod_modes[-1]], 16), device="cuda")
    with pytest.raises(F.FcooError) as e:
        F.fcoo_ttm(h, U, 16, torch.zeros((1, 16), device="cuda"))
    assert e.value.code == F.ERR_SHAPE
    h.destroy()
