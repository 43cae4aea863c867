"""The parity tests can fail: corrupting one flag bit on the device
(fcoo_debug_flip_bit) must make the SpMTTKRP / SpTTM result miss the oracle, and flipping it back
must restore parity.  A cleared bf head merges two segments (the second one's sum lands in the
first one's row); a set sf bit makes a tile that starts inside a segment flush into the wrong row."""
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


def _fails(fn):
    try:
        fn()
    except AssertionError:
        return True
    return False


@pytest.mark.parametrize("layout", ["fcoo", "blocked"])
def test_mttkrp_flag_mutations_trip_parity(F, layout):
    import torch
    dims = (300, 200, 500)
    idx, val = gen.coo(dims, 30000, (0.5, 0.5, 0.5), 91)
    R, T = 16, 64
    fs = gen.factors(dims, R, 92, signed=True)
    ft = [torch.from_numpy(f).cuda() for f in fs]
    M, D = oracle.mttkrp(dims, idx, val, 0, fs)
    h = F.fcoo_build(F.Coo.from_numpy(dims, idx, val), 0, tile_nnz=T, blocked=(layout == "blocked"), block_rows=64)
    out = torch.empty((dims[0], R), device="cuda")

    def check():
        F.fcoo_mttkrp(h, ft, R, out)
        torch.cuda.synchronize()
        assert_parity(out.cpu().numpy(), M, D, what=f"{layout}")

    check()
    ex = F.fcoo_export(h)
    n = h.info.nstream
    bits = np.unpackbits(ex["bf"], bitorder="little")[:n]
    p = int(next(q for q in np.nonzero(bits)[0] if q % T != 0))  # a head inside a tile
    F.fcoo_debug_flip_bit(h, "bf", p)
    assert _fails(check), "a cleared bf head went unnoticed"
    F.fcoo_debug_flip_bit(h, "bf", p)
    check()
    sf = np.unpackbits(ex["sf"].view(np.uint8), bitorder="little")[: h.info.ntiles]
    t = int(np.nonzero(sf == 0)[0][0])  # a tile that starts inside a segment
    F.fcoo_debug_flip_bit(h, "sf", t)
    assert _fails(check), "a set sf bit went unnoticed"
    F.fcoo_debug_flip_bit(h, "sf", t)
    check()
    with pytest.raises(F.FcooError):  # setting a bf bit is refused (not memory-safe)
        F.fcoo_debug_flip_bit(h, "bf", int(np.nonzero(bits == 0)[0][0]))
    h.destroy()


def test_ttm_flag_mutation_trips_parity(F):
    import torch
    dims = (60, 3000, 9)
    idx, val = gen.coo(dims, 50000, None, 93)
    R = 16
    U = gen.uniform((dims[0], R), 94, 0, signed=True)
    coords, Y, D = oracle.ttm(dims, idx, val, 0, U)
    h = F.fcoo_build(F.Coo.from_numpy(dims, idx, val), 0, op=F.OP_TTM, tile_nnz=64)
    Ut = torch.from_numpy(U).cuda()
    out = torch.empty((h.info.nsegs, R), device="cuda")

    def check():
        out.fill_(0)
        F.fcoo_ttm(h, Ut, R, out)
        torch.cuda.synchronize()
        assert_parity(out.cpu().numpy(), Y, D, what="ttm")

    check()
    bits = np.unpackbits(F.fcoo_export(h)["bf"], bitorder="little")[: h.info.nstream]
    p = int(next(q for q in np.nonzero(bits)[0] if q % 64 not in (0, 63)))
    F.fcoo_debug_flip_bit(h, "bf", p)
    assert _fails(check)
    F.fcoo_debug_flip_bit(h, "bf", p)
    check()
    h.destroy()
