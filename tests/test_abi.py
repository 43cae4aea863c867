"""CPU tests of the C ABI boundary: libfcoo.so loads, exports every function include/fcoo.h
declares, and host-checkable errors return before any launch (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "fcoo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([A-Za-z_][A-Za-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("fcoo_", "cp_"))))


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for n in ("fcoo_build", "fcoo_mttkrp", "fcoo_ttm", "cp_als"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1705_09905_b200 import fcoo
    L = fcoo.load_library()
    for n in _declared_functions():
        assert hasattr(L, n), n
    assert set(fcoo.SYMBOLS) == set(_declared_functions())


def test_host_checked_errors_without_gpu():
    from paper_1705_09905_b200 import fcoo
    L = fcoo.load_library()
    dims = (ctypes.c_int64 * 1)(5)
    ptrs = (ctypes.c_void_p * 1)(None)
    coo = fcoo._Coo(1, dims, 10, ptrs, None)
    out = ctypes.c_void_p()
    opts = fcoo._BuildOpts(0, 256, 0)
    # NULL val -> ARG before anything else
    assert L.fcoo_build(ctypes.byref(coo), 0, ctypes.byref(opts), None, None, ctypes.byref(out)) == fcoo.ERR_ARG
    dims3 = (ctypes.c_int64 * 3)(5, 6, 7)
    ptrs3 = (ctypes.c_void_p * 3)(8, 8, 8)
    coo3 = fcoo._Coo(3, dims3, 10, ptrs3, 8)  # fake non-NULL pointers: never dereferenced on these paths
    bad_tile = fcoo._BuildOpts(0, 100, 0)
    assert L.fcoo_build(ctypes.byref(coo3), 0, ctypes.byref(bad_tile), None, None, ctypes.byref(out)) == fcoo.ERR_ARG
    assert L.fcoo_build(ctypes.byref(coo3), 3, ctypes.byref(opts), None, None, ctypes.byref(out)) == fcoo.ERR_MODE
    coo1 = fcoo._Coo(1, dims3, 10, ptrs3, 8)
    assert L.fcoo_build(ctypes.byref(coo1), 0, ctypes.byref(opts), None, None, ctypes.byref(out)) == fcoo.ERR_ORDER
    coo0 = fcoo._Coo(3, dims3, 0, ptrs3, 8)
    assert L.fcoo_build(ctypes.byref(coo0), 0, ctypes.byref(opts), None, None, ctypes.byref(out)) == fcoo.ERR_EMPTY
    big = (ctypes.c_int64 * 5)(*([1 << 30] * 5))  # 150 key bits > 128
    ptrs5 = (ctypes.c_void_p * 5)(8, 8, 8, 8, 8)
    cooK = fcoo._Coo(5, big, 10, ptrs5, 8)
    assert L.fcoo_build(ctypes.byref(cooK), 0, ctypes.byref(opts), None, None, ctypes.byref(out)) == fcoo.ERR_KEY_BITS
    assert L.fcoo_build_sharded(ctypes.byref(coo3), 0, ctypes.byref(opts), None, None, None,
                                ctypes.byref(out)) == fcoo.ERR_ARG  # NULL comm
    assert L.fcoo_mttkrp(None, None, 8, None, None) == fcoo.ERR_ARG
    mc = ctypes.c_void_p()
    assert L.fcoo_mc_alloc(None, 1024, ctypes.byref(mc)) == fcoo.ERR_ARG
    assert L.fcoo_mttkrp_mc(None, None, 32, None, None) == fcoo.ERR_ARG
    assert L.fcoo_mc_free(None) == fcoo.OK
    assert L.fcoo_ttm(None, None, 8, None, None) == fcoo.ERR_ARG
    assert L.fcoo_status_str(fcoo.ERR_DUPLICATE) == b"FCOO_ERR_DUPLICATE"
    assert b"tile_nnz" in L.fcoo_last_error() or len(L.fcoo_last_error()) > 0


def test_status_codes_match_oracle_numbering():
    """The oracle's enum is its own; the numbers were chosen to coincide (documented in both)."""
    import oracle
    from paper_1705_09905_b200 import fcoo
    for name in ("ERR_ARG", "ERR_ORDER", "ERR_MODE", "ERR_INDEX_RANGE", "ERR_DUPLICATE", "ERR_EMPTY"):
        assert getattr(oracle, name) == getattr(fcoo, name)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1705_09905_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "fcoo_oracle" not in txt, fn
                assert "liboracle" not in txt, fn
