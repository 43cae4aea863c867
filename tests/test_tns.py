"""FROSTT .tns reader / writer (fcoo_tns_*, host code in libfcoo.so; no GPU needed).

Pinned against SPEC.md's load_tns / save_tns examples ("1 1 1 1.0" -> dims (1,1,1);
"2 1 3 5.0\\n1 1 1 2.0" -> dims (2,1,3); round trip reproduces indices exactly), against an
independent numpy parse of the same text, and against the error cases the spec lists (wrong arity,
non-numeric, index < 1, empty file)."""
import os

import numpy as np
import pytest

import gen

F = pytest.importorskip("paper_1705_09905_b200.fcoo")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def test_spec_examples(tmp_path):
    dims, idx, val = F.read_tns(_write(tmp_path, "a.tns", "1 1 1 1.0\n"))
    assert dims == (1, 1, 1) and idx.tolist() == [[0], [0], [0]] and val.tolist() == [1.0]
    dims, idx, val = F.read_tns(_write(tmp_path, "b.tns", "2 1 3 5.0\n1 1 1 2.0"))
    assert dims == (2, 1, 3)
    assert idx.tolist() == [[1, 0], [0, 0], [2, 0]] and val.tolist() == [5.0, 2.0]  # file order kept


def test_golden_fixture_matches_numpy_parse():
    """tests/golden/mixed.tns: comments, blank lines, tabs, CRLF, exponent/signed values.  The
    expected arrays come from numpy's own text parser (an independent implementation)."""
    path = os.path.join(GOLDEN, "mixed.tns")
    dims, idx, val = F.read_tns(path)
    rows = []
    with open(path) as fh:
        for line in fh:
            s = line.strip()
            if s and not s.startswith("#"):
                rows.append(s.split())
    ref = np.array(rows)
    ref_idx = ref[:, :-1].astype(np.int64).T - 1
    ref_val = ref[:, -1].astype(np.float64).astype(np.float32)
    assert np.array_equal(idx, ref_idx.astype(np.uint32))
    assert np.array_equal(val, ref_val)
    assert dims == tuple(int(x) for x in ref_idx.max(axis=1) + 1)


@pytest.mark.parametrize("dims,nnz", [((50, 40, 30), 100), ((300, 200, 500, 7), 200_000)])
def test_round_trip(tmp_path, dims, nnz):
    idx, val = gen.coo(dims, nnz, (0.5,) * len(dims), 31)
    val = (val - 0.5) * 3e-3  # signed, small exponents: "%.9g" must round-trip fp32 exactly
    path = str(tmp_path / "r.tns")
    F.write_tns(path, idx, val)
    d2, idx2, val2 = F.read_tns(path)
    assert np.array_equal(idx2, idx) and np.array_equal(val2, val.astype(np.float32))
    assert d2 == tuple(int(x) + 1 for x in idx.max(axis=1))
    # threads do not change the result (file > 1 MB: several chunks)
    for nt in (1, 3, 16):
        d3, idx3, val3 = F.read_tns(path, nthreads=nt)
        assert d3 == d2 and np.array_equal(idx3, idx2) and np.array_equal(val3, val2)


def test_dims_override(tmp_path):
    p = _write(tmp_path, "o.tns", "2 1 3 5.0\n1 1 1 2.0\n")
    dims, _, _ = F.read_tns(p, dims=(10, 20, 30))
    assert dims == (10, 20, 30)
    with pytest.raises(F.FcooError) as e:
        F.read_tns(p, dims=(1, 20, 30))
    assert e.value.code == F.ERR_INDEX_RANGE


@pytest.mark.parametrize("text,code", [
    ("1 1 1 1.0\n1 1 2.0\n", "ERR_IO"),            # wrong arity (too few)
    ("1 1 1 1.0\n1 1 1 1 2.0\n", "ERR_IO"),        # wrong arity (too many)
    ("1 1 1 1.0\n1 x 1 2.0\n", "ERR_IO"),          # non-numeric coordinate
    ("1 1 1 1.0\n1 2 1 abc\n", "ERR_IO"),          # non-numeric value
    ("1 1 1 1.0\n0 1 1 2.0\n", "ERR_IO"),          # index < 1
    ("1 1 1 1.0\n4294967296 1 1 2.0\n", "ERR_IO"),  # index > 2^32 - 1
    ("1 1 1 1.0\n-1 1 1 2.0\n", "ERR_IO"),         # negative index
    ("", "ERR_EMPTY"),
    ("# only a comment\n\n", "ERR_EMPTY"),
    ("1 1.0\n", "ERR_ORDER"),                       # order 1
    (" ".join(["1"] * 9) + " 1.0\n", "ERR_ORDER"),  # order 9
])
def test_errors(tmp_path, text, code):
    with pytest.raises(F.FcooError) as e:
        F.read_tns(_write(tmp_path, "e.tns", text))
    assert e.value.code == getattr(F, code)


def test_error_reports_line_number_in_any_chunk(tmp_path):
    lines = [f"{q % 97 + 1} {q % 89 + 1} {q + 1} 1.5" for q in range(200_000)]
    lines[150_001] = "3 3 oops 1.0"
    p = _write(tmp_path, "big.tns", "# header\n" + "\n".join(lines) + "\n")
    assert os.path.getsize(p) > 3 << 20
    for nt in (1, 4):
        with pytest.raises(F.FcooError) as e:
            F.read_tns(p, nthreads=nt)
        assert e.value.code == F.ERR_IO and ":150003:" in str(e.value)


def test_missing_file():
    with pytest.raises(F.FcooError) as e:
        F.read_tns("/nonexistent/x.tns")
    assert e.value.code == F.ERR_IO
