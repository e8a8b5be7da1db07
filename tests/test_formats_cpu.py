"""Matrix Market ingest (csrc/mmio.cu, xb_mm_read / xb_mm_info) on CPU: the
native parser against the reference's own parse results and error lines
(tests/golden/mm.npz, made by importing the reference), and the reference's
Matrix Market tests (tests/test_formats.py:27-163) through this package."""

import os

import numpy as np
import pytest

from conftest import golden

ACCEPTED = ["general", "symmetric", "pattern", "integer", "no_final_newline", "crlf",
            "zero_entries"]
REJECTED = ["bad_banner", "complex", "array", "blank_before_size", "bad_size", "neg_dims",
            "row_oob", "col_oob", "frac_index", "blank_body", "too_few", "too_many",
            "above_diag", "no_size", "empty"]
# the reference crashes on these under pandas 3 (bare ValueError from its
# arrow-backed string column); its own test expects the ParseError below
PANDAS3 = {"bad_token": (4, "malformed column index 'x'"),
           "bad_value": (4, "malformed value 'abc'"),
           "fields": (4, "expected 3 fields, found 2")}


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    with open(p, "w", newline="") as f:
        f.write(text)
    return str(p)


@pytest.mark.parametrize("name", ACCEPTED)
def test_parse_matches_reference(tmp_path, name):
    import paper_1907_06470_b200 as X

    g = golden("mm")
    path = _write(tmp_path, name, str(g[f"{name}_text"]))
    pool = X.BlockPool()
    mat = X.parse_matrix_market(path, pool, "m", precision=X.Precision.DOUBLE)
    assert tuple(mat.shape) == tuple(g[f"{name}_shape"])
    from paper_1907_06470_b200.pool import canonical_coo

    r, c, v = canonical_coo(mat)
    assert np.array_equal(r, g[f"{name}_r"]) and np.array_equal(c, g[f"{name}_c"])
    assert np.array_equal(v, g[f"{name}_v"])  # bitwise, duplicates summed in the same order
    info = X.read_matrix_market_info(path)
    assert [info["rows"], info["cols"], info["entries"], int(info["symmetric"])] == \
        list(g[f"{name}_info"])


@pytest.mark.parametrize("name", REJECTED + sorted(PANDAS3))
def test_rejections_match_reference(tmp_path, name):
    import paper_1907_06470_b200 as X

    g = golden("mm")
    path = _write(tmp_path, name, str(g[f"{name}_text"]))
    with pytest.raises(X.ParseError) as err:
        X.parse_matrix_market(path, X.BlockPool(), "m")
    if name in PANDAS3:
        line, msg = PANDAS3[name]
        assert err.value.line == line and str(err.value) == f"line {line}: {msg}"
    else:
        assert err.value.line == int(g[f"{name}_err_line"])
        assert str(err.value) == str(g[f"{name}_err_msg"])


def test_threads_and_chunking_do_not_change_bits(tmp_path):
    """Piece boundaries (threads) never move entries; the chunk size sets the
    reference's mirror interleaving, which changes only duplicate-sum order."""
    from paper_1907_06470_b200 import _lib

    g = golden("mm")
    path = _write(tmp_path, "g", str(g["general_text"]))
    outs = [_lib.mm_read(path, threads=t) for t in (1, 3, 8, 0)]
    for o in outs[1:]:
        for a, b in zip(o[2:5], outs[0][2:5]):
            assert np.array_equal(a, b)
    sym = _write(tmp_path, "s", str(g["symmetric_text"]))
    a = _lib.mm_read(sym, threads=4, chunk_lines=100)
    b = _lib.mm_read(sym, threads=1, chunk_lines=100)
    assert all(np.array_equal(x, y) for x, y in zip(a[2:5], b[2:5]))
    # per 100-line chunk: the chunk's 100 entries, then its mirrors
    r, c = a[2], a[3]
    k = int(np.sum(r[:100] > c[:100]))
    assert np.array_equal(r[100:100 + k], c[:100][r[:100] > c[:100]])


# -- the reference's tests (tests/test_formats.py:27-163) ------------------------

def test_parse_general_coordinates(tmp_path):
    import paper_1907_06470_b200 as X

    p = _write(tmp_path, "a", "%%MatrixMarket matrix coordinate real general\n"
                              "3 3 2\n1 1 1.5\n3 2 -2.0\n")
    mat = X.parse_matrix_market(p, X.BlockPool(), "a")
    ref = np.zeros((3, 3))
    ref[0, 0], ref[2, 1] = 1.5, -2.0
    assert np.array_equal(mat.to_array(), ref)
    assert mat.desc.nnz == 2
    assert mat.desc.density is X.Density.SPARSE


def test_parse_symmetric_expands_both_triangles(tmp_path):
    import paper_1907_06470_b200 as X

    p = _write(tmp_path, "s", "%%MatrixMarket matrix coordinate real symmetric\n"
                              "2 2 2\n1 1 4\n2 1 7\n")
    mat = X.parse_matrix_market(p, X.BlockPool(), "s")
    assert np.array_equal(mat.to_array(), [[4.0, 7.0], [7.0, 0.0]])
    assert mat.desc.nnz == 3


def test_parse_sums_duplicates_and_sorts(tmp_path):
    import paper_1907_06470_b200 as X

    p = _write(tmp_path, "d", "%%MatrixMarket matrix coordinate real general\n"
                              "2 2 3\n2 2 1.0\n1 1 2.0\n2 2 0.5\n")
    mat = X.parse_matrix_market(p, X.BlockPool(), "d")
    assert np.array_equal(mat.to_array(), [[2.0, 0.0], [0.0, 1.5]])
    assert mat.desc.nnz == 2


def test_parse_rejects_blank_line_before_size(tmp_path):
    import paper_1907_06470_b200 as X

    p = _write(tmp_path, "b", "%%MatrixMarket matrix coordinate real general\n"
                              "% a comment\n\n2 2 1\n1 2 9.0\n")
    with pytest.raises(X.ParseError) as err:
        X.parse_matrix_market(p, X.BlockPool(), "b")
    assert err.value.line == 3


def test_parse_errors_carry_line_numbers(tmp_path):
    import paper_1907_06470_b200 as X

    cases = [
        ("no banner", "1 1 1\n1 1 2.0\n", 1),
        ("bad token", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 2.0\n", 3),
        ("row out of bounds", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 2.0\n", 3),
        ("too few entries", "%%MatrixMarket matrix coordinate real general\n2 2 5\n1 1 2.0\n",
         None),
        ("bad size line", "%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 2.0\n", 2),
    ]
    for name, text, line in cases:
        p = _write(tmp_path, "bad", text)
        with pytest.raises(X.ParseError) as err:
            X.parse_matrix_market(p, X.BlockPool(), f"bad-{name}")
        if line is not None:
            assert err.value.line == line, name


def test_parse_streams_under_budget(tmp_path):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(0)
    n = 5000
    keys = np.sort(rng.choice(200 * 200, size=n, replace=False))
    rows, cols, vals = keys // 200, keys % 200, rng.standard_normal(n)
    lines = ["%%MatrixMarket matrix coordinate real general", f"200 200 {n}"]
    for i in rng.permutation(n):
        lines.append(f"{rows[i] + 1} {cols[i] + 1} {vals[i]:.17g}")
    p = _write(tmp_path, "big", "\n".join(lines) + "\n")
    mat = X.parse_matrix_market(p, X.BlockPool(), "big", precision=X.Precision.DOUBLE,
                                spill_bytes=4096, chunk_lines=256)
    ref = np.zeros((200, 200))
    ref[rows, cols] = vals
    assert np.array_equal(mat.to_array(), ref)


def test_info_reads_header_only(tmp_path):
    import paper_1907_06470_b200 as X

    p = _write(tmp_path, "h", "%%MatrixMarket matrix coordinate real general\n"
                              "1447360 1447360 5514242\n")
    info = X.read_matrix_market_info(p)
    assert (info["rows"], info["cols"], info["entries"]) == (1447360, 1447360, 5514242)
    assert not info["symmetric"]


def test_write_then_parse_is_identity(tmp_path):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(1)
    a = np.round(rng.standard_normal((30, 20)), 6)
    a[rng.random((30, 20)) > 0.2] = 0.0
    pool = X.BlockPool()
    r, c = np.nonzero(a)
    mat = X.matrix_from_coo(pool, "w", 30, 20, r, c, a[r, c], precision=X.Precision.DOUBLE)
    path = str(tmp_path / "out.mtx")
    X.write_matrix_market(path, mat)
    back = X.parse_matrix_market(path, pool, "w2", precision=X.Precision.DOUBLE)
    assert np.array_equal(back.to_array(), a)
