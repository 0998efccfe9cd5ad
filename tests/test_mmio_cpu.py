"""CPU tests of the matrix store ingest: the host half of the
Matrix Market reader (parallel parse + the reference's line-ordered acceptance
rules) and the writer, against the reference's own read_matrix_market_file /
write_matrix_market_file (src/matrix_market.cpp) compiled in oracle/_ref.
Duplicate detection runs on the device and is covered in test_gpu_parity.py."""
import os

import numpy as np
import pytest

import oracle
import paper_1602_06621_b200 as eq

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference sources absent")

HDR = "%%MatrixMarket matrix coordinate real general\n"
AHDR = "%%MatrixMarket matrix array real general\n"


def _coo_to_csr(m, rows, cols, vals):
    order = np.lexsort((cols, rows))
    r, c, v = rows[order], cols[order], vals[order]
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp), c.astype(np.int32), v


def _write(tmp_path, name, text, newline="\n"):
    p = tmp_path / name
    p.write_bytes(text.replace("\n", newline).encode())
    return str(p)


def _random_sparse_text(rng, m, n, nnz, comments=True):
    flat = rng.choice(m * n, size=nnz, replace=False)
    rows, cols = flat // n, flat % n
    vals = rng.standard_normal(nnz) * np.exp(3 * rng.standard_normal(nnz))
    lines = [HDR, "% a comment\n", "\n", f"{m} {n} {nnz}\n"]
    for k in range(nnz):
        if comments and k % 97 == 5:
            lines.append("% interleaved comment\n")
        if comments and k % 131 == 7:
            lines.append("   \t \n")
        lines.append(f"{rows[k] + 1}  {cols[k] + 1}\t{float(vals[k])!r}\n")
    return "".join(lines), rows, cols, vals


@needs_ref
@pytest.mark.parametrize("newline", ["\n", "\r\n"])
def test_reader_matches_reference_reader(tmp_path, newline):
    rng = np.random.default_rng(1)
    R = oracle.ref_oracle()
    for m, n, nnz in [(7, 5, 12), (300, 200, 1500), (4000, 3000, 200_000)]:
        text, rows, cols, vals = _random_sparse_text(rng, m, n, nnz)
        path = _write(tmp_path, f"a{m}.mtx", text, newline)
        got = eq.parse_matrix_market(path)
        assert not got.dense and (got.m, got.n) == (m, n)
        assert np.array_equal(got.rows, rows) and np.array_equal(got.cols, cols)
        assert np.array_equal(got.vals, vals)
        RM, sparse = R.read_matrix_market(path)
        assert sparse
        want = RM.export()
        rp, c, v = _coo_to_csr(m, got.rows, got.cols, got.vals)
        assert np.array_equal(rp, want.row_ptr) and np.array_equal(c, want.col)
        assert np.array_equal(v, want.val)
    # dense array format, several values per line, comments between
    a = rng.standard_normal((37, 11))
    vals = a.T.ravel()  # column-major
    body = []
    for k in range(0, vals.size, 3):
        body.append(" ".join(repr(float(x)) for x in vals[k:k + 3]) + "\n")
        if k % 30 == 0:
            body.append("% c\n")
    path = _write(tmp_path, "d.mtx", AHDR + "37 11\n" + "".join(body), newline)
    got = eq.parse_matrix_market(path)
    assert got.dense and np.array_equal(got.vals, a)
    RM, sparse = R.read_matrix_market(path)
    assert not sparse and np.array_equal(RM.to_dense(), a)


ERROR_CASES = {
    "empty": "",
    "short_header": "%%MatrixMarket matrix coordinate real\n2 2 0\n",
    "not_mm": "%%Matrix matrix coordinate real general\n2 2 0\n",
    "object": "%%MatrixMarket vector coordinate real general\n2 2 0\n",
    "format": "%%MatrixMarket matrix packed real general\n2 2 0\n",
    "field": "%%MatrixMarket matrix coordinate integer general\n2 2 0\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 2 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate real symmetric\n2 2 0\n",
    "no_size": HDR + "% only\n\n%comments\n",
    "size_tokens": HDR + "2 2\n",
    "size_zero": HDR + "0 2 1\n1 1 1.0\n",
    "size_neg": HDR + "2 2 -1\n",
    "size_alpha": HDR + "2 x 1\n1 1 1.0\n",
    "entry_tokens": HDR + "2 2 2\n1 1 1.0\n2 2\n",
    "entry_malformed": HDR + "2 2 2\n1 1 1.0\n2 b 1.0\n",
    "entry_value": HDR + "2 2 2\n1 1 1.0\n2 2 1.0x\n",
    "entry_float_index": HDR + "2 2 1\n1.0 1 1.0\n",
    "range_low": HDR + "3 3 2\n1 1 1.0\n0 2 1.0\n",
    "range_high": HDR + "3 3 2\n% c\n1 1 1.0\n3 4 1.0\n",
    "eof": HDR + "3 3 3\n1 1 1.0\n% c\n2 2 2.0\n",
    "trailing": HDR + "3 3 1\n1 1 1.0\n\n2 2 2.0\n",
    "trailing_malformed": HDR + "3 3 1\n1 1 1.0\nxx\n",
    "array_size": AHDR + "2 2 4\n1\n2\n3\n4\n",
    "array_invalid": AHDR + "2 0\n",
    "array_malformed": AHDR + "2 2\n1 2\n3 q\n",
    "array_more": AHDR + "2 2\n1 2 3\n4 5\n",
    "array_trailing": AHDR + "2 2\n1 2\n3 4\n5\n",
    "array_eof": AHDR + "2 3\n1 2\n3\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(ERROR_CASES))
def test_reader_errors_match_reference(tmp_path, case):
    path = _write(tmp_path, case + ".mtx", ERROR_CASES[case])
    R = oracle.ref_oracle()
    with pytest.raises(oracle.OracleError) as want:
        R.read_matrix_market(path)
    with pytest.raises(eq.EquilRuntimeError) as got:
        eq.parse_matrix_market(path)
    assert str(got.value).split("] ", 1)[1] == str(want.value)


@needs_ref
def test_reader_error_line_numbers_in_a_later_chunk(tmp_path):
    """Errors deep in a multi-megabyte file (several parse threads) carry the
    same line number as the reference's sequential reader."""
    rng = np.random.default_rng(3)
    text, rows, cols, vals = _random_sparse_text(rng, 5000, 4000, 300_000)
    lines = text.splitlines(keepends=True)
    k = len(lines) * 3 // 4
    while lines[k].startswith("%") or not lines[k].strip():
        k += 1
    lines[k] = "12 zz 1.0\n"
    path = _write(tmp_path, "late.mtx", "".join(lines))
    R = oracle.ref_oracle()
    with pytest.raises(oracle.OracleError) as want:
        R.read_matrix_market(path)
    with pytest.raises(eq.EquilRuntimeError) as got:
        eq.parse_matrix_market(path)
    assert str(got.value).split("] ", 1)[1] == str(want.value)
    assert f"line {k + 1}:" in str(want.value)


@needs_ref
def test_writer_bytes_equal_reference_writer(tmp_path):
    rng = np.random.default_rng(4)
    R = oracle.ref_oracle()
    m, n = 500, 300
    mask = rng.random((m, n)) < 0.05
    vals = rng.standard_normal(mask.sum()) * np.exp(5 * rng.standard_normal(mask.sum()))
    vals[:3] = [0.1, -0.0, 1e-310]  # shortest round trip, negative zero, subnormal
    rp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
    A = oracle.CsrArrays(m, n, rp, np.nonzero(mask)[1].astype(np.int32), vals)
    ours, ref = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    eq.write_matrix_market_csr(str(ours), m, n, A.row_ptr, A.col, A.val)
    R.matrix(A).write_matrix_market(str(ref))
    assert ours.read_bytes() == ref.read_bytes()
    back = eq.parse_matrix_market(str(ours))  # read-after-write is bit for bit
    assert np.array_equal(back.vals, A.val)
    D = rng.standard_normal((23, 17))
    eq.write_matrix_market_dense(str(ours), D)
    R.matrix(oracle.CsrArrays(23, 17, dense=D)).write_matrix_market(str(ref))
    assert ours.read_bytes() == ref.read_bytes()
    assert np.array_equal(eq.parse_matrix_market(str(ours)).vals, D)


def test_reader_missing_file():
    with pytest.raises(eq.EquilRuntimeError, match="cannot open"):
        eq.parse_matrix_market("/nonexistent/x.mtx")
