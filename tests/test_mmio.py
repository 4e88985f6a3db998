"""Matrix Market ingest (reference io.py:24-81) through the native parser:
the reference's own test cases (tests/test_io.py:13-86), on the CPU."""

import numpy as np
import pytest
import scipy.sparse

import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.mmio import MatrixMarketError


def test_read_general_sums_duplicates(tmp_path):
    p = tmp_path / "a.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n% a comment\n3 3 4\n"
                 "1 1 2.5\n2 3 -1\n3 1 4e-2\n1 1 0.5\n")
    A = sg.read_matrix_market(p)
    D = A.to_scipy().toarray()
    assert D[0, 0] == 3.0 and D[1, 2] == -1.0 and D[2, 0] == 0.04
    assert not A.symmetric_expansion_applied


def test_read_symmetric_expands(tmp_path):
    p = tmp_path / "s.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2\n2 1 -1\n2 2 2\n")
    A = sg.read_matrix_market(p)
    assert np.array_equal(A.to_scipy().toarray(), np.array([[2.0, -1.0], [-1.0, 2.0]]))
    assert A.symmetric_expansion_applied


def test_read_integer_field_crlf_and_blank_tail(tmp_path):
    p = tmp_path / "i.mtx"
    p.write_bytes(b"%%MatrixMarket matrix coordinate integer general\r\n2 2 1\r\n1 2 7\r\n\n")
    assert sg.read_matrix_market(p).to_scipy().toarray()[0, 1] == 7.0


@pytest.mark.parametrize("header,body", [
    ("%%MatrixMarket matrix array real general", "2 2\n1\n2\n3\n4\n"),
    ("%%MatrixMarket matrix coordinate complex general", "2 2 1\n1 1 1 0\n"),
    ("%%MatrixMarket matrix coordinate pattern general", "2 2 1\n1 1\n"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric", "2 2 1\n2 1 1\n"),
    ("%%MatrixMarket matrix coordinate real hermitian", "2 2 1\n1 1 1\n"),
    ("not a header at all", "2 2 1\n1 1 1\n"),
    ("%%MatrixMarket matrix coordinate real general", "2 2 2\n1 1 1\n"),       # truncated
    ("%%MatrixMarket matrix coordinate real general", "2 2 1\n1 1\n"),          # 2 tokens
    ("%%MatrixMarket matrix coordinate real general", "2 2\n1 1 1\n"),          # size line
])
def test_rejects(tmp_path, header, body):
    p = tmp_path / "bad.mtx"
    p.write_text(header + "\n" + body)
    with pytest.raises(MatrixMarketError):
        sg.read_matrix_market(p)


def test_bounds_and_square(tmp_path):
    p = tmp_path / "oob.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(MatrixMarketError, match="out of bounds"):
        sg.read_matrix_market(p)
    q = tmp_path / "rect.mtx"
    q.write_text("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n")
    with pytest.raises(MatrixMarketError, match="square"):
        sg.read_matrix_market(q)
    assert issubclass(MatrixMarketError, ValueError)


def test_roundtrip_and_scipy_agreement(tmp_path):
    import scipy.io
    S = scipy.sparse.random(300, 300, density=0.02, random_state=3, format="csr")
    S = S + scipy.sparse.eye(300)
    A = sg.SparseMatrix.from_scipy(S)
    p = tmp_path / "rt.mtx"
    sg.write_matrix_market(A, p)
    B = sg.read_matrix_market(p)
    assert np.array_equal(A.to_scipy().toarray(), B.to_scipy().toarray())  # 17 digits: exact
    C = scipy.io.mmread(str(p)).tocsr()
    assert np.array_equal(C.toarray(), B.to_scipy().toarray())


@pytest.mark.parametrize("name", ["general", "symmetric", "integer"])
def test_matches_reference_parse(tmp_path, name):
    """tests/golden/mm.npz: files and the reference's own read_matrix_market
    CSR of them (oracle/make_golden.py mm_fixtures)."""
    from conftest import golden
    g = golden("mm.npz")
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(g[f"{name}_text"].tobytes())
    A = sg.read_matrix_market(p)
    assert np.array_equal(A.row_ptr, g[f"{name}_rp"])
    assert np.array_equal(A.col_idx, g[f"{name}_ci"])
    assert np.array_equal(A.values, g[f"{name}_v"])
    assert A.symmetric_expansion_applied == bool(g[f"{name}_sym"])
