"""Matrix Market / vector interchange (csrc/mtx.cpp) against the reference's
own cases (proj/tests/test_sparse.cpp:114-229) and messages
(proj/src/sparse.cpp:140-242). Host-only entry points: no GPU needed, except
the device round trip at the end (-m gpu)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from tests import helpers as H


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _dense(rp, ci, v, n, nc):
    return sp.csr_matrix((v, ci, rp), shape=(n, nc)).toarray()


def test_explicit_diagonal_with_comment(rk, tmp_path):
    p = _write(tmp_path, "diag.mtx", "%%MatrixMarket matrix coordinate real general\n"
               "% comment line\n2 2 2\n1 1 2.0\n2 2 3.0\n")
    rp, ci, v, n, nc = rk.load_matrix_market(p)
    assert np.array_equal(_dense(rp, ci, v, n, nc), np.diag([2.0, 3.0]))


def test_symmetric_lower_triangle_expands(rk, tmp_path):
    p = _write(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
               "3 3 4\n1 1 2.0\n2 1 -1.0\n3 2 0.5\n3 3 4.0\n")
    rp, ci, v, n, nc = rk.load_matrix_market(p)
    D = _dense(rp, ci, v, n, nc)
    assert len(v) == 6 and np.array_equal(D, D.T) and D[1, 0] == -1.0 and D[0, 1] == -1.0


def test_duplicates_summed_rows_sorted_and_case_insensitive(rk, tmp_path):
    p = _write(tmp_path, "dup.mtx", "%%MatrixMarket MATRIX Coordinate REAL General\n"
               "2 3 4\n2 3 1.5\n1 2 1.0\n2 3 0.25\n1 1 -2\n")
    rp, ci, v, n, nc = rk.load_matrix_market(p)
    assert (n, nc) == (2, 3)
    assert rp.tolist() == [0, 2, 3] and ci.tolist() == [0, 1, 2] and v.tolist() == [-2.0, 1.0, 1.75]


def test_round_trip_bit_identical(rk, tmp_path):
    A = H.random_sparse(30, 0.12, 21, shift=3.7)
    p = str(tmp_path / "rt.mtx")
    rk.save_matrix_market((A.indptr, A.indices, A.data, A.shape[1]), p)
    rp, ci, v, n, nc = rk.load_matrix_market(p)
    assert (n, nc) == A.shape
    assert np.array_equal(rp, A.indptr) and np.array_equal(ci, A.indices)
    assert np.array_equal(v, A.data)  # 17 significant digits round-trip doubles


def test_empty_and_one_by_one(rk, tmp_path):
    p = str(tmp_path / "empty.mtx")
    rk.save_matrix_market((np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0)), p)
    rp, ci, v, n, nc = rk.load_matrix_market(p)
    assert n == 4 and len(v) == 0
    p1 = str(tmp_path / "one.mtx")
    rk.save_matrix_market((np.array([0, 1]), np.array([0], np.int32), np.array([3.5])), p1)
    lines = [ln for ln in open(p1).read().splitlines() if ln and ln[0] != "%"]
    assert lines == ["1 1 1", "1 1 3.5"]


@pytest.mark.parametrize("text,line,msg", [
    ("", 1, "empty file"),
    ("%%MatrixMarket matrix array real general\n1 1 1\n", 1, "only coordinate format"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n", 1, "only real field"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n", 1, "only general/symmetric"),
    ("%MatrixMarket matrix coordinate real general\n1 1 1\n", 1, "malformed MatrixMarket header"),
    ("%%MatrixMarket matrix coordinate real general\n2 x 1\n", 2, "malformed size line"),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", 2, "missing size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3, "index out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n", 3,
     "malformed coordinate line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 3,
     "entry count does not match header"),
])
def test_malformed_input_reports_the_line(rk, tmp_path, text, line, msg):
    p = _write(tmp_path, "bad.mtx", text)
    with pytest.raises(rk.ParseError) as e:
        rk.load_matrix_market(p)
    assert f"{p}:{line}: " in str(e.value) and msg in str(e.value)


def test_missing_file(rk, tmp_path):
    with pytest.raises(rk.ParseError, match="cannot open"):
        rk.load_matrix_market(str(tmp_path / "nope.mtx"))


def test_vector_round_trip_and_errors(rk, tmp_path):
    v = H.random_vector(9, 33) * 2.5
    p = str(tmp_path / "vec.txt")
    rk.save_vector(v, p)
    w = rk.load_vector(p)
    assert np.array_equal(w, v)
    q = _write(tmp_path, "c.txt", "% header\n\n1.5\n-2e-3\n")
    assert rk.load_vector(q).tolist() == [1.5, -2e-3]
    with pytest.raises(rk.ParseError, match=r":2: expected one decimal value"):
        rk.load_vector(_write(tmp_path, "b1.txt", "1.0\nfoo\n"))
    with pytest.raises(rk.ParseError, match=r":1: expected one value per line"):
        rk.load_vector(_write(tmp_path, "b2.txt", "1.0 2.0\n"))


def test_generator_problem_round_trips_through_mtx(rk, tmp_path):
    """The reference's generate -> external workflow (rkmf_bench.cpp:206-220,
    92-97): a BASELINE-shaped problem written out and read back is the same
    CSR and b bit-for-bit."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg4", 10)
    pm, pb = str(tmp_path / "p.mtx"), str(tmp_path / "p.b.txt")
    rk.save_matrix_market((P.row_ptr, P.col_idx, P.values), pm)
    rk.save_vector(P.b, pb)
    rp, ci, v, n, nc = rk.load_matrix_market(pm)
    assert np.array_equal(rp, P.row_ptr) and np.array_equal(ci, P.col_idx)
    assert np.array_equal(v, P.values) and np.array_equal(rk.load_vector(pb), P.b)


@pytest.mark.gpu
def test_device_load_save_and_solve(rk, oracle, torch, tmp_path):
    """load_matrix_market straight into HBM, solve, and the device matrix
    written back out: the same problem as the generator's."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg2", 16)
    pm = str(tmp_path / "cfg2.mtx")
    rk.save_matrix_market((P.row_ptr, P.col_idx, P.values), pm)
    A = rk.SparseMatrix.from_mtx(pm)
    assert (A.n_rows, A.nnz) == (P.n, P.nnz) and A.ndiag == 7
    rp, ci, v = A.export()
    assert np.array_equal(rp, P.row_ptr) and np.array_equal(ci, P.col_idx)
    assert np.array_equal(v, P.values)
    p2 = str(tmp_path / "back.mtx")
    A.save_mtx(p2)
    assert open(p2).read() == open(pm).read()
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    r = rk.restarted_krylov(A, P.b, rk.FunctionSpec.exp_neg(P.t),
                            rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max), S)
    A0 = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    r0 = rk.restarted_krylov(A0, P.b, rk.FunctionSpec.exp_neg(P.t),
                             rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max), S)
    assert np.array_equal(r.f_hat, r0.f_hat)
    with pytest.raises(rk.ParseError):
        rk.SparseMatrix.from_mtx(str(tmp_path / "missing.mtx"))
