"""CPU tests: pin the oracle (restatement of the reference path) before trusting it.

No GPU. Mirrors the reference's own identities and tolerances
(proj/tests/test_sketch.cpp, test_sparse.cpp, test_basis.cpp, test_restart.cpp,
acceptance.cpp) plus an independent scipy check and the committed golden
fixtures (tests/golden/make_golden.py).
"""
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spl

from tests import helpers as H

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ---------------- SplitMix64 / make_sketch: bit-exact ----------------
def test_splitmix_matches_pure_python_and_golden(oracle):
    g = np.load(os.path.join(GOLD, "splitmix.npz"))
    st = [42]
    py = [H.sm64_next(st) for _ in range(64)]
    assert oracle.splitmix_stream(42, 64).tolist() == py
    assert np.array_equal(oracle.splitmix_stream(0, 64), g["stream_0"])
    assert np.array_equal(oracle.splitmix_stream(42, 64), g["stream_42"])
    der = [oracle.splitmix_derive(s, t) for s in (0, 1, 77) for t in (0, 1, 2, 1000, 2**40)]
    assert der == g["derive"].tolist()
    assert der == [H.sm64_derive(s, t) for s in (0, 1, 77) for t in (0, 1, 2, 1000, 2**40)]
    assert np.array_equal(oracle.gaussian_vector(1, 257), g["gauss_1"])


@pytest.mark.parametrize("d,n,z,s", [(40, 300, 5, 123), (24, 24, 24, 9), (60, 500, 4, 77),
                                     (30, 200, 1, 5), (120, 4096, 8, 1)])
def test_make_sketch_bitexact(oracle, d, n, z, s):
    gold = np.load(os.path.join(GOLD, "sketch.npz"))
    S = oracle.make_sketch(d, n, z, s)
    key = f"d{d}_n{n}_z{z}_s{s}"
    assert np.array_equal(S.rows, gold[key + "_rows"].astype(np.int64))
    assert np.array_equal(S.signs, gold[key + "_signs"])
    if n <= 500:  # independent pure-Python restatement
        rows, signs = H.py_make_sketch(d, n, z, s)
        assert np.array_equal(S.rows, rows) and np.array_equal(S.signs, signs)


def test_sketch_structure(oracle):  # test_sketch.cpp:30-62
    S = oracle.make_sketch(40, 300, 5, 123)
    assert abs(S.scale - 1 / np.sqrt(5)) < 1e-15
    R = S.rows.reshape(300, 5)
    assert (R >= 0).all() and (R < 40).all()
    assert all(len(set(r)) == 5 for r in R)
    assert all((np.diff(r) > 0).all() for r in R)  # sorted
    assert set(np.unique(S.signs)) <= {-1, 1}
    Sq = oracle.make_sketch(24, 24, 24, 9)
    D = H.dense_sketch(Sq.rows, Sq.signs, Sq.scale, 24, 24, 24)
    assert np.allclose(np.linalg.norm(D, axis=0), 1.0, atol=1e-14)
    a, b, c = (oracle.make_sketch(60, 500, 4, s) for s in (77, 77, 78))
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.signs, b.signs)
    assert not np.array_equal(a.rows, c.rows)


def test_make_sketch_validation(oracle):  # test_sketch.cpp:64-68
    for args in [(10, 5, 2, 0), (10, 50, 11, 0), (10, 50, 0, 0)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.make_sketch(*args)
        assert e.value.kind == "ParameterError"


def test_sketch_apply_dense_image_and_linearity(oracle):  # test_sketch.cpp:70-90
    S = oracle.make_sketch(30, 200, 1, 5)
    assert np.linalg.norm(oracle.sketch_apply(S, np.zeros(200))) == 0.0
    x = H.random_vector(200, 6)
    D = H.dense_sketch(S.rows, S.signs, S.scale, 30, 200, 1)
    want = D @ x
    assert np.linalg.norm(oracle.sketch_apply(S, x) - want) <= 1e-14 * np.linalg.norm(want)
    S = oracle.make_sketch(50, 400, 4, 15)
    x, y = H.random_vector(400, 1), H.random_vector(400, 2)
    lhs = oracle.sketch_apply(S, 2.5 * x - y)
    rhs = 2.5 * oracle.sketch_apply(S, x) - oracle.sketch_apply(S, y)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)


# ---------------- sparse core ----------------
def test_spmv_norm1_validate(oracle):  # test_sparse.cpp:43-74
    A = H.random_sparse(120, 0.05, 3)
    x = H.random_vector(120, 4)
    want = A.toarray() @ x
    assert np.linalg.norm(oracle.spmv(A, x) - want) <= 1e-14 * np.linalg.norm(want)
    assert oracle.norm1(A) == pytest.approx(np.abs(A.toarray()).sum(0).max(), rel=1e-15)
    oracle.validate(A)
    bad = A.copy()
    bad.indices[[0, 1]] = bad.indices[[1, 0]] if bad.indptr[1] - bad.indptr[0] > 1 else (0, 0)
    rp, ci, v = bad.indptr.copy(), bad.indices.copy(), bad.data.copy()
    ci[0] = 999
    with pytest.raises(oracle.OracleError) as e:
        oracle.validate((rp, ci, v, 120))
    assert e.value.kind == "ShapeError"
    v2 = A.data.copy()
    v2[3] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.validate((A.indptr, A.indices, v2, 120))
    assert e.value.kind == "NumericalError"


# ---------------- randomized Arnoldi (basis.cpp:92-142) ----------------
def residual_identity(A, dec):  # test_basis.cpp:21-29
    m = dec.m
    AW = A.toarray() @ dec.W[:, :m]
    WR = dec.W @ dec.Rbar
    import scipy.sparse as sp  # noqa
    n1 = np.abs(A.toarray()).sum(0).max()
    return np.linalg.norm(AW - WR) / (n1 * max(1.0, np.linalg.norm(dec.W)))


def test_rgs_identities_50_instances(oracle):  # test_basis.cpp:89-111
    for seed in range(50):
        n, m = 40, 12
        A = H.random_sparse(n, 0.15, seed + 100)
        b = H.random_vector(n, seed + 500)
        S = oracle.make_sketch(2 * m + 2, n, 4, seed)
        dec = oracle.arnoldi_decomp(A, b, m, S)
        assert residual_identity(A, dec) <= 1e-12
        U = dec.U
        assert np.abs(U.T @ U - np.eye(U.shape[1])).max() <= 1e-8
        D = H.dense_sketch(S.rows, S.signs, S.scale, S.d, n, S.zeta)
        assert np.abs(U - D @ dec.W).max() <= 1e-12
        full = oracle.arnoldi_decomp(A, b, m)
        assert residual_identity(A, full) <= 1e-12
        assert np.abs(full.W.T @ full.W - np.eye(m + 1)).max() <= 1e-10


def test_rgs_counters_and_breakdown(oracle):  # test_basis.cpp:230-254, 160-168
    n, m = 80, 17
    A = H.random_sparse(n, 0.1, 31)
    b = H.random_vector(n, 32)
    S = oracle.make_sketch(3 * m, n, 4, 33)
    dec = oracle.arnoldi_decomp(A, b, m, S)
    assert dec.counters == dict(matvecs=m, dot_n=0, dot_d=m * (m + 1) // 2, basis_updates=m,
                                peak_basis_cols=m + 1)
    import scipy.sparse as sp
    D = sp.diags([2.5, 1.0, 3.0, 4.0]).tocsr()
    e0 = np.array([2.0, 0, 0, 0])
    rows, signs = np.arange(4, dtype=np.int64), np.ones(4, np.int8)
    Sid = oracle.Sketch(4, 4, 1, 0, rows, signs, 1.0)
    dec = oracle.arnoldi_decomp(D, e0, 3, Sid)
    assert dec.breakdown_at == 1 and abs(dec.Rbar[0, 0] - 2.5) < 1e-14


def test_identity_sketch_reproduces_classical(oracle):  # test_basis.cpp:170-179
    A = H.random_sparse(60, 0.15, 21)
    b = H.random_vector(60, 22)
    Sid = oracle.Sketch(60, 60, 1, 0, np.arange(60, dtype=np.int64), np.ones(60, np.int8), 1.0)
    cl = oracle.arnoldi_decomp(A, b, 15)
    rd = oracle.arnoldi_decomp(A, b, 15, Sid)
    assert np.abs(np.abs(rd.W) - np.abs(cl.W)).max() <= 1e-8
    assert rd.start_norm == pytest.approx(np.linalg.norm(b), rel=1e-15)


# ---------------- dense f (densefun.cpp:119-157) ----------------
def test_expm_against_scipy(oracle):  # test_densefun.cpp:69-103 tolerance 1e-10
    rng = np.random.default_rng(5)
    for n, scale in [(1, 1.0), (7, 0.1), (20, 3.0), (40, 30.0)]:
        X = rng.standard_normal((n, n)) * scale / np.sqrt(n)
        F = oracle.funm(X, oracle.KIND_EXP_NEG, 0.7)
        E = sla.expm(-0.7 * X)
        assert np.linalg.norm(F - E) <= 1e-10 * max(1.0, np.linalg.norm(E))


def test_inv_sqrt_dense(oracle):
    rng = np.random.default_rng(6)
    Q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    X = Q @ np.diag(np.logspace(-3, 3, 30)) @ Q.T + 0.05 * rng.standard_normal((30, 30)) * 1e-3
    F = oracle.funm(X, oracle.KIND_INV_SQRT, 1.0)
    E = np.linalg.inv(sla.sqrtm(X)).real
    assert np.linalg.norm(F - E) <= 1e-9 * np.linalg.norm(E)


# ---------------- restarted_krylov (restart.cpp:27-122) ----------------
def _manual_two_path(oracle, A, b, t, m, k_max, S):
    """Update form vs the full alpha * W_big f(R) e1 (test_restart.cpp:44-64)."""
    n = A.shape[0]
    f = np.zeros(n)
    start = b.copy()
    R = np.zeros((0, 0))
    Wbig = np.zeros((n, 0))
    coupling, alpha, worst = 0.0, None, 0.0
    for k in range(1, k_max + 1):
        dec = oracle.arnoldi_decomp(A, start, m, S)
        mk = dec.m
        if k == 1:
            alpha = dec.start_norm
        M = R.shape[0]
        G = np.zeros((M + mk, M + mk))
        G[:M, :M] = R
        if M:
            G[M, M - 1] = coupling * dec.start_norm
        G[M:, M:] = dec.Rbar[:mk, :mk]
        R = G
        F = oracle.funm(R, oracle.KIND_EXP_NEG, t)
        y = alpha * (dec.W[:, :mk] @ F[M:, 0])
        f += y
        Wbig = np.hstack([Wbig, dec.W[:, :mk]])
        full = alpha * (Wbig @ F[:, 0])
        worst = max(worst, np.linalg.norm(full - f) / np.linalg.norm(f))
        if dec.breakdown_at:
            break
        coupling = dec.Rbar[mk, mk - 1]
        start = dec.W[:, mk].copy()
    return f, R, worst


def test_two_path_identity_and_restart_agree(oracle):  # test_restart.cpp:114-129
    A = H.random_spd_tridiag(200, 1.0, 9.0, 7)
    b = H.random_vector(200, 8)
    S = oracle.make_sketch(64, 200, 4, 11)
    f, R, worst = _manual_two_path(oracle, A, b, 1.0, 4, 4, S)
    assert worst <= 1e-11
    res = oracle.restarted_krylov(A, b, oracle.KIND_EXP_NEG, 1.0, m_r=4, tol=1e-30, k_max=4, S=S,
                                  want_R=True)
    assert res.cycles == 4
    assert np.linalg.norm(res.f_hat - f) <= 1e-13 * np.linalg.norm(f)
    assert np.array_equal(res.R_accum, R)
    C = H.conv_diff_2d(12, 12, 0.01, 1.0, 0.5)
    S2 = oracle.make_sketch(64, C.shape[0], 4, 12)
    _, R2, worst = _manual_two_path(oracle, C, H.random_vector(C.shape[0], 1), 1.0, 8, 4, S2)
    assert worst <= 1e-11
    m = 8  # block pattern (test_restart.cpp:131-164)
    for i in range(R2.shape[0]):
        for j in range(R2.shape[1]):
            bi, bj = i // m, j // m
            in_blk = bi == bj and (i % m) <= (j % m) + 1
            coup = bi == bj + 1 and i % m == 0 and j % m == m - 1
            if not (in_blk or coup):
                assert R2[i, j] == 0.0
    for k in range(1, 4):
        assert R2[k * m, k * m - 1] != 0.0


def test_restart_converges_to_exact(oracle):  # test_restart.cpp:166-207
    n = 200
    A = H.random_spd_tridiag(n, 1.0, 9.0, 7)
    b = H.random_vector(n, 8)
    exact = sla.expm(-A.toarray()) @ b
    S = oracle.make_sketch(160, n, 4, 9)
    res = oracle.restarted_krylov(A, b, oracle.KIND_EXP_NEG, 1.0, m_r=10, tol=1e-12, k_max=50,
                                  S=S, reference=exact)
    assert res.converged and res.cycles <= 10
    assert np.linalg.norm(res.f_hat - exact) <= 1e-11 * np.linalg.norm(exact)
    assert res.counters["peak_basis_cols"] == 11
    for h in res.history:
        assert h["total_matvecs"] == h["cycle"] * 10
        assert h["alpha_dev"] <= 0.5
    assert res.history[-1]["update_norm"] <= 1e-12
    assert res.history[-1]["error_vs_reference"] == pytest.approx(
        np.linalg.norm(res.f_hat - exact) / np.linalg.norm(exact), rel=1e-12)


def test_restart_kmax_budget_and_validation(oracle):  # test_restart.cpp:209-277
    A = H.random_spd_tridiag(120, 1.0, 9.0, 31)
    b = H.random_vector(120, 32)
    S = oracle.make_sketch(40, 120, 4, 1)
    r = oracle.restarted_krylov(A, b, 0, 1.0, m_r=10, tol=1e-30, k_max=3, S=S)
    assert r.cycles == 3 and not r.converged and r.total_m == 30
    r = oracle.restarted_krylov(A, b, 0, 1.0, m_r=10, tol=1e-30, k_max=50, budget_total_m=25, S=S)
    assert r.cycles == 2 and r.total_m == 20 and not r.converged
    for kw in [dict(m_r=0), dict(k_max=0), dict(tol=0.0), dict(m_r=10, budget_total_m=5)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.restarted_krylov(A, b, 0, 1.0, S=S, **kw)
        assert e.value.kind == "ParameterError"


def test_divergence_guard(oracle):  # test_restart.cpp:231-246
    C = H.conv_diff_2d(60, 60, 0.001, 10.0, 0.0)
    b = H.random_vector(C.shape[0], 1)
    S = oracle.make_sketch(6, C.shape[0], 1, 3)
    with pytest.raises(oracle.OracleError) as e:
        oracle.restarted_krylov(C, b, 0, 10.0 / oracle.norm1(C), m_r=5, tol=1e-12, k_max=60, S=S)
    assert str(e.value).startswith("restart divergence")


def test_cfg1_oracle_matches_scipy(oracle):
    """cfg1 (2D 5-pt 256^2) end to end vs an independent scipy expm_multiply."""
    import paper_2503_22631_b200.configs as cfgs
    P = cfgs.build("cfg1")
    S = oracle.make_sketch(P.d, P.n, P.zeta, cfgs.SKETCH_SEED)
    r = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, 0, P.t, m_r=P.m,
                                tol=P.tol, k_max=P.k_max, S=S)
    ex = spl.expm_multiply(-P.t * P.scipy(), P.b)
    assert r.converged and r.cycles == 3
    assert np.linalg.norm(r.f_hat - ex) <= 1e-9 * np.linalg.norm(ex)


def test_restart_golden_histories(oracle):
    import paper_2503_22631_b200.configs as cfgs
    g = np.load(os.path.join(GOLD, "restart.npz"))
    for name, N in [("cfg1", 32), ("cfg2", 12), ("cfg4", 10)]:
        P = cfgs.build(name, N)
        S = oracle.make_sketch(P.d, P.n, P.zeta, cfgs.SKETCH_SEED)
        r = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, 0, P.t, m_r=P.m,
                                    tol=P.tol, k_max=P.k_max, S=S)
        key = f"{name}_N{N}"
        assert [r.cycles, r.total_m, int(r.converged)] == g[key + "_meta"].tolist()
        assert np.allclose(r.f_hat, g[key + "_f"], rtol=0, atol=1e-12 * np.abs(g[key + "_f"]).max())
        ex = spl.expm_multiply(-P.t * P.scipy(), P.b)
        assert np.linalg.norm(r.f_hat - ex) <= 1e-7 * np.linalg.norm(ex) + 1e-12 * np.linalg.norm(P.b)


def test_inv_sqrt_restart_small(oracle):
    """InvSqrt (BASELINE cfg3 kind, not in the reference) on a small Dirichlet Q1 case."""
    import paper_2503_22631_b200 as rk
    rp, ci, v = rk.gen_q1_hex(8, True, 1, True)
    import scipy.sparse as sp
    n = len(rp) - 1
    A = sp.csr_matrix((v, ci, rp), shape=(n, n))
    b = rk.gen_gaussian(1, n)
    S = oracle.make_sketch(4 * 10, n, 8, 1)
    r = oracle.restarted_krylov((rp, ci, v), b, oracle.KIND_INV_SQRT, 1.0, m_r=10,
                                tol=1e-10 * np.linalg.norm(b), k_max=200, S=S)
    w, V = np.linalg.eigh(A.toarray())
    ex = V @ ((V.T @ b) / np.sqrt(w))
    assert r.converged
    assert np.linalg.norm(r.f_hat - ex) <= 1e-8 * np.linalg.norm(ex)
