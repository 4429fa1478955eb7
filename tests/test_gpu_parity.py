"""GPU parity: the sm_100a path through the C ABI against the CPU oracle.

Bars (BASELINE.json north_star / SURVEY.md §7-8): sketch bit-exact; SpMV within
1e-14 and the sketch within 1e-13 relative; restarted f(A)b within 1e-9
relative 2-norm with the cycle count within +-1; the reference's identities at
its own tolerances (test_basis.cpp, test_restart.cpp, acceptance.cpp).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from tests import helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as T
    assert T.cuda.is_available()
    return T


@pytest.fixture(autouse=True, params=["fused", "steps"])
def cycle_path(request, rk):
    """Every test twice: small matrices through the fused cycle kernel
    (cycle_small.cu, the default) and through the per-step K2/K3/K4 kernels."""
    ctx = rk.Context.default()
    ctx.set_fused_cycle(request.param == "fused")
    yield request.param
    ctx.set_fused_cycle(True)


def rel(a, b):
    a = np.asarray(a.cpu() if hasattr(a, "cpu") else a)
    b = np.asarray(b.cpu() if hasattr(b, "cpu") else b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------- K1: sketch generation, bit-exact ----------------
@pytest.mark.parametrize("d,n,z,s", [(40, 300, 5, 123), (24, 24, 24, 9), (60, 500, 4, 77),
                                     (30, 200, 1, 5), (120, 65536, 8, 1), (200, 100003, 8, 1),
                                     (800, 3600, 4, 5)])
def test_sketch_bitexact(rk, oracle, d, n, z, s):
    S = rk.make_sketch(d, n, z, s)
    rows, signs, scale = S.export()
    O = oracle.make_sketch(d, n, z, s)
    assert np.array_equal(rows, O.rows)
    assert np.array_equal(signs, O.signs)
    assert scale == O.scale


def test_sketch_validation(rk):
    for args in [(10, 5, 2, 0), (10, 50, 11, 0), (10, 50, 0, 0)]:
        with pytest.raises(rk.ParameterError):
            rk.make_sketch(*args)


# ---------------- K2: SpMV + sketch ----------------
# the sketch tile layout (quad words + tail bytes per 32-slot group, snake
# passes of 128 slots) across its shapes: one and several passes, partial
# groups, ragged last tile, long bins (zeta = d), zeta up to the device limit
@pytest.mark.parametrize("d,n,z", [(40, 300, 5), (24, 24, 24), (30, 200, 1), (120, 65613, 8),
                                   (200, 100003, 8), (800, 3600, 4), (300, 1000, 64),
                                   (129, 5000, 16), (1, 129, 1)])
def test_sketch_layout_shapes(rk, oracle, torch, d, n, z):
    S = rk.make_sketch(d, n, z, 3)
    OS = oracle.make_sketch(d, n, z, 3)
    x = np.random.default_rng(d + n).standard_normal(n)
    p = rk.sketch_apply(S, x)
    assert rel(p, oracle.sketch_apply(OS, x)) <= 1e-13
    # fused with an SpMV (identity-free: a 1D Laplacian, 3 diagonals)
    rp = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                cols.append(j)
                vals.append(v)
        rp[i + 1] = len(cols)
    ci, vv = np.array(cols, np.int32), np.array(vals)
    A = rk.SparseMatrix.from_csr(rp, ci, vv)
    zo = oracle.spmv((rp, ci, vv), x)
    z2, p2 = rk.spmv_sketch(A, S, x)
    assert rel(z2, zo) <= 1e-14
    assert rel(p2, oracle.sketch_apply(OS, zo)) <= 1e-13


@pytest.mark.parametrize("name,N", [("cfg1", 256), ("cfg2", 40), ("cfg4", 24), ("cfg3", 20)])
def test_spmv_and_sketch(rk, oracle, torch, name, N):
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    OS = oracle.make_sketch(P.d, P.n, P.zeta, 1)
    x = P.b
    z = rk.spmv(A, x)
    zo = oracle.spmv((P.row_ptr, P.col_idx, P.values), x)
    assert rel(z, zo) <= 1e-14
    p = rk.sketch_apply(S, x)
    assert rel(p, oracle.sketch_apply(OS, x)) <= 1e-13
    z2, p2 = rk.spmv_sketch(A, S, x)
    assert rel(z2, zo) <= 1e-14
    assert rel(p2, oracle.sketch_apply(OS, zo)) <= 1e-13
    assert A.norm1 == pytest.approx(oracle.norm1((P.row_ptr, P.col_idx, P.values)), rel=1e-13)


# diagonal copy (dia.cu): the fused kernel streaming [tile][diag][128] values
# must give exactly the CSR kernel's z and sketch, ragged tails included
@pytest.mark.parametrize("name,N,nd", [("cfg1", 256, 5), ("cfg2", 41, 7), ("cfg4", 23, 7)])
def test_dia_bitexact_vs_csr(rk, oracle, torch, name, N, nd):
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    assert A.ndiag == nd
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    x = P.b
    z1, p1 = rk.spmv_sketch(A, S, x)
    assert A.set_diagonal_copy(False) == 0
    z0, p0 = rk.spmv_sketch(A, S, x)
    # z bit-identical (both sum each row sequentially in column order); the
    # sketch's cross-block sums follow the grid, which differs between the
    # two streams (rounding only)
    assert torch.equal(z1, z0) and rel(p1, p0) <= 1e-14
    zo = oracle.spmv((P.row_ptr, P.col_idx, P.values), x)
    assert rel(z1, zo) <= 1e-14
    assert A.set_diagonal_copy(True) == nd


@pytest.mark.parametrize("name,N,ntup", [("cfg1", 100, 9), ("cfg2", 41, 27), ("cfg4", 23, 27),
                                         ("cfg1", 256, 9)])
def test_row_dictionary(rk, oracle, torch, name, N, ntup):
    """Constant-coefficient stencils: the diagonal copy's rows take few value
    tuples (3 x 3 boundary classes in 2D, 27 in 3D), so K2 streams one byte
    per row (dia.cu row dictionary). z is bit-identical to the copy without
    the dictionary and to the CSR kernel; whole solves (through the per-step
    kernels: the fused small-matrix cycle reads CSR) agree to rounding (the
    sketch's cross-block sums follow the grid). Dictionaries of at most 224
    doubles travel as a kernel parameter, larger ones in shared memory: rows
    scaled by 9 factors take the second path (up to 9 x the tuples)."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    assert A.ndiag > 0 and A.ntuples == ntup
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    b = torch.tensor(P.b, device="cuda")
    A.ctx.set_fused_cycle(False)
    try:
        z1, p1 = rk.spmv_sketch(A, S, P.b)
        r1 = rk.restarted_krylov(A, b, f, opts, S)
        assert A.set_row_dictionary(False) == 0 and A.ntuples == 0 and A.ndiag > 0
        z0, p0 = rk.spmv_sketch(A, S, P.b)
        r0 = rk.restarted_krylov(A, b, f, opts, S)
        assert torch.equal(z1, z0) and rel(p1, p0) <= 1e-14
        assert r1.cycles == r0.cycles and rel(r1.f_hat, r0.f_hat) <= 1e-12
        assert A.set_diagonal_copy(False) == 0 and A.ntuples == 0
        zc, _ = rk.spmv_sketch(A, S, P.b)
        assert torch.equal(z1, zc)
        assert rel(z1, oracle.spmv((P.row_ptr, P.col_idx, P.values), P.b)) <= 1e-14
        assert A.set_diagonal_copy(True) > 0 and A.ntuples == ntup
        # up to 9 x the tuples: the shared-memory dictionary (ntup * ndiag > 224)
        rows = np.repeat(np.arange(P.n), np.diff(P.row_ptr))
        v8 = P.values * (1.0 + 1e-3 * (rows % 9))
        B8 = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, v8)
        assert B8.ndiag > 0 and ntup < B8.ntuples <= 256 and B8.ntuples * B8.ndiag > 224
        zd, pd = rk.spmv_sketch(B8, S, P.b)
        rd = rk.restarted_krylov(B8, b, f, opts, S)
        assert B8.set_row_dictionary(False) == 0
        zn, pn = rk.spmv_sketch(B8, S, P.b)
        rn = rk.restarted_krylov(B8, b, f, opts, S)
        assert torch.equal(zd, zn) and rel(pd, pn) <= 1e-14
        assert rd.cycles == rn.cycles and rel(rd.f_hat, rn.f_hat) <= 1e-12
        assert rel(zd, oracle.spmv((P.row_ptr, P.col_idx, v8), P.b)) <= 1e-14
    finally:
        A.ctx.set_fused_cycle(True)
    # values that vary per row (> 256 tuples): the copy stays, no dictionary
    v = P.values * (1.0 + 1e-3 * np.random.default_rng(3).random(P.values.size))
    B = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, v)
    assert B.ndiag > 0 and B.ntuples == 0


def test_dia_eligibility(rk, torch):
    rng = np.random.default_rng(5)
    # scattered nonzeros: CSR only
    assert rk.SparseMatrix.from_scipy(H.random_sparse(2000, 0.01, 3)).ndiag == 0
    # 9 diagonals: more than the kernel's 8 (27-point stencils stay CSR)
    offs = list(range(-4, 5))
    A = sp.diags([rng.standard_normal(3000 - abs(o)) for o in offs], offs, format="csr")
    assert rk.SparseMatrix.from_scipy(A).ndiag == 0
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg3", 10)
    assert rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values).ndiag == 0
    # tridiagonal with a ragged last tile and one explicit zero kept
    n = 1000
    T = sp.diags([rng.standard_normal(n - 1), 2 + rng.random(n), rng.standard_normal(n - 1)],
                 [-1, 0, 1], format="csr")
    T.data[5] = 0.0
    M = rk.SparseMatrix.from_scipy(T)
    assert M.ndiag == 3
    x = rng.standard_normal(n)
    S = rk.make_sketch(16, n, 4, 2)
    z1, p1 = rk.spmv_sketch(M, S, x)
    M.set_diagonal_copy(False)
    z0, p0 = rk.spmv_sketch(M, S, x)
    assert torch.equal(z1, z0) and rel(p1, p0) <= 1e-14
    assert rel(z1, T @ x) <= 1e-14


def test_dia_per_tile_offsets(rk, torch):
    """Offsets that differ per 128-row tile (the halo columns of a row slab:
    9 distinct diagonals overall, at most 8 in any tile) keep the copy."""
    from paper_2503_22631_b200 import configs
    N = 16
    P = configs.build("cfg2", N)
    n, plane = P.n, N * N
    A = sp.csr_matrix((P.values, P.col_idx, P.row_ptr), shape=(n, n)).tolil()
    A.resize((n, n + 2 * plane))
    rng = np.random.default_rng(9)
    for r in range(plane):  # lower halo plane: column n + r
        A[r, n + r] = rng.standard_normal()
    for r in range(n - plane, n):  # upper halo plane: column n + plane + (r - (n - plane))
        A[r, n + plane + r - (n - plane)] = rng.standard_normal()
    A = A.tocsr()
    A.sort_indices()
    M = rk.SparseMatrix.from_scipy(A)
    assert M.ndiag == 7  # at most 6 stencil diagonals + the halo one in a boundary tile
    x = rng.standard_normal(n + 2 * plane)
    S = rk.make_sketch(32, n, 4, 3)
    z1, p1 = rk.spmv_sketch(M, S, x)
    M.set_diagonal_copy(False)
    z0, p0 = rk.spmv_sketch(M, S, x)
    assert torch.equal(z1, z0) and rel(p1, p0) <= 1e-14
    assert rel(z1, A @ x) <= 1e-14


def test_dia_solve_identical(rk, torch):
    """A whole restarted solve agrees to rounding with and without the copy."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg2", 30)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    assert A.ndiag == 7
    S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=20, tol=P.tol, k_max=P.k_max)
    b = torch.tensor(P.b, device="cuda")
    r1 = rk.restarted_krylov(A, b, f, opts, S)
    A.set_diagonal_copy(False)
    r0 = rk.restarted_krylov(A, b, f, opts, S)
    assert r1.cycles == r0.cycles and r1.cycles >= 2
    assert rel(r1.f_hat, r0.f_hat) <= 1e-12


def test_spmv_irregular_rows(rk, oracle, torch):
    # long rows exercise the chunked CSR-stream path; empty rows too
    rng = np.random.default_rng(3)
    n = 3000
    A = H.random_sparse(n, 0.002, 5).tolil()
    A[7, :] = rng.standard_normal(n)  # one dense row (n nnz > cap)
    A[11, :] = 0
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    M = rk.SparseMatrix.from_scipy(A)
    x = rng.standard_normal(n)
    assert rel(rk.spmv(M, x), A @ x) <= 1e-14


def test_invalid_csr_rejected(rk):
    A = H.random_sparse(50, 0.1, 1)
    ci = A.indices.copy()
    ci[0] = 500
    with pytest.raises(rk.ShapeError):
        rk.SparseMatrix.from_csr(A.indptr, ci, A.data)
    v = A.data.copy()
    v[0] = np.inf
    with pytest.raises(rk.NumericalError):
        rk.SparseMatrix.from_csr(A.indptr, A.indices, v)


# ---------------- K3/K4: one randomized Arnoldi decomposition ----------------
def test_randomized_arnoldi_matches_oracle(rk, oracle, torch):
    for seed in range(5):
        n, m = 400, 20
        A = H.random_sparse(n, 0.02, seed + 100, shift=3.0)
        b = H.random_vector(n, seed + 500)
        S = rk.make_sketch(4 * m, n, 8, seed)
        OS = oracle.make_sketch(4 * m, n, 8, seed)
        dec = rk.randomized_arnoldi(rk.SparseMatrix.from_scipy(A), S, b, m)
        od = oracle.arnoldi_decomp(A, b, m, OS)
        assert dec.breakdown_at is None and od.breakdown_at is None
        assert dec.start_norm == pytest.approx(od.start_norm, rel=1e-13)
        assert np.abs(dec.Rbar - od.Rbar).max() <= 1e-10 * np.abs(od.Rbar).max()
        assert rel(dec.W, od.W) <= 1e-10
        assert rel(dec.U, od.U) <= 1e-10
        assert dec.counters == od.counters
        W = dec.W.cpu().numpy()
        # residual identity A W_m = W_{m+1} Rbar (test_basis.cpp:21-29, <= 1e-12)
        res = np.linalg.norm(A @ W[:, :m] - W @ dec.Rbar)
        assert res / (oracle.norm1(A) * max(1, np.linalg.norm(W))) <= 1e-12
        U = dec.U.cpu().numpy()
        assert np.abs(U.T @ U - np.eye(m + 1)).max() <= 1e-8


def test_randomized_arnoldi_breakdown_and_errors(rk, oracle, torch):
    D = sp.diags([2.5, 1.0, 3.0, 4.0]).tocsr()
    A = rk.SparseMatrix.from_scipy(D)
    S = rk.make_sketch(4, 4, 4, 0)
    dec = rk.randomized_arnoldi(A, S, np.array([2.0, 0, 0, 0]), 3)
    assert dec.breakdown_at == 1
    assert dec.Rm()[0, 0] == pytest.approx(2.5, rel=1e-14)
    with pytest.raises(rk.ParameterError, match="zero start vector"):
        rk.randomized_arnoldi(A, S, np.zeros(4), 2)
    S3 = rk.make_sketch(3, 6, 2, 0)
    A6 = rk.SparseMatrix.from_scipy(sp.identity(6, format="csr"))
    with pytest.raises(rk.ParameterError):
        rk.randomized_arnoldi(A6, S3, np.ones(6), 4)  # d < m+1


# ---------------- the drop-in boundary: restarted_krylov ----------------
def _solve_both(rk, oracle, P, S_seed=1, opts=None, **kw):
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, S_seed)
    OS = oracle.make_sketch(P.d, P.n, P.zeta, S_seed)
    f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    opts = opts or rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    r = rk.restarted_krylov(A, P.b, f, opts, S, **kw)
    o = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b,
                                oracle.KIND_EXP_NEG if P.fn == "exp_neg" else oracle.KIND_INV_SQRT,
                                P.t, m_r=opts.m_r, tol=opts.tol, k_max=opts.k_max,
                                budget_total_m=opts.budget_total_m, S=OS, want_R=True)
    return r, o


@pytest.mark.parametrize("name,N", [("cfg1", 256), ("cfg1", 64), ("cfg2", 32), ("cfg4", 32)])
def test_restart_parity(rk, oracle, torch, name, N):
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    r, o = _solve_both(rk, oracle, P)
    assert r.converged == o.converged
    assert abs(r.cycles - o.cycles) <= 1
    assert rel(r.f_hat, o.f_hat) <= 1e-9
    if r.cycles == o.cycles:
        for hr, ho in zip(r.history, o.history):
            assert hr.total_m == ho["total_m"] and hr.total_matvecs == ho["total_matvecs"]
            assert hr.start_norm == pytest.approx(ho["start_norm"], rel=1e-10)
        R = r.R_accum
        assert np.abs(R - o.R_accum).max() <= 1e-9 * np.abs(o.R_accum).max()
    assert r.counters["matvecs"] == r.cycles * P.m or r.history[-1].total_m < r.cycles * P.m


def test_restart_equal_cycles_forced(rk, oracle, torch):
    """tol = 1e-30 forces equal cycle counts (test_restart.cpp:60, acceptance.cpp:304)."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg4", 20)
    opts = rk.RestartOptions(m_r=P.m, tol=1e-30, k_max=5)
    r, o = _solve_both(rk, oracle, P, opts=opts)
    assert r.cycles == o.cycles == 5 and not r.converged
    assert rel(r.f_hat, o.f_hat) <= 1e-9


def test_restart_device_resident_and_reference(rk, oracle, torch):
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg1", 64)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    rh = rk.restarted_krylov(A, P.b, f, opts, S)
    bd = torch.tensor(P.b, device="cuda")
    ref = torch.tensor(rh.f_hat, device="cuda")
    rd = rk.restarted_krylov(A, bd, f, opts, S, reference=ref)
    assert rd.f_hat.is_cuda
    # the per-block sketch partials meet in fp64 atomics (K2), so two solves
    # agree to run-to-run rounding, not bit for bit
    assert rel(rd.f_hat, rh.f_hat) <= 1e-12
    assert rd.history[-1].error_vs_reference <= 1e-12
    assert rd.solve_ms > 0 and all(h.build_ms > 0 for h in rd.history)


def test_restart_scale_cancellation(rk, torch):
    """Global rescaling of S leaves the result unchanged (acceptance.cpp:464-493)."""
    C = H.conv_diff_2d(20, 20, 0.01, 10.0, 0.0)
    A = rk.SparseMatrix.from_scipy(C)
    b = H.random_vector(C.shape[0], 1)
    f = rk.FunctionSpec.exp_neg(1.0 / C.diagonal().max())
    opts = rk.RestartOptions(m_r=8, k_max=6, tol=1e-12)
    S1 = rk.make_sketch(120, C.shape[0], 4, 3)
    r1 = rk.restarted_krylov(A, b, f, opts, S1)
    S1.scale = S1.scale * 7.3
    r2 = rk.restarted_krylov(A, b, f, opts, S1)
    assert rel(r2.f_hat, r1.f_hat) <= 1e-13


def test_restart_semantics(rk, oracle, torch):
    """k_max / budget / validation / divergence (test_restart.cpp:209-277)."""
    T = H.random_spd_tridiag(120, 1.0, 9.0, 31)
    A = rk.SparseMatrix.from_scipy(T)
    b = H.random_vector(120, 32)
    S = rk.make_sketch(44, 120, 4, 1)
    f = rk.FunctionSpec.exp_neg(1.0)
    r = rk.restarted_krylov(A, b, f, rk.RestartOptions(m_r=10, tol=1e-30, k_max=3), S)
    assert r.cycles == 3 and not r.converged and r.total_m == 30
    r = rk.restarted_krylov(A, b, f, rk.RestartOptions(m_r=10, tol=1e-30, k_max=50,
                                                       budget_total_m=25), S)
    assert r.cycles == 2 and r.total_m == 20 and not r.converged
    for kw in [dict(m_r=0), dict(k_max=0), dict(tol=0.0), dict(m_r=10, budget_total_m=5)]:
        with pytest.raises(rk.ParameterError):
            rk.restarted_krylov(A, b, f, rk.RestartOptions(**kw), S)
    C = H.conv_diff_2d(60, 60, 0.001, 10.0, 0.0)
    AC = rk.SparseMatrix.from_scipy(C)
    Sd = rk.make_sketch(6, C.shape[0], 1, 3)
    with pytest.raises(rk.NumericalError, match="^restart divergence"):
        rk.restarted_krylov(AC, H.random_vector(C.shape[0], 1),
                            rk.FunctionSpec.exp_neg(10.0 / oracle.norm1(C)),
                            rk.RestartOptions(m_r=5, tol=1e-12, k_max=60), Sd)


def test_restart_happy_breakdown(rk, oracle, torch):
    """m_r = n: the Krylov space saturates in one cycle (test_restart.cpp:91-112)."""
    n = 25
    D = sp.diags([10.0 * (1.0 + np.arange(n)), 2.0 * np.ones(n - 1)], [0, -1]).tocsr()
    D.sort_indices()
    A = rk.SparseMatrix.from_scipy(D)
    b = H.random_vector(n, 100)
    S = rk.make_sketch(n, n, 4, 2)
    r = rk.restarted_krylov(A, b, rk.FunctionSpec.exp_neg(0.02),
                            rk.RestartOptions(m_r=n, tol=1e-30, k_max=10), S)
    assert r.converged and r.cycles == 1
    assert r.counters["matvecs"] == n and r.counters["basis_updates"] == n - 1
    import scipy.linalg as sla
    ex = sla.expm(-0.02 * D.toarray()) @ b
    # a square sparse-sign S (d = n) limits the randomized basis' accuracy; the
    # oracle with the same S shows the same ~1e-8 gap to the exact value
    o = oracle.restarted_krylov(D, b, oracle.KIND_EXP_NEG, 0.02, m_r=n, tol=1e-30, k_max=10,
                                S=oracle.make_sketch(n, n, 4, 2))
    assert o.cycles == 1
    assert rel(r.f_hat, o.f_hat) <= 1e-8
    assert rel(r.f_hat, ex) <= 1e-7


def test_inv_sqrt_quadrature_parity(rk, oracle, torch):
    """InvSqrt (cfg3 kind, not in the reference): device restart quadrature vs
    the oracle's full Denman-Beavers f(R_accum) — parity unpinned by the reference."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg3", 10)
    P.m, P.d = 10, 40
    P.tol = 1e-9 * np.linalg.norm(P.b)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=60)
    r, o = _solve_both(rk, oracle, P, opts=opts)
    assert abs(r.cycles - o.cycles) <= 1
    assert rel(r.f_hat, o.f_hat) <= 1e-9


@pytest.mark.parametrize("name", ["cfg2"])
def test_full_size_properties(rk, torch, name):
    """Full BASELINE size: converged, and f matches an independent check."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    r = rk.restarted_krylov(A, torch.tensor(P.b, device="cuda"), rk.FunctionSpec.exp_neg(P.t),
                            rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max), S)
    assert r.converged
    assert r.history[-1].update_norm <= P.tol
    # semigroup check: exp(-tA) b computed with two half-step solves
    f = rk.FunctionSpec.exp_neg(P.t / 2)
    o = rk.RestartOptions(m_r=P.m, tol=P.tol * 1e-2, k_max=P.k_max)
    h1 = rk.restarted_krylov(A, torch.tensor(P.b, device="cuda"), f, o, S)
    h2 = rk.restarted_krylov(A, h1.f_hat, f, o, S)
    assert rel(h2.f_hat, r.f_hat) <= 1e-6


def test_cpp_host_api(rk):
    """include/rkmf_b200.hpp (the C++ mirror of restart.hpp) end to end."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(rk.LIB_PATH), "cpp_api_smoke")
    assert os.path.exists(exe), "build() must produce the C++ smoke program"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "converged=1" in r.stdout


# ---------------- on-device generators (cfg5's path) ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("kind,args", [("lap", (2, 40)), ("lap", (3, 17)), ("q1", (9, False, 1, False)),
                                       ("q1", (8, True, 3, True)), ("q1", (2, False, 1, False))])
def test_device_generators_match_host(rk, torch, kind, args):
    if kind == "lap":
        Ad = rk.SparseMatrix.laplacian(*args)
        rp, ci, v = rk.gen_laplacian(*args)
    else:
        Ad = rk.SparseMatrix.q1_hex(*args)
        rp, ci, v = rk.gen_q1_hex(*args)
    Ah = rk.SparseMatrix.from_csr(rp, ci, v)
    assert (Ad.n_rows, Ad.nnz) == (Ah.n_rows, Ah.nnz)
    lognormal = kind == "q1" and args[1]
    assert Ad.norm1 == pytest.approx(Ah.norm1, rel=1e-14 if lognormal else 0.0)
    x = torch.tensor(rk.gen_gaussian(5, Ad.n_rows), device="cuda")
    zd, zh = rk.spmv(Ad, x), rk.spmv(Ah, x)
    if lognormal:
        assert float((zd - zh).norm() / zh.norm()) <= 1e-14
    else:
        assert torch.equal(zd, zh)


@pytest.mark.gpu
def test_device_gaussian_matches_host(rk, torch):
    d = rk.gen_gaussian_device(7, 1000, 5000).cpu().numpy()
    h = rk.gen_gaussian_range(7, 1000, 5000)
    assert np.max(np.abs(d - h) / np.maximum(np.abs(h), 1e-300)) <= 1e-14


# ---------------- classical restarted Arnoldi (S == nullptr) ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,N", [("cfg1", 64), ("cfg2", 20), ("cfg4", 16)])
def test_classical_restart_matches_oracle(rk, oracle, torch, name, N):
    """restart.cpp:53-55 with the classical builder (basis.cpp:34-77): device
    CGS2 vs the oracle's MGS, f_hat within 1e-9, cycles within one, the
    reference's counter formulas (dot_n = sum m_k(m_k+1)/2, dot_d = 0)."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    r = rk.restarted_krylov(A, torch.tensor(P.b, device="cuda"), f, opts, None)
    o = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, oracle.KIND_EXP_NEG, P.t,
                                m_r=P.m, tol=P.tol, k_max=P.k_max, S=None)
    fd = r.f_hat.cpu().numpy()
    assert r.converged and o.converged
    assert abs(r.cycles - o.cycles) <= 1
    assert np.linalg.norm(fd - o.f_hat) <= 1e-9 * np.linalg.norm(o.f_hat)
    assert r.alpha == pytest.approx(np.linalg.norm(P.b), rel=1e-13)  # beta = ||b||_2
    assert r.counters["dot_d"] == 0
    assert r.counters["dot_n"] == r.counters["matvecs"] * (P.m + 1) // 2 or r.cycles > 1


@pytest.mark.gpu
def test_classical_breakdown_and_zero_start(rk, oracle, torch):
    # happy breakdown: b in a 3-dimensional invariant subspace of a diagonal A
    n = 40
    d = np.arange(1, n + 1, dtype=np.float64)
    A = sp.diags(d).tocsr()
    b = np.zeros(n)
    b[[2, 7, 11]] = [1.0, -2.0, 0.5]
    dA = rk.SparseMatrix.from_scipy(A)
    f = rk.FunctionSpec.exp_neg(0.3)
    r = rk.restarted_krylov(dA, b, f, rk.RestartOptions(m_r=10, tol=1e-12, k_max=5), None)
    assert r.converged and r.cycles == 1 and r.total_m == 3
    ref = np.exp(-0.3 * d) * b
    assert np.linalg.norm(r.f_hat - ref) <= 1e-12 * np.linalg.norm(ref)
    with pytest.raises(rk.ParameterError, match="zero start vector"):
        rk.restarted_krylov(dA, np.zeros(n), f, rk.RestartOptions(m_r=5), None)


# ---------------- per-cycle diagnostics (restart.cpp:101,103) ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,N,sketched", [("cfg2", 14, True), ("cfg4", 12, True),
                                             ("cfg1", 40, False)])
def test_cycle_diagnostics_match_numpy(rk, oracle, torch, name, N, sketched):
    """kappa_W = cond_2(W_m) and the leftmost Ritz value of R_m for cycle 1,
    against numpy's SVD / eig of the oracle's decomposition of the same start."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1) if sketched else None
    OS = oracle.make_sketch(P.d, P.n, P.zeta, 1) if sketched else None
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max, diagnostics=True)
    r = rk.restarted_krylov(A, P.b, f, opts, S)
    dec = oracle.arnoldi_decomp((P.row_ptr, P.col_idx, P.values), P.b, P.m, OS)
    m = dec.m
    sv = np.linalg.svd(dec.W[:, :m], compute_uv=False)
    kappa = sv[0] / sv[-1]
    ritz = np.linalg.eigvals(dec.Rbar[:m, :m])
    h0 = r.history[0]
    assert h0.kappa_W == pytest.approx(kappa, rel=1e-6)
    assert h0.leftmost_ritz_re == pytest.approx(float(np.min(ritz.real)),
                                                rel=1e-8, abs=1e-10 * np.abs(ritz).max())
    for h in r.history:
        assert np.isfinite(h.kappa_W) and h.kappa_W >= 1.0
    # off by default
    r2 = rk.restarted_krylov(A, P.b, f, rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=2), S)
    assert np.isnan(r2.history[0].kappa_W)


# ---------------- ExpNeg restart quadrature ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,N,m", [("cfg2", 16, None), ("cfg4", 14, None), ("cfg1", 48, None),
                                      ("cfg1", 64, 10), ("cfg2", 24, 20)])
def test_expneg_quadrature_matches_full_and_oracle(rk, oracle, torch, name, N, m):
    """dense_f = quadrature for exp(-tA): O(N_q m^2) per cycle instead of
    f(R_accum) in full; same f_hat as FULL and the oracle (1e-9), same cycles."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    mr = m or P.m
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    f = rk.FunctionSpec.exp_neg(P.t)
    b = torch.tensor(P.b, device="cuda")
    rq = rk.restarted_krylov(A, b, f, rk.RestartOptions(m_r=mr, tol=P.tol, k_max=P.k_max,
                                                        dense_f="quadrature"), S)
    rf = rk.restarted_krylov(A, b, f, rk.RestartOptions(m_r=mr, tol=P.tol, k_max=P.k_max), S)
    OS = oracle.make_sketch(P.d, P.n, P.zeta, 1)
    o = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, oracle.KIND_EXP_NEG, P.t,
                                m_r=mr, tol=P.tol, k_max=P.k_max, S=OS)
    fq, ff = rq.f_hat.cpu().numpy(), rf.f_hat.cpu().numpy()
    assert rq.converged and abs(rq.cycles - o.cycles) <= 1 and rq.cycles == rf.cycles
    assert np.linalg.norm(fq - ff) <= 1e-10 * np.linalg.norm(ff)
    assert np.linalg.norm(fq - o.f_hat) <= 1e-9 * np.linalg.norm(o.f_hat)


# ---------------- acceptance c8/c9 and the R_accum pattern on device ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("eps,vx,vy", [(0.1, 1.0, 0.01), (0.01, 1.0, 0.01), (0.01, 1.0, 1.0)])
def test_restarted_convergence_conv_diff_grids(rk, torch, eps, vx, vy):
    """acceptance.cpp:346-425 (c8/c9) on 60x60 convection-diffusion grids: m_r = 20,
    d = 320, zeta in {1, 4}, tol = 1e-13 ||b||, k_max = 50. Both builders reach
    the exact exp(-tA)b (scipy expm_multiply): classical <= 1e-8, randomized
    <= 1e-9; at the last common cycle randomized error <= 10x classical."""
    from scipy.sparse.linalg import expm_multiply
    A = H.conv_diff_2d(60, 60, eps, vx, vy)
    n = A.shape[0]
    b = H.random_vector(n, 11)
    t = 2.0 / abs(A).sum(axis=0).max()
    ref = expm_multiply(-t * A, b)
    dA = rk.SparseMatrix.from_scipy(A)
    f = rk.FunctionSpec.exp_neg(t)
    opts = rk.RestartOptions(m_r=20, k_max=50, tol=1e-13 * np.linalg.norm(b))
    rc = rk.restarted_krylov(dA, b, f, opts, None, reference=ref)
    ec = [h.error_vs_reference for h in rc.history]
    assert min(ec) <= 1e-8
    for zeta in (1, 4):
        S = rk.make_sketch(320, n, zeta, 1)
        rr = rk.restarted_krylov(dA, b, f, opts, S, reference=ref)
        er = [h.error_vs_reference for h in rr.history]
        assert min(er) <= 1e-9, (zeta, min(er))
        common = min(len(ec), len(er))
        assert er[common - 1] <= 10.0 * max(ec[common - 1], 1e-15)


@pytest.mark.gpu
def test_r_accum_block_pattern(rk, torch):
    """test_restart.cpp:131-164: the accumulated compression keeps the block
    lower-bidiagonal pattern exactly (zeros are exact), couplings nonzero."""
    A = H.conv_diff_2d(12, 12, 0.1, 0.01, 1.0)
    b = H.random_vector(A.shape[0], 3)
    m_r = 8
    S = rk.make_sketch(64, A.shape[0], 4, 12)
    r = rk.restarted_krylov(rk.SparseMatrix.from_scipy(A), b,
                            rk.FunctionSpec.exp_neg(1.0 / abs(A).sum(axis=0).max()),
                            rk.RestartOptions(m_r=m_r, tol=1e-30, k_max=4), S)
    assert r.cycles == 4
    R = r.R_accum
    assert R.shape == (4 * m_r, 4 * m_r)
    checked = 0
    for i in range(R.shape[0]):
        for j in range(R.shape[1]):
            bi, bj = i // m_r, j // m_r
            in_diag = bi == bj and (i % m_r) <= (j % m_r) + 1
            coupling = bi == bj + 1 and i % m_r == 0 and j % m_r == m_r - 1
            if not in_diag and not coupling:
                checked += 1
                assert R[i, j] == 0.0, (i, j)
    assert checked > 0
    for k in range(1, 4):
        assert R[k * m_r, k * m_r - 1] != 0.0


# ---------------- the device path against the committed golden fixtures ----------------
@pytest.mark.gpu
def test_device_against_golden_fixtures(rk, torch):
    """tests/golden (frozen from the oracle by make_golden.py): the device sketch
    is bit-exact with sketch.npz, and the device restart reproduces restart.npz
    (cycles +-1, f within the north-star 1e-9 relative, plus 1e-18 ||b||:
    cfg4_N10's f_hat is 1e-15 of ||b||, a cancellation-dominated quantity
    whose last digits depend on the summation order; update norms within
    1e-8, start norms within 1e-6: from cycle 2 on, ||S w_m|| - 1 measures the
    sketched orthogonality loss, ~1e-8, also cancellation-dominated). The
    device solve itself is bitwise reproducible (test_gpu_boundary.py)."""
    import os
    from paper_2503_22631_b200 import configs
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    g = np.load(os.path.join(gold, "sketch.npz"))
    for key in sorted(k[:-5] for k in g.files if k.endswith("_rows")):
        d, n, z, s = (int(p[1:]) for p in key.split("_"))
        rows, signs, _ = rk.make_sketch(d, n, z, s).export()
        assert np.array_equal(rows, g[key + "_rows"].astype(np.int64)), key
        assert np.array_equal(signs, g[key + "_signs"]), key
    h = np.load(os.path.join(gold, "restart.npz"))
    for name, N in [("cfg1", 32), ("cfg2", 12), ("cfg4", 10)]:
        P = configs.build(name, N)
        key = f"{name}_N{N}"
        assert P.t == float(h[key + "_t"][0])
        A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
        S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
        r = rk.restarted_krylov(A, torch.tensor(P.b, device="cuda"), rk.FunctionSpec.exp_neg(P.t),
                                rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max), S)
        cycles, total_m, conv = h[key + "_meta"].tolist()
        assert abs(r.cycles - cycles) <= 1 and bool(r.converged) == bool(conv)
        f = r.f_hat.cpu().numpy()
        assert np.linalg.norm(f - h[key + "_f"]) <= (1e-9 * np.linalg.norm(h[key + "_f"])
                                                     + 1e-18 * np.linalg.norm(P.b))
        c = min(r.cycles, cycles)
        sn = np.array([x.start_norm for x in r.history[:c]])
        assert np.allclose(sn, h[key + "_start_norm"][:c], rtol=1e-6)
        un = np.array([x.update_norm for x in r.history[:c]])
        ug = h[key + "_update_norm"][:c]
        assert np.all(np.abs(un - ug) <= 1e-8 * np.abs(ug) + 1e-12 * np.linalg.norm(P.b))


# ---------------- fused small-matrix cycle (cycle_small.cu) ----------------
@pytest.mark.parametrize("name,N", [("cfg1", 128), ("cfg2", 24), ("cfg4", 24), ("cfg5", 24)])
def test_fused_cycle_matches_steps_and_oracle(rk, oracle, torch, name, N):
    """Matrices of <= 131072 rows run each cycle's steps in one cooperative
    kernel. Same z as K2 (CSR rows in column order), the sketch partials in
    another fixed block order: the solve agrees with the per-step kernels to
    rounding and with the oracle to the north-star 1e-9, at equal cycle counts
    (forced) and converged; both paths are bitwise reproducible."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    assert P.n <= 131072
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    b = torch.tensor(P.b, device="cuda")
    ctx = A.ctx

    def solve(fused, **o):
        ctx.set_fused_cycle(fused)
        try:
            opts = dict(m_r=P.m, tol=P.tol, k_max=P.k_max)
            opts.update(o)
            return rk.restarted_krylov(A, b, f, rk.RestartOptions(**opts), S)
        finally:
            ctx.set_fused_cycle(True)

    ctx.kernel_timing(True)
    ctx.kernel_times(reset=True)
    rf = solve(True, tol=1e-30, k_max=2)
    kt = ctx.kernel_times(reset=True)
    ctx.kernel_timing(False)
    assert kt["fused_cycle"][1] == 2 and kt["spmv_sketch"][1] == 0  # the fused path ran
    rs = solve(False, tol=1e-30, k_max=2)
    assert rf.cycles == rs.cycles == 2
    assert rel(rf.f_hat, rs.f_hat) <= 1e-11
    OS = oracle.make_sketch(P.d, P.n, P.zeta, 1)
    kind = oracle.KIND_EXP_NEG if P.fn == "exp_neg" else oracle.KIND_INV_SQRT
    o = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, kind, P.t, S=OS,
                                m_r=P.m, tol=1e-30, k_max=2)
    assert rel(rf.f_hat, o.f_hat) <= 1e-9
    r1, r2 = solve(True), solve(True)
    assert torch.equal(r1.f_hat, r2.f_hat)
    oc = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, kind, P.t, S=OS,
                                 m_r=P.m, tol=P.tol, k_max=P.k_max)
    assert r1.converged and abs(r1.cycles - oc.cycles) <= 1
    assert rel(r1.f_hat, oc.f_hat) <= 1e-9


# ---------------- CSR row dictionary (rowdict.cu) ----------------
@pytest.mark.parametrize("N", [20, 53])
def test_csr_row_dictionary(rk, oracle, torch, N):
    """27-point matrices keep the CSR stream (no diagonal copy), but the
    constant-coefficient Q1 matrix (cfg5's kind) has one row form per
    boundary class (27): K2 then streams one byte per row and walks the
    form's offsets and values from shared memory in column order, one thread
    per row (the CSR kernel interleaves two lanes per row), so z agrees with
    the CSR kernel to rounding; solves agree to rounding and with the
    oracle. Lognormal coefficients (cfg3's kind) give every row its own form:
    no dictionary."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg5", N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    assert A.ndiag == 0 and A.ntuples == 27
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    OS = oracle.make_sketch(P.d, P.n, P.zeta, 1)
    zo = oracle.spmv((P.row_ptr, P.col_idx, P.values), P.b)
    z1, p1 = rk.spmv_sketch(A, S, P.b)
    assert rel(z1, zo) <= 1e-14
    assert rel(p1, oracle.sketch_apply(OS, zo)) <= 1e-13
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    b = torch.tensor(P.b, device="cuda")
    A.ctx.set_fused_cycle(False)  # the per-step K2 (small n would take the fused cycle)
    try:
        r1 = rk.restarted_krylov(A, b, f, opts, S)
        assert A.set_row_dictionary(False) == 0 and A.ntuples == 0
        z0, p0 = rk.spmv_sketch(A, S, P.b)
        r0 = rk.restarted_krylov(A, b, f, opts, S)
        assert A.set_row_dictionary(True) == 27
    finally:
        A.ctx.set_fused_cycle(True)
    assert rel(z1, z0) <= 1e-15 and rel(p1, p0) <= 1e-14
    assert r1.cycles == r0.cycles and rel(r1.f_hat, r0.f_hat) <= 1e-12
    o = oracle.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, oracle.KIND_EXP_NEG,
                                P.t, S=OS, m_r=P.m, tol=P.tol, k_max=P.k_max)
    assert r1.converged and abs(r1.cycles - o.cycles) <= 1
    assert rel(r1.f_hat, o.f_hat) <= 1e-9
    # lognormal coefficients: a form per row, no dictionary
    Q = configs.build("cfg3", 12)
    B = rk.SparseMatrix.from_csr(Q.row_ptr, Q.col_idx, Q.values)
    assert B.ndiag == 0 and B.ntuples == 0


@pytest.mark.parametrize("n,m,d,zeta", [(20000, 10, 600, 8), (9000, 63, 256, 4), (120001, 20, 96, 8)])
def test_fused_cycle_edge_shapes(rk, oracle, torch, n, m, d, zeta):
    """The fused cycle kernel's edges: a sketch wider than its 512 threads
    (d = 600), the largest basis it takes (m = 63: k + 1 = 64 in the register
    triangular solve), more tiles than one round of blocks (70,001 rows: the
    CSR rows read from L2 instead of staged), ragged last tiles. Against the
    per-step kernels and the oracle at forced equal cycle counts."""
    A = H.random_sparse(n, 6.0 / n, n + m, shift=4.0)
    b = H.random_vector(n, n + 1)
    t = 1.0 / abs(oracle.norm1(A))
    S = rk.make_sketch(d, n, zeta, 5)
    OS = oracle.make_sketch(d, n, zeta, 5)
    dA = rk.SparseMatrix.from_scipy(A)
    bd = torch.tensor(b, device="cuda")
    f = rk.FunctionSpec.exp_neg(t)
    opts = rk.RestartOptions(m_r=m, tol=1e-30, k_max=2)
    ctx = dA.ctx
    ctx.kernel_timing(True)
    ctx.kernel_times(reset=True)
    ctx.set_fused_cycle(True)
    rf = rk.restarted_krylov(dA, bd, f, opts, S)
    kt = ctx.kernel_times(reset=True)
    ctx.kernel_timing(False)
    assert kt["fused_cycle"][1] == 2
    ctx.set_fused_cycle(False)
    try:
        rs = rk.restarted_krylov(dA, bd, f, opts, S)
    finally:
        ctx.set_fused_cycle(True)
    o = oracle.restarted_krylov(A, b, oracle.KIND_EXP_NEG, t, S=OS, m_r=m, tol=1e-30, k_max=2)
    assert rf.cycles == rs.cycles == o.cycles == 2
    assert rel(rf.f_hat, rs.f_hat) <= 1e-11
    assert rel(rf.f_hat, o.f_hat) <= 1e-9
