"""InvSqrt robustness (BASELINE cfg3): the adaptive restart
quadrature for z^{-1/2} (engine.cu, densef.cu design_invsqrt).

* complex spectrum: eigenvalues at up to 83 degrees from the positive axis
  need a finer step than the positive-spectrum design; the design (verified
  by node doubling: the cycle's coefficients at half the step agree to
  1e-12) takes more nodes and the solve matches the eigendecomposition
  A^{-1/2} b. (At 2.2 rad the field of values straddles the branch cut and
  restarted FOM itself stagnates: the oracle's Denman-Beavers run does not
  converge in 60 cycles either, so that spectrum cannot be a parity case.)
* branch-cut guard: Ritz values on (-inf, 0] raise NumericalError (the
  reference has no InvSqrt kind; its point Schur-Parlett route would throw
  on clustered values, densefun.cpp:407-417);
* fixed node counts (quad_nodes > 0) keep the previous fixed-interval rule.
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def _rotation_blocks(n2, rmin, rmax, thmax, seed):
    """Block-diagonal 2x2 rotations: eigenvalues r e^{+-i theta}."""
    rng = np.random.default_rng(seed)
    r = np.exp(rng.uniform(np.log(rmin), np.log(rmax), n2))
    th = rng.uniform(0.0, thmax, n2)
    a, b = r * np.cos(th), r * np.sin(th)
    rows, cols, vals = [], [], []
    for i in range(n2):
        p = 2 * i
        rows += [p, p, p + 1, p + 1]
        cols += [p, p + 1, p, p + 1]
        vals += [a[i], -b[i], b[i], a[i]]
    A = sp.csr_matrix((vals, (rows, cols)), shape=(2 * n2, 2 * n2))
    A.sort_indices()
    return A


def _exact_inv_sqrt(A, b):
    lam, V = np.linalg.eig(A.toarray())
    return np.real(V @ (lam ** -0.5 * np.linalg.solve(V, b)))


def test_complex_spectrum_design(rk, oracle, torch):
    A = _rotation_blocks(150, 1.0, 30.0, 1.45, 3)
    n = A.shape[0]
    b = np.random.default_rng(4).standard_normal(n)
    ref = _exact_inv_sqrt(A, b)
    S = rk.make_sketch(160, n, 8, 1)
    r = rk.restarted_krylov(rk.SparseMatrix.from_scipy(A), b, rk.FunctionSpec.inv_sqrt(),
                            rk.RestartOptions(m_r=40, tol=1e-12 * np.linalg.norm(b), k_max=60), S)
    assert r.converged
    # the 1.45 rad eigenvalue angle needs h <= pi (pi - 1.55)/38 (~0.13): about
    # twice the nodes of the positive-spectrum design (h = 0.25, ~320 here)
    assert r.quad_nodes > 450
    f = r.f_hat if isinstance(r.f_hat, np.ndarray) else r.f_hat.cpu().numpy()
    assert np.linalg.norm(f - ref) <= 1e-9 * np.linalg.norm(ref)
    OS = oracle.make_sketch(160, n, 8, 1)
    o = oracle.restarted_krylov((A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data), b,
                                oracle.KIND_INV_SQRT, 0.0, m_r=40, tol=1e-12 * np.linalg.norm(b),
                                k_max=60, S=OS)
    assert o.converged and abs(o.cycles - r.cycles) <= 1
    assert np.linalg.norm(f - o.f_hat) <= 1e-9 * np.linalg.norm(o.f_hat)


def test_positive_spectrum_matches_exact(rk, torch):
    from tests import helpers as H
    A = H.random_spd_tridiag(400, 0.01, 50.0, 5)
    b = H.random_vector(400, 6)
    ref = _exact_inv_sqrt(A, b)
    S = rk.make_sketch(120, 400, 8, 2)
    r = rk.restarted_krylov(rk.SparseMatrix.from_scipy(A), b, rk.FunctionSpec.inv_sqrt(),
                            rk.RestartOptions(m_r=30, tol=1e-12 * np.linalg.norm(b), k_max=80), S)
    assert r.converged and 0 < r.quad_nodes <= 2048
    assert np.linalg.norm(r.f_hat - ref) <= 1e-9 * np.linalg.norm(ref)


def test_branch_cut_guard(rk, torch):
    """A symmetric matrix with negative eigenvalues: z^{-1/2} is undefined on
    its spectrum, the first cycle's Ritz values say so."""
    n = 300
    d = np.linspace(-5.0, 20.0, n)
    A = sp.diags([-np.ones(n - 1), d, -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    A.sort_indices()
    b = np.random.default_rng(7).standard_normal(n)
    S = rk.make_sketch(80, n, 8, 3)
    with pytest.raises(rk.NumericalError, match="branch cut"):
        rk.restarted_krylov(rk.SparseMatrix.from_scipy(A), b, rk.FunctionSpec.inv_sqrt(),
                            rk.RestartOptions(m_r=20, tol=1e-10, k_max=5), S)


def test_fixed_node_count_still_available(rk, torch):
    from tests import helpers as H
    A = H.random_spd_tridiag(300, 0.5, 20.0, 8)
    b = H.random_vector(300, 9)
    ref = _exact_inv_sqrt(A, b)
    S = rk.make_sketch(100, 300, 8, 4)
    r = rk.restarted_krylov(rk.SparseMatrix.from_scipy(A), b, rk.FunctionSpec.inv_sqrt(),
                            rk.RestartOptions(m_r=25, tol=1e-12 * np.linalg.norm(b), k_max=60,
                                              quad_nodes=512), S)
    assert r.converged and r.quad_nodes == 512
    assert np.linalg.norm(r.f_hat - ref) <= 1e-9 * np.linalg.norm(ref)
