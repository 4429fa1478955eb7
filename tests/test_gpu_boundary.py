"""Boundary completeness and reproducibility on the device path.

* The reference's two-path identity (proj/tests/test_restart.cpp:44-64,
  119-129; acceptance.cpp:294-344) through the test-only CycleObserver
  (restart.hpp:42-54): at every cycle, alpha * [W_1 .. W_k] f(R_accum) e_1
  equals the update-form f_hat to 1e-11.
* Bitwise reproducibility (test_restart.cpp:405-443): two solves with the same
  inputs give identical bits (the sketch partials and ||y||^2 are reduced in a
  fixed order, detred.cuh).
* RestartResult.R_accum refuses to return another solve's matrix.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from tests import helpers as H

pytestmark = pytest.mark.gpu


def _two_path_gap(rk, A_sp, b, t, m_r, k_max, S):
    import torch
    A = rk.SparseMatrix.from_scipy(A_sp)
    n = A_sp.shape[0]
    blocks, worst, seen = [], [0.0], []

    def obs(info):
        assert info.W.shape[0] == n and info.W.shape[1] in (info.m_k, info.m_k + 1)
        blocks.append(info.W[:, :info.m_k])
        Wbig = np.concatenate(blocks, axis=1)
        F = sla.expm(-t * info.R_accum)
        full = info.alpha * (Wbig @ F[:, 0])
        worst[0] = max(worst[0], np.linalg.norm(full - info.f_hat) / np.linalg.norm(info.f_hat))
        seen.append((info.cycle, info.update.copy(), info.f_hat.copy()))

    r = rk.restarted_krylov(A, torch.tensor(b, device="cuda"), rk.FunctionSpec.exp_neg(t),
                            rk.RestartOptions(m_r=m_r, tol=1e-30, k_max=k_max), S, observer=obs)
    assert [c for c, _, _ in seen] == list(range(1, r.cycles + 1))
    # the last observed f_hat is the result, and the updates telescope to it
    f = r.f_hat.cpu().numpy()
    assert np.array_equal(seen[-1][2], f)
    ysum = np.sum([y for _, y, _ in seen], axis=0)
    assert np.linalg.norm(ysum - f) <= 1e-13 * np.linalg.norm(f)
    return worst[0]


def test_two_path_identity_spd(rk):
    A = H.random_spd_tridiag(200, 1.0, 9.0, 7)
    b = H.random_vector(200, 8)
    assert _two_path_gap(rk, A, b, 1.0, 4, 4, None) <= 1e-11
    assert _two_path_gap(rk, A, b, 1.0, 4, 4, rk.make_sketch(64, 200, 4, 11)) <= 1e-11


def test_two_path_identity_nonnormal(rk):
    A = H.conv_diff_2d(12, 12, 0.1, 1.0, 0.01)
    n = A.shape[0]
    b = H.random_vector(n, 9)
    assert _two_path_gap(rk, A, b, 1.0, 8, 4, None) <= 1e-11
    assert _two_path_gap(rk, A, b, 1.0, 8, 4, rk.make_sketch(64, n, 4, 12)) <= 1e-11


def test_observer_basis_block_is_the_decomposition(rk, torch):
    """Cycle 1's observed W equals randomized_arnoldi's W (basis.cpp:92-142)."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg2", 14)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    got = []
    rk.restarted_krylov(A, P.b, rk.FunctionSpec.exp_neg(P.t),
                        rk.RestartOptions(m_r=P.m, tol=1e-30, k_max=2), S,
                        observer=lambda i: got.append(i.W.copy()))
    dec = rk.randomized_arnoldi(A, S, P.b, P.m)
    W = dec.W.cpu().numpy()
    assert got[0].shape == W.shape
    assert np.abs(got[0] - W).max() <= 1e-12 * np.abs(W).max()


@pytest.mark.parametrize("name,N,classical", [("cfg2", 40, False), ("cfg4", 32, False),
                                              ("cfg3", 16, False), ("cfg1", 256, False),
                                              ("cfg2", 24, True)])
def test_solves_are_bitwise_reproducible(rk, torch, name, N, classical):
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = None if classical else rk.make_sketch(P.d, P.n, P.zeta, 1)
    f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    b = torch.tensor(P.b, device="cuda")
    r1 = rk.restarted_krylov(A, b, f, opts, S)
    r2 = rk.restarted_krylov(A, b, f, opts, S)
    assert torch.equal(r1.f_hat, r2.f_hat)
    assert [h.update_norm for h in r1.history] == [h.update_norm for h in r2.history]
    # and through a fresh context (fresh scratch, fresh tickets)
    ctx = rk.Context(0)
    A2 = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values, ctx=ctx)
    S2 = None if classical else rk.make_sketch(P.d, P.n, P.zeta, 1, ctx=ctx)
    r3 = rk.restarted_krylov(A2, P.b, f, opts, S2)
    assert np.array_equal(r3.f_hat, r1.f_hat.cpu().numpy())


def test_norm1_and_diagnostics_reproducible(rk, torch, oracle):
    """norm1 (fixed-point column sums, spmv.cu) and the per-cycle kappa_W
    (Gram partials summed in block order, diag.cu) are the same bits on every
    run: the CSV harness prints them (acceptance.cpp:545-582, c14)."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg3", 24)  # lognormal values: column sums round
    n1 = {rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values).norm1 for _ in range(4)}
    assert len(n1) == 1
    assert n1.pop() == pytest.approx(oracle.norm1((P.row_ptr, P.col_idx, P.values)), rel=1e-15)
    P = configs.build("cfg1", 64)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max, diagnostics=True)
    b = torch.tensor(P.b, device="cuda")
    runs = [rk.restarted_krylov(A, b, rk.FunctionSpec.exp_neg(P.t), opts, S) for _ in range(3)]
    k = [[h.kappa_W for h in r.history] for r in runs]
    assert k[0] == k[1] == k[2] and all(np.isfinite(k[0]))


def test_sketch_reduction_reproducible(rk, torch):
    """The fused kernel's sketch (many blocks) is the same bits every launch."""
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg2", 64)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    x = torch.tensor(P.b, device="cuda")
    ps = [rk.spmv_sketch(A, S, x)[1] for _ in range(5)] + [rk.sketch_apply(S, x) for _ in range(2)]
    for p in ps[1:5]:
        assert torch.equal(p, ps[0])
    assert torch.equal(ps[5], ps[6])


def test_r_accum_guard(rk, torch):
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg1", 32)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    f = rk.FunctionSpec.exp_neg(P.t)
    o = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    r1 = rk.restarted_krylov(A, P.b, f, o, S, keep_R_accum=True)
    r2 = rk.restarted_krylov(A, P.b, f, rk.RestartOptions(m_r=P.m - 1, tol=P.tol, k_max=3), S)
    assert r1.R_accum.shape == (r1.total_m, r1.total_m)  # copied eagerly
    r3 = rk.restarted_krylov(A, P.b, f, o, S)
    with pytest.raises(rk.Error):
        r2.R_accum  # noqa: B018 - the context moved on
    assert np.array_equal(r3.R_accum, r1.R_accum)
