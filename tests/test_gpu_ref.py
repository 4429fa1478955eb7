"""The device path against the REFERENCE'S OWN sources (oracle/_ref) and the
fixture frozen from them (tests/golden/ref_pin.npz).

oracle/_ref/librkmf_ref.so is /root/reference/proj/src/{restart, basis, sketch,
sparse, densefun, approximants, leastsq}.cpp compiled unmodified against the
Eigen-API stand-in (oracle/eigen_standin; tests/test_ref_pin.py has the
details). The library travels to the GPU box with the snapshot; where it is
absent the live tests skip and the fixture tests still hold the device path
to the reference's bytes. Bars are BASELINE.json's: f_hat within 1e-9 relative
2-norm, restart-cycle counts equal (the north star allows +-1).
"""
import os

import numpy as np
import pytest

from tests import ref_cases

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_pin.npz")


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref did not travel with this snapshot")
    return R


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def _device_case(rk, torch, P, sketched=True, **kw):
    rp, ci, v, n = P["A"]
    A = rk.SparseMatrix.from_csr(rp, ci, v)
    S = rk.make_sketch(P["d"], n, P["zeta"], P["seed"]) if sketched else None
    opts = rk.RestartOptions(m_r=P["m"], tol=P["tol"], k_max=P["k_max"], **kw)
    return rk.restarted_krylov(A, torch.tensor(P["b"], device="cuda"),
                               rk.FunctionSpec.exp_neg(P["t"]), opts, S, keep_R_accum=True)


@pytest.mark.parametrize("name", list(ref_cases.CASES))
@pytest.mark.parametrize("builder", ["rand", "classical"])
def test_device_matches_reference_fixture(rk, torch, gold, name, builder):
    P = ref_cases.build(name)
    r = _device_case(rk, torch, P, sketched=(builder == "rand"))
    cycles, total_m, converged = gold[f"{name}/{builder}_meta"].tolist()
    assert (r.cycles, r.total_m, int(r.converged)) == (cycles, total_m, converged)
    f = gold[f"{name}/{builder}_f"]
    assert _rel(r.f_hat.cpu().numpy(), f) <= 1e-9
    assert r.alpha == pytest.approx(gold[f"{name}/{builder}_alpha"][0], rel=1e-13)
    un = gold[f"{name}/{builder}_update_norm"]
    got = np.array([h.update_norm for h in r.history])
    assert np.all(np.abs(got - un) <= 1e-6 * un + 1e-10 * un[0])
    R = gold[f"{name}/{builder}_R_accum"]
    assert np.abs(np.asarray(r.R_accum) - R).max() <= 1e-6 * np.abs(R).max()
    assert [r.counters[k] for k in ("matvecs", "dot_n", "dot_d", "basis_updates",
                                    "peak_basis_cols")] == \
        gold[f"{name}/{builder}_counters"].tolist()


@pytest.mark.parametrize("name", list(ref_cases.CASES))
def test_device_diagnostics_match_reference_fixture(rk, torch, gold, name):
    """kappa_W and the leftmost Ritz value of every cycle (restart.cpp:101,103;
    approximants.cpp:29-47) against the reference's CycleRecords."""
    P = ref_cases.build(name)
    r = _device_case(rk, torch, P, diagnostics=True)
    kap = gold[f"{name}/rand_kappa_W"]
    ritz = gold[f"{name}/rand_ritz_left"]
    assert len(r.history) == len(kap)
    for h, k, z in zip(r.history, kap, ritz):
        assert h.kappa_W == pytest.approx(k, rel=1e-6)
        assert h.leftmost_ritz_re == pytest.approx(z, rel=1e-6, abs=1e-9 * np.abs(ritz).max())


@pytest.mark.parametrize("cfg,N", [("cfg1", None), ("cfg2", 44), ("cfg4", 40), ("cfg5", 24)])
def test_device_matches_reference_sources_on_baseline_kinds(rk, torch, ref, cfg, N):
    """BASELINE.json's problem kinds through the reference's restarted_krylov
    itself: cfg1 at its full size (65,536 rows), the others on grids the
    single-threaded reference finishes in seconds."""
    from paper_2503_22631_b200 import configs
    P = configs.build(cfg) if N is None else configs.build(cfg, N)
    Rf = ref.front()
    S = Rf.make_sketch(P.d, P.n, P.zeta, 1)
    q = Rf.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, 0, P.t, m_r=P.m, tol=P.tol,
                            k_max=P.k_max, S=S, want_R=True)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    Sd = rk.make_sketch(P.d, P.n, P.zeta, 1)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max, diagnostics=True)
    r = rk.restarted_krylov(A, torch.tensor(P.b, device="cuda"), rk.FunctionSpec.exp_neg(P.t),
                            opts, Sd, keep_R_accum=True)
    assert r.converged and q.converged and r.cycles == q.cycles and r.total_m == q.total_m
    assert _rel(r.f_hat.cpu().numpy(), q.f_hat) <= 1e-9
    assert np.abs(np.asarray(r.R_accum) - q.R_accum).max() <= 1e-6 * np.abs(q.R_accum).max()
    for h, g in zip(r.history, q.history):
        assert h.update_norm == pytest.approx(g["update_norm"], rel=1e-5, abs=1e-3 * P.tol)
        assert h.kappa_W == pytest.approx(g["kappa_W"], rel=1e-6)
        assert h.leftmost_ritz_re == pytest.approx(g["leftmost_ritz_re"], rel=1e-6)
    assert r.counters == q.counters


def test_device_sketch_and_decomposition_match_reference_sources(rk, torch, ref):
    from paper_2503_22631_b200 import configs
    P = configs.build("cfg4", 24)
    Rf = ref.front()
    S = Rf.make_sketch(P.d, P.n, P.zeta, 7)
    Sd = rk.make_sketch(P.d, P.n, P.zeta, 7)
    rows, signs, _ = Sd.export()
    assert np.array_equal(rows, S.rows) and np.array_equal(signs, S.signs)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    dec = rk.randomized_arnoldi(A, Sd, torch.tensor(P.b, device="cuda"), P.m)
    q = Rf.arnoldi_decomp((P.row_ptr, P.col_idx, P.values), P.b, P.m, S)
    assert np.abs(dec.W.cpu().numpy() - q.W).max() <= 1e-10
    assert np.abs(dec.U.cpu().numpy() - q.U).max() <= 1e-10
    assert np.abs(np.asarray(dec.Rbar) - q.Rbar).max() <= 1e-10 * np.abs(q.Rbar).max()
    assert dec.start_norm == pytest.approx(q.start_norm, rel=1e-13)


def test_solve_on_a_file_written_by_the_reference(rk, torch, ref, tmp_path):
    """The external-problem workflow (problems.cpp:494-508): the reference
    writes A and b, the device side loads them and solves; same f_hat."""
    P = ref_cases.build("convdiff_N10")
    rp, ci, v, n = P["A"]
    pa, pb = str(tmp_path / "A.mtx"), str(tmp_path / "b.vec")
    ref.save_mtx(pa, rp, ci, v, n)
    ref.save_vector(pb, P["b"])
    A = rk.SparseMatrix.from_mtx(pa)
    b = rk.load_vector(pb)
    assert np.array_equal(b, P["b"])
    S = rk.make_sketch(P["d"], n, P["zeta"], P["seed"])
    r = rk.restarted_krylov(A, torch.tensor(b, device="cuda"), rk.FunctionSpec.exp_neg(P["t"]),
                            rk.RestartOptions(m_r=P["m"], tol=P["tol"], k_max=P["k_max"]), S)
    Rf = ref.front()
    q = Rf.restarted_krylov(ref.load_mtx(pa)[:3] + (n,), ref.load_vector(pb), 0, P["t"],
                            m_r=P["m"], tol=P["tol"], k_max=P["k_max"],
                            S=Rf.make_sketch(P["d"], n, P["zeta"], P["seed"]))
    assert r.cycles == q.cycles and _rel(r.f_hat.cpu().numpy(), q.f_hat) <= 1e-9


def test_device_sweep_matches_reference_sweep(rk, torch, ref):
    """restart::convergence_sweep (restart.cpp:124-305) row by row: restarted
    methods on the device against the reference's own sweep on the same
    {A, b, ExpNeg(t)}; error cells carry the reference's sanitised messages."""
    P = ref_cases.build("lap3d_N20_cfg1shape")
    rp, ci, v, n = P["A"]
    ms = [rk.MethodSpec("restart-rand", m=P["m"], d=P["d"], zeta=P["zeta"], tol=P["tol"],
                        k_max=P["k_max"], seed=P["seed"]),
          rk.MethodSpec("restart-rand", m=12, tol=P["tol"], k_max=60, seed=9),  # d = 16 m, zeta 4
          rk.MethodSpec("restart", m=P["m"], tol=P["tol"], k_max=P["k_max"]),
          rk.MethodSpec("rand", m=24, seed=5),                      # one-shot: d = 4 m, cycle 0
          rk.MethodSpec("rand", m=P["m"], d=P["d"], zeta=P["zeta"], seed=P["seed"]),
          rk.MethodSpec("arnoldi", m=18),
          rk.MethodSpec("rand", m=0),
          rk.MethodSpec("bogus"),
          rk.MethodSpec("restart-rand", m=0),
          rk.MethodSpec("restart", m=10, tol=0.0)]
    exact = ref.front().restarted_krylov(P["A"], P["b"], 0, P["t"], m_r=40, tol=1e-13, S=None).f_hat
    want = ref.convergence_sweep(P["A"], P["b"], P["t"], ms, reference=exact)
    A = rk.SparseMatrix.from_csr(rp, ci, v)
    got = rk.convergence_sweep(A, P["b"], rk.FunctionSpec.exp_neg(P["t"]), ms, reference=exact)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for k in ("method", "n", "m_or_totalm", "cycle", "matvecs", "note"):
            assert g[k] == w[k], (k, g, w)
        if w["note"]:
            assert np.isnan(g["rel_error"]) and np.isnan(w["rel_error"])
            continue
        assert g["update_norm"] == pytest.approx(w["update_norm"], rel=1e-5, abs=1e-3 * P["tol"])
        assert g["rel_error"] == pytest.approx(w["rel_error"], rel=1e-4, abs=1e-12)
        assert g["kappa_W"] == pytest.approx(w["kappa_W"], rel=1e-6)
        assert g["leftmost_ritz_re"] == pytest.approx(w["leftmost_ritz_re"], rel=1e-6)
