"""The oracle pinned against the REFERENCE'S OWN sources.

`oracle/_ref/librkmf_ref.so` is /root/reference/proj/src/{restart, basis,
sketch, sparse, densefun, approximants, leastsq}.cpp compiled unmodified
(oracle/Makefile target `ref`) against the Eigen-API stand-in
oracle/eigen_standin (Eigen is not on the image). Two layers:

* golden: tests/golden/ref_pin.npz holds outputs of that library
  (tests/golden/make_ref_golden.py). The contraction-free oracle build
  (liboracle_strict.so) must reproduce them BIT FOR BIT, the shipped oracle
  (FMA contraction) to rounding. These run anywhere.
* live: where the library is present (the build container, and the GPU box,
  to which it travels) the same comparisons run against it directly, plus
  error behaviour and the Matrix Market reader/writer of the product's host
  side (csrc/mtx.cpp) against the reference's (sparse.cpp:140-242).

What this pins is the reference's algorithm as its source text states it; the
rounding order of Eigen's own kernels is not reproducible without Eigen.
"""
import os

import numpy as np
import pytest

from tests import helpers as H
from tests import ref_cases

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_pin.npz")
CASE_NAMES = list(ref_cases.CASES)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def strict():
    from oracle import ref as R
    return R.strict()


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    R.build()
    if not R.available():
        pytest.skip("oracle/_ref is not built here (needs /root/reference at build time)")
    R.front()
    return R


def _solve(O, P, Sk, **kw):
    return O.restarted_krylov(P["A"], P["b"], 0, P["t"], m_r=P["m"], tol=P["tol"],
                              k_max=P["k_max"], S=Sk, want_R=True, **kw)


# ---------------------------------------------------------------- golden ----
@pytest.mark.parametrize("name", CASE_NAMES)
def test_strict_oracle_reproduces_reference_fixture_bit_for_bit(strict, gold, name):
    O = strict
    P = ref_cases.build(name, O)
    S = O.make_sketch(P["d"], P["n"], P["zeta"], P["seed"])
    assert np.array_equal(S.rows.astype(np.int16), gold[f"{name}/sketch_rows"])
    assert np.array_equal(S.signs, gold[f"{name}/sketch_signs"])
    assert np.array_equal(O.sketch_apply(S, P["b"]), gold[f"{name}/Sb"])
    assert np.array_equal(O.spmv(P["A"], P["b"]), gold[f"{name}/Ab"])
    assert O.norm1(P["A"]) == gold[f"{name}/norm1"][0]
    dec = O.arnoldi_decomp(P["A"], P["b"], P["m"], S)
    assert np.array_equal(dec.U, gold[f"{name}/dec_U"])
    assert np.array_equal(dec.Rbar, gold[f"{name}/dec_Rbar"])
    assert np.array_equal(dec.W[:, -1], gold[f"{name}/dec_w_last"])
    assert dec.start_norm == gold[f"{name}/dec_start_norm"][0]
    assert list(dec.counters.values()) == gold[f"{name}/dec_counters"].tolist()
    for tag, Sk in (("rand", S), ("classical", None)):
        r = _solve(O, P, Sk)
        assert [r.cycles, r.total_m, int(r.converged)] == gold[f"{name}/{tag}_meta"].tolist()
        assert np.array_equal(r.f_hat, gold[f"{name}/{tag}_f"])
        assert np.array_equal(r.R_accum, gold[f"{name}/{tag}_R_accum"])
        assert np.array_equal([h["update_norm"] for h in r.history],
                              gold[f"{name}/{tag}_update_norm"])
        assert np.array_equal([h["alpha_dev"] for h in r.history], gold[f"{name}/{tag}_alpha_dev"])
        assert r.alpha == gold[f"{name}/{tag}_alpha"][0]
        assert list(r.counters.values()) == gold[f"{name}/{tag}_counters"].tolist()


@pytest.mark.parametrize("name", CASE_NAMES)
def test_shipped_oracle_matches_reference_fixture_to_rounding(oracle, gold, name):
    O = oracle
    P = ref_cases.build(name, O)
    S = O.make_sketch(P["d"], P["n"], P["zeta"], P["seed"])
    for tag, Sk in (("rand", S), ("classical", None)):
        r = _solve(O, P, Sk)
        f = gold[f"{name}/{tag}_f"]
        assert [r.cycles, r.total_m, int(r.converged)] == gold[f"{name}/{tag}_meta"].tolist()
        assert np.linalg.norm(r.f_hat - f) <= 1e-12 * np.linalg.norm(f)
        un = gold[f"{name}/{tag}_update_norm"]
        got = np.array([h["update_norm"] for h in r.history])
        # the last update is ~tol: a difference of rounding size in f is a large relative one there
        assert np.all(np.abs(got - un) <= 1e-9 * un + 1e-12 * un[0])
        assert list(r.counters.values()) == gold[f"{name}/{tag}_counters"].tolist()


def test_funm_fixture(strict, oracle, gold):
    X = gold["funm/X"]
    assert np.array_equal(X, ref_cases.dense_f_input())
    for t in (0.05, 0.7, 3.0):
        F = gold[f"funm/F_t{t}"]
        assert np.array_equal(strict.funm(X, 0, t), F)
        assert np.abs(oracle.funm(X, 0, t) - F).max() <= 1e-13 * np.abs(F).max()


def test_next_below_fixture(gold):  # rng.hpp:34-43 against the pure-Python restatement
    def below(seed, bound, count):
        st, out = [seed], []
        limit = (bound * (H.M64 // bound)) & H.M64
        for _ in range(count):
            while True:
                v = H.sm64_next(st)
                if v < limit:
                    break
            out.append(v % bound)
        return out
    assert below(99, 1000, 256) == gold["rng/below_1000"].tolist()
    assert below(7, (1 << 63) + 12345, 64) == gold["rng/below_big"].tolist()


# ------------------------------------------------------------------ live ----
def test_fixture_is_current(ref, gold):
    """The committed fixture is what the library produces now."""
    O = ref.front()
    name = CASE_NAMES[0]
    P = ref_cases.build(name, O)
    S = O.make_sketch(P["d"], P["n"], P["zeta"], P["seed"])
    r = _solve(O, P, S)
    assert np.array_equal(r.f_hat, gold[f"{name}/rand_f"])
    assert np.array_equal(r.R_accum, gold[f"{name}/rand_R_accum"])


def test_rng_and_sketch_bit_exact_live(ref, oracle):
    Rf = ref.front()
    for seed in (0, 1, 42, 2**63 + 5):
        assert np.array_equal(oracle.splitmix_stream(seed, 512), Rf.splitmix_stream(seed, 512))
        assert oracle.splitmix_derive(seed, 17) == Rf.splitmix_derive(seed, 17)
        assert np.array_equal(oracle.gaussian_vector(seed, 300), Rf.gaussian_vector(seed, 300))
    for (d, n, z, s) in [(40, 300, 5, 123), (24, 24, 24, 9), (30, 200, 1, 5), (120, 4096, 8, 1),
                         (160, 100003, 8, 3), (800, 5000, 8, 11)]:
        a, b = oracle.make_sketch(d, n, z, s), Rf.make_sketch(d, n, z, s)
        assert np.array_equal(a.rows, b.rows) and np.array_equal(a.signs, b.signs)
        assert a.scale == b.scale


@pytest.mark.parametrize("seed", range(6))
def test_random_nonsymmetric_instances_bit_identical_live(ref, strict, seed):
    """test_basis.cpp:89-111's instance family through both implementations."""
    Rf = ref.front()
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(60, 400))
    m = int(rng.integers(3, 25))
    zeta = int(rng.integers(1, 6))
    d = int(rng.integers(max(m + 1, zeta), 3 * m + 8))
    A = H.random_sparse(n, 0.05, 200 + seed, shift=4.0)
    b = H.random_vector(n, 300 + seed)
    S = strict.make_sketch(d, n, zeta, 400 + seed)
    a, c = strict.arnoldi_decomp(A, b, m, S), Rf.arnoldi_decomp(A, b, m, S)
    assert np.array_equal(a.W, c.W) and np.array_equal(a.U, c.U)
    assert np.array_equal(a.Rbar, c.Rbar) and a.counters == c.counters
    a, c = strict.arnoldi_decomp(A, b, m), Rf.arnoldi_decomp(A, b, m)
    assert np.array_equal(a.W, c.W) and np.array_equal(a.Rbar, c.Rbar) and a.counters == c.counters
    t = 2.0 / strict.norm1(A)
    for Sk in (S, None):
        x = strict.restarted_krylov(A, b, 0, t, m_r=m, tol=1e-10, k_max=30, S=Sk, want_R=True)
        y = Rf.restarted_krylov(A, b, 0, t, m_r=m, tol=1e-10, k_max=30, S=Sk, want_R=True)
        assert (x.cycles, x.total_m, x.converged) == (y.cycles, y.total_m, y.converged)
        assert np.array_equal(x.f_hat, y.f_hat) and np.array_equal(x.R_accum, y.R_accum)


def test_happy_breakdown_and_saturation_live(ref, strict):
    """m = n (the Krylov space saturates, basis.cpp:131) and an invariant
    subspace (breakdown before m): same kept sizes, same bytes."""
    Rf = ref.front()
    A = H.random_spd_tridiag(12, 1.0, 9.0, 5)
    b = H.random_vector(12, 6)
    S = strict.make_sketch(12, 12, 3, 1)
    for Sk in (S, None):
        a, c = strict.arnoldi_decomp(A, b, 12, Sk), Rf.arnoldi_decomp(A, b, 12, Sk)
        assert a.m == c.m == 12 and a.breakdown_at == c.breakdown_at == 12
        assert a.Rbar.shape == c.Rbar.shape and np.array_equal(a.Rbar, c.Rbar)
        assert np.array_equal(a.W, c.W)
    import scipy.sparse as sp
    D = sp.diags([np.array([1.0, 2.0, 3.0] * 10)], [0]).tocsr()  # 3 distinct eigenvalues
    b = np.ones(30)
    S = strict.make_sketch(20, 30, 2, 9)
    a, c = strict.arnoldi_decomp(D, b, 8, S), Rf.arnoldi_decomp(D, b, 8, S)
    assert a.breakdown_at == c.breakdown_at and a.m == c.m and a.m < 8
    x = strict.restarted_krylov(D, b, 0, 0.5, m_r=8, tol=1e-12, S=S)
    y = Rf.restarted_krylov(D, b, 0, 0.5, m_r=8, tol=1e-12, S=S)
    assert x.converged and y.converged and x.cycles == y.cycles == 1
    assert np.array_equal(x.f_hat, y.f_hat)


def test_error_behaviour_live(ref, oracle):
    """Same exception class and message (restart.cpp:34-39, basis.cpp:14-23,
    97-101, sparse.cpp:61-81, sketch.cpp:14-16, restart.cpp:82-89)."""
    Rf = ref.front()
    A = H.random_spd_tridiag(120, 1.0, 9.0, 31)
    b = H.random_vector(120, 32)
    S = oracle.make_sketch(40, 120, 4, 1)

    def both(fn):
        out = []
        for M in (oracle, Rf):
            with pytest.raises(M.OracleError) as e:
                fn(M)
            out.append((e.value.kind, str(e.value)))
        assert out[0] == out[1], out
        return out[0]

    for kw in [dict(m_r=0), dict(k_max=0), dict(tol=0.0), dict(m_r=10, budget_total_m=5)]:
        assert both(lambda M: M.restarted_krylov(A, b, 0, 1.0, S=S, **kw))[0] == "ParameterError"
    both(lambda M: M.restarted_krylov(A, np.zeros(120), 0, 1.0, S=S))  # zero start vector
    both(lambda M: M.restarted_krylov(A, np.zeros(120), 0, 1.0, S=None))
    both(lambda M: M.arnoldi_decomp(A, b, 45, S))  # d too small for m
    both(lambda M: M.arnoldi_decomp(A, b, 0, S))
    both(lambda M: M.arnoldi_decomp(A, b, 121, S))
    both(lambda M: M.make_sketch(4, 10, 5, 1))
    both(lambda M: M.make_sketch(4, 10, 0, 1))
    both(lambda M: M.make_sketch(11, 10, 2, 1))
    bad = (A.indptr.astype(np.int64), A.indices[::-1].astype(np.int32).copy(), A.data.copy(), 120)
    both(lambda M: M.validate(bad))
    nanv = A.data.copy(); nanv[7] = np.nan
    both(lambda M: M.validate((A.indptr.astype(np.int64), A.indices.astype(np.int32), nanv, 120)))
    # divergence guard (test_restart.cpp:231-246)
    C = H.conv_diff_2d(60, 60, 0.001, 10.0, 0.0)
    bc = H.random_vector(C.shape[0], 1)
    S6 = oracle.make_sketch(6, C.shape[0], 1, 3)
    kind, msg = both(lambda M: M.restarted_krylov(C, bc, 0, 10.0 / oracle.norm1(C), m_r=5,
                                                  tol=1e-12, k_max=60, S=S6))
    assert kind == "NumericalError" and msg.startswith("restart divergence")
    # k_max / budget semantics (test_restart.cpp:209-229)
    for kw in [dict(k_max=3), dict(k_max=50, budget_total_m=25)]:
        x = oracle.restarted_krylov(A, b, 0, 1.0, m_r=10, tol=1e-30, S=S, **kw)
        y = Rf.restarted_krylov(A, b, 0, 1.0, m_r=10, tol=1e-30, S=S, **kw)
        assert (x.cycles, x.total_m, x.converged) == (y.cycles, y.total_m, y.converged)


def test_matrix_market_reader_writer_against_the_reference_live(ref, rk, tmp_path):
    """csrc/mtx.cpp against sparse.cpp:140-242: the same bytes on disk, the
    same CSR back, the same line-numbered errors."""
    A = H.random_sparse(40, 0.1, 21, shift=3.7)
    csr = (A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.copy(), 40)
    p1, p2 = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    rk.save_matrix_market(csr, p1)
    ref.save_mtx(p2, csr[0], csr[1], csr[2], 40)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    for p in (p1, p2):
        a, b = rk.load_matrix_market(p), ref.load_mtx(p)
        for u, w in zip(a, b):
            assert np.array_equal(u, w)
    x = H.random_vector(57, 3) * 1e-7
    v1, v2 = str(tmp_path / "ours.vec"), str(tmp_path / "ref.vec")
    rk.save_vector(x, v1)
    ref.save_vector(v2, x)
    assert open(v1, "rb").read() == open(v2, "rb").read()
    assert np.array_equal(rk.load_vector(v2), x) and np.array_equal(ref.load_vector(v1), x)
    texts = {
        "sym": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 2.0\n2 1 -1.0\n3 2 0.5\n3 3 4.0\n",
        "dup": "%%MatrixMarket MATRIX Coordinate REAL General\n% c\n2 3 4\n2 3 1.5\n1 2 1.0\n2 3 0.25\n1 1 -2\n",
        "upper": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n",
        "trailing": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0 7\n",
        "blank": "%%MatrixMarket matrix coordinate real general\n\n2 2 1\n\n1 1 1.0\n",
        "banner": "%%NotMatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n",
        "format": "%%MatrixMarket matrix array real general\n2 2\n1.0\n",
        "field": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1.0 0.0\n",
        "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n",
        "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1.0\n",
        "range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
        "short": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
        "extra": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n",
        "token": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n",
        "nan": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n",
        "size": "%%MatrixMarket matrix coordinate real general\n2 two 1\n1 1 1.0\n",
        "neg": "%%MatrixMarket matrix coordinate real general\n-2 2 1\n1 1 1.0\n",
        "empty": "",
    }
    raised = 0
    for k, text in texts.items():
        p = tmp_path / f"{k}.mtx"
        p.write_text(text)
        out = []
        for load in (rk.load_matrix_market, ref.load_mtx):
            try:
                out.append(("ok", [np.asarray(x).tolist() for x in load(str(p))]))
            except Exception as e:  # the product's ParseError / RefError(kind ParseError)
                out.append(("ParseError", str(e)))
                assert type(e).__name__ == "ParseError" or getattr(e, "kind", "") == "ParseError"
                raised += 1
        assert out[0] == out[1], (k, out)
    assert raised == 2 * 13
    for name, load in (("vec_bad", rk.load_vector), ("vec_bad", ref.load_vector)):
        p = tmp_path / "bad.vec"
        p.write_text("1.0\n% comment\n\n2.0 3.0\n")
    msgs = []
    for load in (rk.load_vector, ref.load_vector):
        with pytest.raises(Exception) as e:
            load(str(tmp_path / "bad.vec"))
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] and ":4:" in msgs[0]
