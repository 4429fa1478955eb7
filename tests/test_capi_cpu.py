"""CPU tests of the product library: it loads, exports every symbol the C
header declares, refuses to run without a GPU (no CPU fallback), and its host
generators produce the BASELINE matrices (checked against scipy constructions)."""
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "rkmf_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rkmf_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(rk):
    import ctypes
    L = ctypes.CDLL(rk.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(s[0] for s in rk.SYMBOLS) == declared


def test_no_cpu_fallback(rk):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rk.Error):
        rk.Context(0)


def test_kernels_are_sm100a(rk):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rk.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _csr(rp, ci, v):
    n = len(rp) - 1
    return sp.csr_matrix((v, ci, rp), shape=(n, n))


def lap1d(N):
    h = 1.0 / (N + 1)
    return sp.diags([-np.ones(N - 1), 2 * np.ones(N), -np.ones(N - 1)], [-1, 0, 1]) / h**2


def test_gen_laplacian_matches_kron(rk):
    for dim, N, nnz in [(2, 256, 326656), (3, 12, 7 * 12**3 - 6 * 144)]:
        rp, ci, v = rk.gen_laplacian(dim, N)
        assert rp[-1] == nnz
        T, I = lap1d(N), sp.eye(N)
        if dim == 2:
            K = sp.kron(T, I) + sp.kron(I, T)
        else:
            K = sp.kron(sp.kron(T, I), I) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(I, I), T)
        A = _csr(rp, ci, v)
        assert abs(A - K.tocsr()).max() <= 1e-9 * abs(K).max()
        assert all((np.diff(ci[rp[i]:rp[i + 1]]) > 0).all() for i in range(0, len(rp) - 1, 97))


def test_cfg_sizes_match_baseline(rk):
    # nnz quoted in BASELINE.json / SURVEY.md §8
    n, nnz = rk.lib().rkmf_gen_laplacian, None
    import ctypes as C
    for fn, args, want in [
        (rk.lib().rkmf_gen_laplacian, (3, 128), (2097152, 14581760)),
        (rk.lib().rkmf_gen_q1_hex, (200, 1, C.c_uint64(1), 1), (8000000, 213847192)),
        (rk.lib().rkmf_gen_convdiff_upwind, (256, 10.0, 1.0, 0.5, 0.25), (16777216, 117047296)),
        (rk.lib().rkmf_gen_q1_hex, (512, 0, C.c_uint64(1), 0), (134217728, 3609741304)),
    ]:
        a, b = C.c_int64(), C.c_int64()
        assert fn(*args, C.byref(a), C.byref(b), None, None, None) == 0
        assert (a.value, b.value) == want


def test_gen_q1_properties(rk):
    N = 7
    rp, ci, v = rk.gen_q1_hex(N, False, 1, False)
    A = _csr(rp, ci, v)
    assert rp[-1] == (3 * N - 2) ** 3
    assert abs(A - A.T).max() < 1e-15
    assert np.abs(A @ np.ones(N**3)).max() < 1e-14  # pure Neumann: constants in the kernel
    h = 1.0 / (N - 1)
    c = (3 * N**2 + 3 * N + 1) // 1
    mid = ((N // 2) * N + N // 2) * N + N // 2
    row = A.getrow(mid).toarray().ravel()
    assert row[mid] == pytest.approx(h * 8 / 3, rel=1e-14)
    assert row[mid + 1] == 0.0
    assert row[mid + N + 1] == pytest.approx(-h / 6, rel=1e-14)
    assert row[mid + N * N + N + 1] == pytest.approx(-h / 12, rel=1e-14)
    # lognormal + Dirichlet: SPD, identity boundary rows, pattern kept
    rp2, ci2, v2 = rk.gen_q1_hex(N, True, 1, True)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)
    B = _csr(rp2, ci2, v2).toarray()
    assert np.abs(B - B.T).max() < 1e-15
    assert np.linalg.eigvalsh(B).min() > 0
    assert B[0, 0] == 1.0 and np.count_nonzero(B[0]) == 1


def test_gen_convdiff_upwind(rk):
    N = 9
    rp, ci, v = rk.gen_convdiff_upwind(N, 10.0, (1.0, 0.5, 0.25))
    A = _csr(rp, ci, v).toarray()
    assert rp[-1] == 7 * N**3 - 6 * N**2
    off = A - np.diag(np.diag(A))
    assert (off <= 0).all()  # M-matrix sign pattern
    assert (np.diag(A) + off.sum(1) >= -1e-9).all()  # weakly diagonally dominant
    h = 1.0 / (N + 1)
    eps = 1.0 * h / (2 * 10.0)
    c = (N // 2 * N + N // 2) * N + N // 2
    assert A[c, c - N * N] == pytest.approx(-eps / h**2 - 1.0 / h)  # upwind in x
    assert A[c, c + N * N] == pytest.approx(-eps / h**2)


def test_gaussian_matches_oracle(rk, oracle):
    assert np.array_equal(rk.gen_gaussian(1, 1000), oracle.gaussian_vector(1, 1000))


def test_algorithmic_bytes_formula():
    from paper_2503_22631_b200 import configs
    # cfg2 34.84 GB / cycle
    b = configs.algorithmic_bytes_per_cycle(2097152, 14581760, 50)
    assert abs(b / 1e9 - 34.84) < 0.05
