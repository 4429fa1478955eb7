"""The product's host generators (csrc/problems.cpp, in librkmf_b200.so)
against the independent restatement in oracle/problems_oracle.cpp: the same
CSR arrays and b bit-for-bit (no GPU needed: host-only entry points).
The device generators are checked against these in tests/test_gpu_parity.py."""
import numpy as np
import pytest


@pytest.mark.parametrize("args", [(2, 1), (2, 37), (2, 256), (3, 1), (3, 19), (3, 40)])
def test_laplacian_matches_oracle(rk, oracle, args):
    for a, b in zip(rk.gen_laplacian(*args), oracle.gen_laplacian(*args)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("args", [(2, False, 1, False), (9, False, 1, False), (11, True, 1, True),
                                  (13, True, 5, False), (24, True, 1, True)])
def test_q1_hex_matches_oracle(rk, oracle, args):
    for a, b in zip(rk.gen_q1_hex(*args), oracle.gen_q1_hex(*args)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("args", [(1,), (17,), (9, 3.0, (-1.0, 0.5, 2.0)), (48, 10.0, (1.0, 0.5, 0.25))])
def test_convdiff_matches_oracle(rk, oracle, args):
    for a, b in zip(rk.gen_convdiff_upwind(*args), oracle.gen_convdiff_upwind(*args)):
        assert np.array_equal(a, b)


def test_gaussian_matches_oracle(rk, oracle):
    assert np.array_equal(rk.gen_gaussian(1, 200003), oracle.gaussian_vector(1, 200003))
    assert np.array_equal(rk.gen_gaussian_range(1, 777, 5000),
                          oracle.gaussian_vector(1, 5777)[777:])


@pytest.mark.parametrize("name,N", [("cfg1", None), ("cfg2", 24), ("cfg3", 12), ("cfg4", 20),
                                    ("cfg5", 10)])
def test_config_backends_agree(name, N):
    """configs.build with the product generators and with the oracle's give
    the same problem (arrays, b, t, tol): the bench's two arms see one input."""
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    Q = configs.build(name, N, backend="oracle")
    for f in ("row_ptr", "col_idx", "values", "b"):
        assert np.array_equal(getattr(P, f), getattr(Q, f)), f
    assert (P.t, P.tol, P.m, P.d, P.k_max) == (Q.t, Q.tol, Q.m, Q.d, Q.k_max)
