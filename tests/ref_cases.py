"""Inputs of the reference pins (tests/test_ref_pin.py, tests/test_gpu_ref.py,
tests/golden/make_ref_golden.py): small seeded problems built from the oracle's
generators (oracle/problems_oracle.cpp) and tests/helpers.py, so the same
bytes reach the reference's sources (oracle/_ref), the oracle and the device."""
from __future__ import annotations

import numpy as np

from tests import helpers as H

# name -> (builder, m, d, zeta, sketch_seed, t_scale, tol_rel, k_max)
#   t = t_scale / norm1(A); tol = tol_rel * ||b||
CASES = {
    "lap3d_N12": ("lap3d", 12, 20, 80, 8, 1, 12.0, 1e-9, 40),
    "lap3d_N20_cfg1shape": ("lap3d", 20, 30, 120, 8, 1, 8.0, 1e-10, 40),
    "convdiff_N10": ("convdiff", 10, 20, 80, 8, 2, 6.0, 1e-9, 40),
    "q1_lognormal_N8": ("q1", 8, 16, 64, 4, 3, 10.0, 1e-8, 60),
    "centred_convdiff_2d": ("cd2d", 24, 12, 48, 2, 5, 4.0, 1e-9, 60),
    "zeta1_tridiag": ("tridiag", 300, 10, 40, 1, 7, 5.0, 1e-10, 60),
}


def build(name, O=None):
    """Inputs always come from the contraction-free oracle build (O is kept for
    call-site symmetry and ignored), so every implementation sees the same bytes."""
    from oracle import ref as _R
    O = _R.strict()
    kind, N, m, d, zeta, seed, t_scale, tol_rel, k_max = CASES[name]
    if kind == "lap3d":
        rp, ci, v = O.gen_laplacian(3, N)
    elif kind == "convdiff":
        rp, ci, v = O.gen_convdiff_upwind(N, 10.0)
    elif kind == "q1":
        rp, ci, v = O.gen_q1_hex(N, lognormal=True, coef_seed=4, dirichlet=True)
    elif kind == "cd2d":
        A = H.conv_diff_2d(N, N, 0.02, 1.0, 0.5)
        rp, ci, v = A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.copy()
    elif kind == "tridiag":
        A = H.random_spd_tridiag(N, 1.0, 9.0, 31)
        rp, ci, v = A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.copy()
    else:
        raise KeyError(kind)
    n = len(rp) - 1
    A = (rp, ci, v, n)
    b = O.gaussian_vector(seed, n)
    t = t_scale / O.norm1(A)
    return dict(A=A, n=n, b=b, t=t, m=m, d=d, zeta=zeta, seed=seed,
                tol=tol_rel * float(np.linalg.norm(b)), k_max=k_max)


def dense_f_input(n: int = 48, seed: int = 11) -> np.ndarray:
    """An upper Hessenberg block pattern like R_accum, large enough in norm
    that expm scales and squares (densefun.cpp:127-131)."""
    rng = np.random.default_rng(seed)
    X = np.triu(rng.standard_normal((n, n)), -1)
    return X + 6.0 * np.eye(n)
