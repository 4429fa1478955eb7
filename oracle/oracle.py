"""ctypes front-end of the CPU oracle (liboracle.so) — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module. The product package ``paper_2503_22631_b200`` never does.

Every function restates a reference function (see rkmf_oracle.cpp for the
file:line map into /root/reference/proj): SplitMix64 (rng.hpp:17-63),
make_sketch / sketch_apply (sketch.cpp:13-63), spmv / norm1 / validate
(sparse.cpp:61-102), randomized and classical Arnoldi (basis.cpp:34-142),
funm / expm (densefun.cpp:119-157, 429-450) and restarted_krylov
(restart.cpp:27-122).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

KIND_EXP_NEG = 0
KIND_INV_SQRT = 4

_ERR_CLASSES = {1: "ParameterError", 2: "ShapeError", 3: "NumericalError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = _ERR_CLASSES.get(code, "Error")


class CycleRecord(C.Structure):
    _fields_ = [("cycle", C.c_int64), ("total_m", C.c_int64), ("total_matvecs", C.c_int64),
                ("update_norm", C.c_double), ("error_vs_reference", C.c_double),
                ("kappa_W", C.c_double), ("leftmost_ritz_re", C.c_double),
                ("alpha_dev", C.c_double), ("elapsed_ms", C.c_double), ("build_ms", C.c_double),
                ("funm_ms", C.c_double), ("start_norm", C.c_double), ("subdiag", C.c_double)]


class Result(C.Structure):
    _fields_ = [("converged", C.c_int64), ("cycles", C.c_int64), ("total_m", C.c_int64),
                ("alpha", C.c_double), ("matvecs", C.c_int64), ("dot_n", C.c_int64),
                ("dot_d", C.c_int64), ("basis_updates", C.c_int64),
                ("peak_basis_cols", C.c_int64), ("n_records", C.c_int64)]


def build() -> str:
    """Compile liboracle.so with the committed Makefile (g++ only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, u64, d, i32 = C.c_int64, C.c_uint64, C.c_double, C.c_int
        L.orc_splitmix_derive.restype = u64
        L.orc_splitmix_derive.argtypes = [u64, u64]
        L.orc_splitmix_stream.argtypes = [u64, i64, P]
        L.orc_gaussian_vector.argtypes = [u64, i64, P]
        L.orc_make_sketch.argtypes = [i64, i64, i64, u64, P, P, P, C.c_char_p]
        L.orc_sketch_apply.argtypes = [i64, i64, i64, P, P, d, P, P]
        L.orc_spmv.argtypes = [i64, i64, P, P, P, P, P, i32]
        L.orc_norm1.restype = d
        L.orc_norm1.argtypes = [i64, i64, P, P, P]
        L.orc_validate.argtypes = [i64, i64, P, P, P, C.c_char_p]
        L.orc_funm.argtypes = [i64, P, i32, d, P, C.c_char_p]
        L.orc_arnoldi_decomp.argtypes = [i64, P, P, P, i64, i64, P, P, d, i32, P, i64, P, P, P,
                                         P, P, P, P, P, C.c_char_p]
        L.orc_restarted_krylov.argtypes = [i64, P, P, P, P, i32, d, i64, d, i64, i64, d, i32, i64,
                                           i64, P, P, d, P, i32, P, P, P, i64, P, i64, C.c_char_p]
        for name, nargs in (("orc_gen_laplacian", [i32, i64]),
                            ("orc_gen_q1_hex", [i64, i32, u64, i32]),
                            ("orc_gen_convdiff_upwind", [i64, d, d, d, d])):
            fn = getattr(L, name)
            fn.restype = i32
            fn.argtypes = nargs + [P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(code, err):
    if code != 0:
        raise OracleError(code, err.value.decode())


def _csr(A):
    """Accept a scipy CSR matrix or a (row_ptr, col, val, n_cols) tuple."""
    if hasattr(A, "indptr"):
        rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.indices, dtype=np.int32)
        v = np.ascontiguousarray(A.data, dtype=np.float64)
        return rp, ci, v, A.shape[0], A.shape[1]
    rp, ci, v = A[0], A[1], A[2]
    n_cols = A[3] if len(A) > 3 else len(rp) - 1
    return (np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int32),
            np.ascontiguousarray(v, np.float64), len(rp) - 1, n_cols)


def splitmix_derive(seed: int, tag: int) -> int:
    return int(lib().orc_splitmix_derive(seed, tag))


def splitmix_stream(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    lib().orc_splitmix_stream(seed, count, _p(out))
    return out


def gaussian_vector(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().orc_gaussian_vector(seed, n, _p(out))
    return out


def _gen(fn, *args):
    n, nnz = C.c_int64(), C.c_int64()
    if fn(*args, C.byref(n), C.byref(nnz), None, None, None) != 0:
        raise OracleError(1, "generator: invalid parameters")
    rp = np.empty(n.value + 1, np.int64)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    fn(*args, C.byref(n), C.byref(nnz), _p(rp), _p(ci), _p(v))
    return rp, ci, v


# BASELINE problem generators restated independently of the product's
# (problems_oracle.cpp): the reference arm's inputs and the tests' second
# implementation of the same definitions.
def gen_laplacian(dim: int, N: int):
    return _gen(lib().orc_gen_laplacian, dim, N)


def gen_q1_hex(N: int, lognormal: bool = False, coef_seed: int = 1, dirichlet: bool = False):
    return _gen(lib().orc_gen_q1_hex, N, int(lognormal), C.c_uint64(coef_seed), int(dirichlet))


def gen_convdiff_upwind(N: int, peclet: float = 10.0, v=(1.0, 0.5, 0.25)):
    return _gen(lib().orc_gen_convdiff_upwind, N, float(peclet), float(v[0]), float(v[1]),
                float(v[2]))


@dataclass
class Sketch:
    d: int
    n: int
    zeta: int
    seed: int
    rows: np.ndarray  # int64 [n*zeta]
    signs: np.ndarray  # int8 [n*zeta]
    scale: float


def make_sketch(d: int, n: int, zeta: int, seed: int) -> Sketch:
    rows = np.empty(max(n * zeta, 0), np.int64)
    signs = np.empty(max(n * zeta, 0), np.int8)
    scale = np.zeros(1)
    err = C.create_string_buffer(512)
    _check(lib().orc_make_sketch(d, n, zeta, seed, _p(rows), _p(signs), _p(scale), err), err)
    return Sketch(d, n, zeta, seed, rows, signs, float(scale[0]))


def sketch_apply(S: Sketch, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(S.d)
    lib().orc_sketch_apply(S.d, S.n, S.zeta, _p(S.rows), _p(S.signs), S.scale, _p(x), _p(y))
    return y


def spmv(A, x, threads: int = 1) -> np.ndarray:
    rp, ci, v, nr, nc = _csr(A)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(nr)
    lib().orc_spmv(nr, nc, _p(rp), _p(ci), _p(v), _p(x), _p(y), threads)
    return y


def norm1(A) -> float:
    rp, ci, v, nr, nc = _csr(A)
    return float(lib().orc_norm1(nr, nc, _p(rp), _p(ci), _p(v)))


def validate(A) -> None:
    rp, ci, v, nr, nc = _csr(A)
    err = C.create_string_buffer(512)
    _check(lib().orc_validate(nr, nc, _p(rp), _p(ci), _p(v), err), err)


def funm(X: np.ndarray, kind: int, t: float) -> np.ndarray:
    n = X.shape[0]
    Xc = np.asfortranarray(X, np.float64)
    F = np.zeros((n, n), order="F")
    err = C.create_string_buffer(512)
    _check(lib().orc_funm(n, _p(Xc), kind, t, _p(F), err), err)
    return F


@dataclass
class Decomposition:
    W: np.ndarray
    U: np.ndarray | None
    Rbar: np.ndarray
    start_norm: float
    m: int
    breakdown_at: int | None
    counters: dict


def arnoldi_decomp(A, b, m: int, S: Sketch | None = None) -> Decomposition:
    rp, ci, v, n, _ = _csr(A)
    b = np.ascontiguousarray(b, np.float64)
    d = S.d if S else 1
    W = np.zeros((m + 1, n))  # rows of this array are columns of W
    U = np.zeros((m + 1, d))
    R = np.zeros((m, m + 1))
    sn = np.zeros(1)
    mk = np.zeros(1, np.int64)
    cols = np.zeros(1, np.int64)
    bd = np.zeros(1, np.int64)
    ctr = np.zeros(5, np.int64)
    err = C.create_string_buffer(512)
    code = lib().orc_arnoldi_decomp(
        n, _p(rp), _p(ci), _p(v), d, S.zeta if S else 1, _p(S.rows) if S else None,
        _p(S.signs) if S else None, S.scale if S else 1.0, 1 if S else 0, _p(b), m, _p(W),
        _p(U), _p(R), _p(sn), _p(mk), _p(cols), _p(bd), _p(ctr), err)
    _check(code, err)
    c, k = int(cols[0]), int(mk[0])
    Rbar = R.T[: (k + 1 if c == k + 1 else k), :k].copy()
    return Decomposition(W=W[:c].T.copy(), U=U[:c].T.copy() if S else None, Rbar=Rbar,
                         start_norm=float(sn[0]), m=k,
                         breakdown_at=int(bd[0]) or None,
                         counters=dict(zip(["matvecs", "dot_n", "dot_d", "basis_updates",
                                            "peak_basis_cols"], ctr.tolist())))


@dataclass
class RestartResult:
    f_hat: np.ndarray
    history: list
    converged: bool
    alpha: float
    cycles: int
    total_m: int
    counters: dict
    R_accum: np.ndarray | None = field(default=None)


def restarted_krylov(A, b, kind: int, t: float, m_r: int = 20, tol: float = 1e-10,
                     k_max: int = 100, budget_total_m: int = 4000,
                     divergence_factor: float = 1e6, S: Sketch | None = None,
                     reference: np.ndarray | None = None, threads: int = 1,
                     want_R: bool = False) -> RestartResult:
    rp, ci, v, n, _ = _csr(A)
    b = np.ascontiguousarray(b, np.float64)
    f = np.zeros(n)
    res = Result()
    cap = int(k_max) + 1
    recs = (CycleRecord * cap)()
    Rcap = min(budget_total_m, k_max * m_r) if want_R else 0
    Rbuf = np.zeros(Rcap * Rcap) if want_R else None
    ref = None if reference is None else np.ascontiguousarray(reference, np.float64)
    err = C.create_string_buffer(512)
    code = lib().orc_restarted_krylov(
        n, _p(rp), _p(ci), _p(v), _p(b), kind, t, m_r, tol, k_max, budget_total_m,
        divergence_factor, 1 if S else 0, S.d if S else 0, S.zeta if S else 0,
        _p(S.rows) if S else None, _p(S.signs) if S else None, S.scale if S else 1.0,
        _p(ref), threads, _p(f), C.byref(res), C.cast(recs, C.c_void_p), cap, _p(Rbuf), Rcap,
        err)
    _check(code, err)
    hist = []
    for i in range(res.n_records):
        r = recs[i]
        hist.append({k: getattr(r, k) for k, _ in CycleRecord._fields_})
    Racc = None
    if want_R:
        M = res.total_m
        Racc = Rbuf[: M * M].reshape(M, M).T.copy()
    return RestartResult(f_hat=f, history=hist, converged=bool(res.converged), alpha=res.alpha,
                         cycles=res.cycles, total_m=res.total_m,
                         counters=dict(matvecs=res.matvecs, dot_n=res.dot_n, dot_d=res.dot_d,
                                       basis_updates=res.basis_updates,
                                       peak_basis_cols=res.peak_basis_cols),
                         R_accum=Racc)
