"""ctypes front-end of oracle/_ref/librkmf_ref.so — TEST INFRASTRUCTURE ONLY.

``librkmf_ref.so`` is the REFERENCE'S OWN solver-path sources
(/root/reference/proj/src/{restart,basis,sketch,sparse,densefun,approximants,
leastsq}.cpp), compiled unmodified where they lie by ``make -C oracle ref``
against the Eigen-API stand-in ``oracle/eigen_standin/`` (Eigen is absent from
the image) plus the C-ABI layer ``oracle/ref_capi.cpp``. Its ``ref_*`` entry
points have the signatures of the oracle's ``orc_*``, so this module is the
oracle front-end (``oracle/oracle.py``) loaded a second time onto that
library: ``ref.restarted_krylov(...)`` etc. take and return the same objects.

Used only by tests/ (the restated oracle is checked against it) and by
tests/golden/make_ref_golden.py (which freezes its outputs as fixtures so the
pins also hold where the library is absent). The library is git-ignored and
travels to the GPU box with the snapshot; nothing reads /root/reference at
run time.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "librkmf_ref.so")
REFERENCE_ROOT = "/root/reference/proj"


def build() -> str | None:
    """Compile _ref/librkmf_ref.so if the reference sources are mounted."""
    if not os.path.isdir(os.path.join(REFERENCE_ROOT, "src")):
        return LIB_PATH if os.path.exists(LIB_PATH) else None
    subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return LIB_PATH


def available() -> bool:
    return os.path.exists(LIB_PATH)


class _Adapter:
    """Presents ref_* under the orc_* names, with the oracle's argtypes."""

    def __init__(self, ref_lib, orc_lib):
        self._ref = ref_lib
        self._orc = orc_lib

    def __getattr__(self, name):
        if not name.startswith("orc_"):
            raise AttributeError(name)
        fn = getattr(self._ref, "ref_" + name[4:])
        proto = getattr(self._orc, name)
        fn.argtypes = proto.argtypes
        fn.restype = proto.restype
        setattr(self, name, fn)
        return fn


_front = None
_raw = None


def raw():
    global _raw
    if _raw is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} is not built (make -C oracle ref)")
        L = C.CDLL(LIB_PATH)
        P, i64, u64, d = C.c_void_p, C.c_int64, C.c_uint64, C.c_double
        L.ref_splitmix_below.argtypes = [u64, u64, i64, P]
        L.ref_rand_fom.argtypes = [i64, P, P, P, i64, i64, P, P, d, P, i64, d, P, P, P, P,
                                   C.c_char_p]
        L.ref_load_mtx.argtypes = [C.c_char_p, P, P, P, P, P, P, C.c_char_p]
        L.ref_save_mtx.argtypes = [C.c_char_p, i64, i64, P, P, P, C.c_char_p]
        L.ref_load_vector.argtypes = [C.c_char_p, P, P, i64, C.c_char_p]
        L.ref_save_vector.argtypes = [C.c_char_p, P, i64, C.c_char_p]
        L.ref_convergence_sweep.argtypes = [i64, P, P, P, P, d, P, P, i64, C.c_int, P, i64, P,
                                            C.c_char_p]
        _raw = L
    return _raw


def front():
    """oracle.py bound to the reference library (same functions and types)."""
    global _front
    if _front is None:
        from oracle import oracle as O
        spec = importlib.util.spec_from_file_location("oracle._ref_front",
                                                      os.path.join(_HERE, "oracle.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[spec.name] = mod
        spec.loader.exec_module(mod)
        mod._lib = _Adapter(raw(), O.lib())
        _front = mod
    return _front


def __getattr__(name):  # ref.make_sketch, ref.restarted_krylov, ...
    return getattr(front(), name)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.kind = {1: "ParameterError", 2: "ShapeError", 3: "NumericalError",
                     4: "ParseError"}.get(code, "Error")


def _check(code, err):
    if code != 0:
        raise RefError(code, err.value.decode())


def splitmix_below(seed: int, bound: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    raw().ref_splitmix_below(seed, bound, count, _p(out))
    return out


def rand_fom(A, S, b, m: int, t: float):
    """(value, kappa_W, ritz) of the reference's rand_fom approximant."""
    O = front()
    rp, ci, v, n, _ = O._csr(A)
    b = np.ascontiguousarray(b, np.float64)
    value = np.zeros(n)
    kappa = np.zeros(1)
    rr, ri = np.zeros(m), np.zeros(m)
    err = C.create_string_buffer(512)
    _check(raw().ref_rand_fom(n, _p(rp), _p(ci), _p(v), S.d, S.zeta, _p(S.rows), _p(S.signs),
                              S.scale, _p(b), m, t, _p(value), _p(kappa), _p(rr), _p(ri), err),
           err)
    return value, float(kappa[0]), rr + 1j * ri


def load_mtx(path: str):
    nr, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    err = C.create_string_buffer(512)
    _check(raw().ref_load_mtx(path.encode(), C.byref(nr), C.byref(nc), C.byref(nnz), None, None,
                              None, err), err)
    rp = np.empty(nr.value + 1, np.int64)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    _check(raw().ref_load_mtx(path.encode(), C.byref(nr), C.byref(nc), C.byref(nnz), _p(rp),
                              _p(ci), _p(v), err), err)
    return rp, ci, v, nr.value, nc.value


def save_mtx(path: str, rp, ci, v, n_cols: int) -> None:
    rp = np.ascontiguousarray(rp, np.int64)
    ci = np.ascontiguousarray(ci, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    err = C.create_string_buffer(512)
    _check(raw().ref_save_mtx(path.encode(), len(rp) - 1, n_cols, _p(rp), _p(ci), _p(v), err),
           err)


def load_vector(path: str) -> np.ndarray:
    n = C.c_int64()
    err = C.create_string_buffer(512)
    _check(raw().ref_load_vector(path.encode(), C.byref(n), None, 0, err), err)
    out = np.empty(n.value)
    _check(raw().ref_load_vector(path.encode(), C.byref(n), _p(out), n.value, err), err)
    return out


def save_vector(path: str, x) -> None:
    x = np.ascontiguousarray(x, np.float64)
    err = C.create_string_buffer(512)
    _check(raw().ref_save_vector(path.encode(), _p(x), len(x), err), err)


class MethodSpecC(C.Structure):  # layout of rkmf_method_spec (include/rkmf_b200.h)
    _fields_ = [("name", C.c_char * 32), ("m", C.c_int64), ("d", C.c_int64), ("zeta", C.c_int64),
                ("tol", C.c_double), ("k_max", C.c_int64), ("seed", C.c_uint64)]


class SweepRecordC(C.Structure):  # layout of rkmf_sweep_record
    _fields_ = [("method", C.c_char * 32), ("n", C.c_int64), ("m_or_totalm", C.c_int64),
                ("cycle", C.c_int64), ("matvecs", C.c_int64), ("rel_error", C.c_double),
                ("update_norm", C.c_double), ("kappa_W", C.c_double),
                ("leftmost_ritz_re", C.c_double), ("elapsed_ms", C.c_double),
                ("note", C.c_char * 256), ("phase_build_ms", C.c_double),
                ("phase_eval_ms", C.c_double)]


def convergence_sweep(A, b, t: float, methods, reference=None, with_timing: bool = False):
    """restart::convergence_sweep (restart.cpp:124-305) on {A, b, ExpNeg(t)};
    methods: objects with name, m, d, zeta, tol, k_max, seed. Rows as dicts."""
    O = front()
    rp, ci, v, n, _ = O._csr(A)
    b = np.ascontiguousarray(b, np.float64)
    ref = None if reference is None else np.ascontiguousarray(reference, np.float64)
    ms = (MethodSpecC * max(len(methods), 1))()
    for i, m in enumerate(methods):
        ms[i] = MethodSpecC(m.name.encode()[:31], m.m, m.d, m.zeta, m.tol, m.k_max, m.seed)
    cap = 4096
    recs = (SweepRecordC * cap)()
    n_out = C.c_int64()
    err = C.create_string_buffer(512)
    _check(raw().ref_convergence_sweep(n, _p(rp), _p(ci), _p(v), _p(b), t, _p(ref),
                                       C.cast(ms, C.c_void_p), len(methods), int(with_timing),
                                       C.cast(recs, C.c_void_p), cap, C.byref(n_out), err), err)
    rows = []
    for i in range(min(n_out.value, cap)):
        r = recs[i]
        rows.append({k: (getattr(r, k).decode() if isinstance(getattr(r, k), bytes)
                         else getattr(r, k)) for k, _ in SweepRecordC._fields_})
    return rows


_strict = None
STRICT_LIB_PATH = os.path.join(_HERE, "liboracle_strict.so")


def strict():
    """oracle.py bound to liboracle_strict.so: the restated oracle compiled
    without FMA contraction (oracle/Makefile), the build that reproduces the
    reference's sources bit for bit."""
    global _strict
    if _strict is None:
        if not os.path.exists(STRICT_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE, "liboracle_strict.so"], check=True)
        spec = importlib.util.spec_from_file_location("oracle._strict_front",
                                                      os.path.join(_HERE, "oracle.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[spec.name] = mod
        spec.loader.exec_module(mod)
        mod._LIB_PATH = STRICT_LIB_PATH
        mod.lib()
        _strict = mod
    return _strict
