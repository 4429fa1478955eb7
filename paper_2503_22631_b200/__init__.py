"""rkmf_b200 — B200-native restarted randomized-Arnoldi f(A)b (arXiv 2503.22631).

Python mirror of the reference artifact's solver interface
(/root/reference/proj/include/rkmf/restart.hpp, sketch.hpp, basis.hpp,
densefun.hpp) over the C ABI in include/rkmf_b200.h. The compute path is the
hand-written sm_100a library ``_lib/librkmf_b200.so``; there is no CPU
fallback: if the library or a CUDA device is missing, calls raise.

Reference name map (reference -> here):
    restart::restarted_krylov        -> restarted_krylov
    restart::RestartOptions          -> RestartOptions
    restart::RestartResult           -> RestartResult
    restart::CycleRecord             -> CycleRecord
    sketch::make_sketch              -> make_sketch   (device-generated, bit-exact)
    sketch::sketch_apply(S, vec)     -> sketch_apply
    sparse::spmv                     -> spmv
    basis::randomized_arnoldi        -> randomized_arnoldi
    densefun::FunctionSpec::exp_neg  -> FunctionSpec.exp_neg
    (new) z^{-1/2}                   -> FunctionSpec.inv_sqrt
    rkmf::{Error, ShapeError, ParameterError, NumericalError} -> same names
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RKMF_LIB_PATH selects an alternative build (A/B experiments with build flags)
LIB_PATH = os.environ.get("RKMF_LIB_PATH") or os.path.join(_HERE, "_lib", "librkmf_b200.so")
CSRC = os.path.join(_HERE, "csrc")

RKMF_OK = 0
FN_EXP_NEG = 0
FN_INV_SQRT = 4
DENSE_AUTO, DENSE_FULL, DENSE_QUADRATURE = 0, 1, 2


# ---- error hierarchy: types.hpp:25-48 ----
class Error(RuntimeError):
    """rkmf::Error"""


class ShapeError(Error):
    """rkmf::ShapeError"""


class ParameterError(Error):
    """rkmf::ParameterError"""


class ParseError(Error):
    """rkmf::ParseError"""


class NumericalError(Error):
    """rkmf::NumericalError"""


class DeviceError(Error):
    """CUDA / NCCL failure inside the device library."""


_CODE = {1: ParameterError, 2: ShapeError, 3: NumericalError, 4: DeviceError, 5: Error,
         6: ParseError}


class RestartOptionsC(C.Structure):
    _fields_ = [("m_r", C.c_int64), ("tol", C.c_double), ("k_max", C.c_int64),
                ("budget_total_m", C.c_int64), ("divergence_factor", C.c_double),
                ("dense_f", C.c_int32), ("quad_nodes", C.c_int32), ("diagnostics", C.c_int32),
                ("reserved", C.c_int32)]


class CycleRecordC(C.Structure):
    _fields_ = [("cycle", C.c_int64), ("total_m", C.c_int64), ("total_matvecs", C.c_int64),
                ("update_norm", C.c_double), ("error_vs_reference", C.c_double),
                ("kappa_W", C.c_double), ("leftmost_ritz_re", C.c_double),
                ("alpha_dev", C.c_double), ("elapsed_ms", C.c_double), ("build_ms", C.c_double),
                ("funm_ms", C.c_double), ("start_norm", C.c_double), ("subdiag", C.c_double)]


class RestartResultC(C.Structure):
    _fields_ = [("converged", C.c_int64), ("cycles", C.c_int64), ("total_m", C.c_int64),
                ("alpha", C.c_double), ("matvecs", C.c_int64), ("dot_n", C.c_int64),
                ("dot_d", C.c_int64), ("basis_updates", C.c_int64),
                ("peak_basis_cols", C.c_int64), ("n_records", C.c_int64),
                ("solve_ms", C.c_double), ("quad_nodes", C.c_int64)]


class CycleInfoC(C.Structure):
    _fields_ = [("cycle", C.c_int64), ("n", C.c_int64), ("m_k", C.c_int64),
                ("w_cols", C.c_int64), ("W", C.POINTER(C.c_double)), ("total_m", C.c_int64),
                ("R_accum", C.POINTER(C.c_double)), ("update", C.POINTER(C.c_double)),
                ("f_hat", C.POINTER(C.c_double)), ("alpha", C.c_double)]


_OBSERVER_CB = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(CycleInfoC))


class MethodSpecC(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("m", C.c_int64), ("d", C.c_int64), ("zeta", C.c_int64),
                ("tol", C.c_double), ("k_max", C.c_int64), ("seed", C.c_uint64)]


class SweepRecordC(C.Structure):
    _fields_ = [("method", C.c_char * 32), ("n", C.c_int64), ("m_or_totalm", C.c_int64),
                ("cycle", C.c_int64), ("matvecs", C.c_int64), ("rel_error", C.c_double),
                ("update_norm", C.c_double), ("kappa_W", C.c_double),
                ("leftmost_ritz_re", C.c_double), ("elapsed_ms", C.c_double),
                ("note", C.c_char * 256), ("phase_build_ms", C.c_double),
                ("phase_eval_ms", C.c_double)]

# Every symbol declared in include/rkmf_b200.h: (name, restype, argtypes)
_P, _I64, _U64, _D, _I32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int32
_PP = C.POINTER(C.c_void_p)
SYMBOLS = [
    ("rkmf_context_create", C.c_int, [C.c_int, _PP]),
    ("rkmf_context_destroy", C.c_int, [_P]),
    ("rkmf_last_error", C.c_char_p, [_P]),
    ("rkmf_context_set_stream", C.c_int, [_P, _P]),
    ("rkmf_restart_options_default", None, [_P]),
    ("rkmf_context_launch_count", C.c_int64, [_P]),
    ("rkmf_context_kernel_timing", C.c_int, [_P, C.c_int]),
    ("rkmf_context_kernel_times", C.c_int, [_P, _P, _P, C.c_int]),
    ("rkmf_context_set_fused_cycle", C.c_int, [_P, C.c_int]),
    ("rkmf_matrix_create_host", C.c_int, [_P, _I64, _I64, _P, _P, _P, _PP]),
    ("rkmf_matrix_create_device", C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _PP]),
    ("rkmf_matrix_destroy", C.c_int, [_P]),
    ("rkmf_matrix_info", C.c_int, [_P, _P, _P, _P, _P]),
    ("rkmf_matrix_dia", C.c_int, [_P, C.c_int, _P]),
    ("rkmf_matrix_dia_dict", C.c_int, [_P, C.c_int, _P]),
    ("rkmf_sketch_create", C.c_int, [_P, _I64, _I64, _I64, _U64, _PP]),
    ("rkmf_sketch_destroy", C.c_int, [_P]),
    ("rkmf_sketch_set_scale", C.c_int, [_P, _D]),
    ("rkmf_sketch_layout_info", C.c_int, [_P, _P, _P]),
    ("rkmf_sketch_export", C.c_int, [_P, _P, _P, _P, _P]),
    ("rkmf_spmv", C.c_int, [_P, _P, _P, _P]),
    ("rkmf_sketch_apply", C.c_int, [_P, _P, _P, _P]),
    ("rkmf_spmv_sketch", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("rkmf_kernel_bench", C.c_int, [_P, _P, _P, _I32, _P, _P, _P, _I32, _P]),
    ("rkmf_randomized_arnoldi", C.c_int,
     [_P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P]),
    ("rkmf_restarted_krylov", C.c_int,
     [_P, _P, _P, _P, C.c_int, _I32, _D, _P, _P, C.c_int, _P, _P, _P, _I64]),
    ("rkmf_last_r_accum", C.c_int, [_P, _P, _I64, _P]),
    ("rkmf_context_set_observer", C.c_int, [_P, _OBSERVER_CB, _P]),
    ("rkmf_nccl_unique_id", C.c_int, [_P]),
    ("rkmf_context_init_comm", C.c_int, [_P, _I32, _I32, _P]),
    ("rkmf_context_init_host_comm", C.c_int, [_P, _I32, _I32, _P]),
    ("rkmf_matrix_create_partitioned", C.c_int, [_P, _I64, _P, _P, _P, _P, _PP]),
    ("rkmf_sketch_create_partitioned", C.c_int, [_P, _I64, _I64, _I64, _U64, _I64, _I64, _PP]),
    ("rkmf_partition_rows", C.c_int, [_I64, _P, _I32, _P]),
    ("rkmf_partition_halo", C.c_int, [_I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    ("rkmf_gen_laplacian", C.c_int, [_I32, _I64, _P, _P, _P, _P, _P]),
    ("rkmf_gen_q1_hex", C.c_int, [_I64, _I32, _U64, _I32, _P, _P, _P, _P, _P]),
    ("rkmf_gen_convdiff_upwind", C.c_int, [_I64, _D, _D, _D, _D, _P, _P, _P, _P, _P]),
    ("rkmf_gen_gaussian", C.c_int, [_U64, _I64, _P]),
    ("rkmf_gen_gaussian_range", C.c_int, [_U64, _I64, _I64, _P]),
    ("rkmf_matrix_gen_q1_hex", C.c_int, [_P, _I64, _I32, _U64, _I32, _PP]),
    ("rkmf_matrix_gen_laplacian", C.c_int, [_P, _I32, _I64, _PP]),
    ("rkmf_gen_gaussian_device", C.c_int, [_P, _U64, _I64, _I64, _P]),
    ("rkmf_matrix_export", C.c_int, [_P, _P, _P, _P, _P]),
    ("rkmf_matrix_rp64", C.c_int, [_P, C.c_int, _P]),
    ("rkmf_matrix_gen_convdiff", C.c_int, [_P, _I64, _D, _D, _D, _D, _PP]),
    ("rkmf_matrix_gen_q1_hex_partitioned", C.c_int, [_P, _I64, _I32, _U64, _I32, _P, _PP]),
    ("rkmf_context_comm_info", C.c_int, [_P, _P, _P, _P]),
    ("rkmf_mtx_load", C.c_int, [C.c_char_p, _P, _P, _P, _P, _P, _P, C.c_char_p, _I64]),
    ("rkmf_mtx_save", C.c_int, [C.c_char_p, _I64, _I64, _P, _P, _P, C.c_char_p, _I64]),
    ("rkmf_vector_load", C.c_int, [C.c_char_p, _P, _P, C.c_char_p, _I64]),
    ("rkmf_vector_save", C.c_int, [C.c_char_p, _I64, _P, C.c_char_p, _I64]),
    ("rkmf_host_free", None, [_P]),
    ("rkmf_matrix_load_mtx", C.c_int, [_P, C.c_char_p, _PP]),
    ("rkmf_matrix_save_mtx", C.c_int, [_P, _P, C.c_char_p]),
    ("rkmf_convergence_sweep", C.c_int,
     [_P, _P, _P, _I32, _D, _P, _P, _I64, _I32, _P, _I64, _P]),
    ("rkmf_sweep_write_csv", C.c_int, [_P, _I64, C.c_char_p, C.c_char_p, _I64]),
]

_lib = None


def build(force: bool = False) -> str:
    """Compile the sm_100a library in-tree (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(["make", "-s", "-j", jobs, "-C", CSRC], check=True)
    return LIB_PATH


def lib():
    """Load the device library; raises if it is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"rkmf_b200 CUDA library not built: {LIB_PATH} "
                              "(run paper_2503_22631_b200.build() or __graft_entry__.build())")
        try:  # torch first: the library's libnccl.so.2 then binds to torch's
            import torch  # noqa: F401  (newer) NCCL instead of the system one
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            if os.environ.get("RKMF_LIB_PATH") and not hasattr(L, name):
                continue  # an older build under A/B comparison (tools/)
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


def _is_torch(a) -> bool:
    return hasattr(a, "data_ptr") and hasattr(a, "is_cuda")


class Context:
    """One device + stream (rkmf_context). Solves on one context are serialised."""

    _default = {}

    def __init__(self, device: int = 0):
        self.device = device
        self.solves = 0  # solves run on this context (RestartResult.R_accum guard)
        h = C.c_void_p()
        code = lib().rkmf_context_create(device, C.byref(h))
        if code != RKMF_OK:
            raise _CODE.get(code, Error)(f"rkmf_context_create failed (code {code}): "
                                         "no CUDA device? (there is no CPU fallback)")
        self.h = h

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def check(self, code: int):
        if code != RKMF_OK:
            msg = lib().rkmf_last_error(self.h).decode()
            raise _CODE.get(code, Error)(msg)

    def set_stream(self, stream) -> None:
        """Launch on a torch.cuda.Stream / raw cudaStream_t (None = own stream)."""
        raw = None if stream is None else getattr(stream, "cuda_stream", stream)
        self.check(lib().rkmf_context_set_stream(self.h, raw))

    def comm_info(self) -> dict:
        """The communicator as the library sees it (NCCL: ncclCommCount)."""
        n, r, t = C.c_int32(), C.c_int32(), C.c_int32()
        self.check(lib().rkmf_context_comm_info(self.h, C.byref(n), C.byref(r), C.byref(t)))
        return {"nranks": n.value, "rank": r.value,
                "transport": {0: "none", 1: "nccl", 2: "host"}.get(t.value, "?")}

    @property
    def launch_count(self) -> int:
        return int(lib().rkmf_context_launch_count(self.h))

    KERNEL_CLASSES = ("spmv_sketch", "rgs_step", "basis_update", "dense_f", "final_update",
                      "start_sketch_init", "fused_cycle")

    def set_fused_cycle(self, enable: bool) -> None:
        """Small matrices: each cycle's steps as one cooperative kernel (default on)."""
        self.check(lib().rkmf_context_set_fused_cycle(self.h, int(enable)))

    def kernel_timing(self, enable: bool) -> None:
        """Events around every solve launch (diagnostic runs only)."""
        self.check(lib().rkmf_context_kernel_timing(self.h, int(enable)))

    def kernel_times(self, reset: bool = True) -> dict:
        ms = np.zeros(len(self.KERNEL_CLASSES))
        cnt = np.zeros(len(self.KERNEL_CLASSES), np.int64)
        self.check(lib().rkmf_context_kernel_times(self.h, _ptr(ms), _ptr(cnt), int(reset)))
        return {c: (float(ms[i]), int(cnt[i])) for i, c in enumerate(self.KERNEL_CLASSES)}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().rkmf_context_destroy(self.h)
        except Exception:
            pass


class SparseMatrix:
    """Device CSR (sparse.hpp:16-24): int32 columns, fp64 values."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle
        nr, nc, nz, n1 = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        lib().rkmf_matrix_info(handle, C.byref(nr), C.byref(nc), C.byref(nz), C.byref(n1))
        self.n_rows, self.n_cols, self.nnz, self.norm1 = nr.value, nc.value, nz.value, n1.value

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def set_diagonal_copy(self, enable: bool) -> int:
        """Drop (False) or build (True, if the matrix qualifies) the diagonal
        copy the fused SpMV + sketch streams instead of the CSR arrays;
        returns the diagonal count (0 = CSR only). Results are identical."""
        nd = C.c_int()
        self.ctx.check(lib().rkmf_matrix_dia(self.h, int(bool(enable)), C.byref(nd)))
        return nd.value

    def set_row_dictionary(self, enable: bool) -> int:
        """Drop (False) or build (True, if the rows take at most 256 distinct
        forms: the diagonal copy's value tuples, or without a copy the CSR rows
        up to translation) the row dictionary the fused SpMV + sketch then
        streams (one byte per row); returns the form count (0 = none). z is
        identical."""
        nt = C.c_int()
        self.ctx.check(lib().rkmf_matrix_dia_dict(self.h, int(bool(enable)), C.byref(nt)))
        return nt.value

    @property
    def ntuples(self) -> int:
        """Distinct row forms of the row dictionary K2 streams (0 = none): the
        diagonal copy's value tuples, or, without a copy, the CSR rows up to
        translation (rowdict.cu)."""
        nt = C.c_int()
        self.ctx.check(lib().rkmf_matrix_dia_dict(self.h, 2, C.byref(nt)))
        return nt.value

    def use_rp64(self) -> bool:
        """Widen the device row pointers to int64 (the storage cfg5's 3.6e9
        nonzeros need) so the int64 kernel instantiations run; returns the width."""
        w = C.c_int()
        self.ctx.check(lib().rkmf_matrix_rp64(self.h, 1, C.byref(w)))
        return bool(w.value)

    @property
    def rp64(self) -> bool:
        w = C.c_int()
        self.ctx.check(lib().rkmf_matrix_rp64(self.h, 0, C.byref(w)))
        return bool(w.value)

    @property
    def ndiag(self) -> int:
        """Diagonals of the stored diagonal copy (0 = CSR only)."""
        nd = C.c_int()
        self.ctx.check(lib().rkmf_matrix_dia(self.h, 2, C.byref(nd)))
        return nd.value

    @classmethod
    def from_csr(cls, row_ptr, col_idx, values, n_cols: Optional[int] = None,
                 ctx: Optional[Context] = None) -> "SparseMatrix":
        ctx = ctx or Context.default()
        if _is_torch(row_ptr) and row_ptr.is_cuda:
            import torch
            rp = row_ptr.to(torch.int64).contiguous()
            ci = col_idx.to(torch.int32).contiguous()
            v = values.to(torch.float64).contiguous()
            n = rp.numel() - 1
            h = C.c_void_p()
            ctx.check(lib().rkmf_matrix_create_device(ctx.h, n, n if n_cols is None else n_cols,
                                                      v.numel(), rp.data_ptr(), ci.data_ptr(),
                                                      v.data_ptr(), C.byref(h)))
            return cls(ctx, h)
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col_idx, np.int32)
        v = np.ascontiguousarray(values, np.float64)
        n = len(rp) - 1
        h = C.c_void_p()
        ctx.check(lib().rkmf_matrix_create_host(ctx.h, n, n if n_cols is None else n_cols,
                                                _ptr(rp), _ptr(ci), _ptr(v), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def q1_hex(cls, N: int, lognormal: bool = False, coef_seed: int = 1, dirichlet: bool = False,
               ctx: Optional[Context] = None) -> "SparseMatrix":
        """Q1 hexahedral stiffness on N^3 nodes, generated in HBM (cfg3, cfg5)."""
        ctx = ctx or Context.default()
        h = C.c_void_p()
        ctx.check(lib().rkmf_matrix_gen_q1_hex(ctx.h, N, int(lognormal), C.c_uint64(coef_seed),
                                               int(dirichlet), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def laplacian(cls, dim: int, N: int, ctx: Optional[Context] = None) -> "SparseMatrix":
        """5/7-point Dirichlet Laplacian (h^-2 scaled), generated in HBM (cfg1, cfg2)."""
        ctx = ctx or Context.default()
        h = C.c_void_p()
        ctx.check(lib().rkmf_matrix_gen_laplacian(ctx.h, dim, N, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def convdiff(cls, N: int, peclet: float = 10.0, v=(1.0, 0.5, 0.25),
                 ctx: Optional[Context] = None) -> "SparseMatrix":
        """3D upwind convection-diffusion (cfg4), generated in HBM."""
        ctx = ctx or Context.default()
        h = C.c_void_p()
        ctx.check(lib().rkmf_matrix_gen_convdiff(ctx.h, N, float(peclet), float(v[0]), float(v[1]),
                                                 float(v[2]), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def q1_hex_partitioned(cls, ctx: Context, N: int, row_starts, lognormal: bool = False,
                           coef_seed: int = 1, dirichlet: bool = False) -> "SparseMatrix":
        """This rank's whole x-planes of the Q1 matrix (cfg5 partitioned), in HBM."""
        rs = np.ascontiguousarray(row_starts, np.int64)
        h = C.c_void_p()
        ctx.check(lib().rkmf_matrix_gen_q1_hex_partitioned(ctx.h, N, int(lognormal),
                                                           C.c_uint64(coef_seed), int(dirichlet),
                                                           _ptr(rs), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_mtx(cls, path: str, ctx: Optional[Context] = None) -> "SparseMatrix":
        """sparse::load_matrix_market (sparse.cpp:140-192) into HBM."""
        ctx = ctx or Context.default()
        h = C.c_void_p()
        ctx.check(lib().rkmf_matrix_load_mtx(ctx.h, os.fsencode(path), C.byref(h)))
        return cls(ctx, h)

    def export(self):
        """(row_ptr int64, col_idx int32, values float64) host copies of the
        device CSR (local numbering when partitioned)."""
        rp = np.empty(self.n_rows + 1, np.int64)
        ci = np.empty(self.nnz, np.int32)
        v = np.empty(self.nnz, np.float64)
        self.ctx.check(lib().rkmf_matrix_export(self.ctx.h, self.h, _ptr(rp), _ptr(ci), _ptr(v)))
        return rp, ci, v

    def save_mtx(self, path: str) -> None:
        """sparse::save_matrix_market (sparse.cpp:194-211) of the device matrix."""
        self.ctx.check(lib().rkmf_matrix_save_mtx(self.ctx.h, self.h, os.fsencode(path)))

    @classmethod
    def from_scipy(cls, A, ctx: Optional[Context] = None) -> "SparseMatrix":
        A = A.tocsr()
        A.sort_indices()
        return cls.from_csr(A.indptr, A.indices, A.data, A.shape[1], ctx)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().rkmf_matrix_destroy(self.h)
        except Exception:
            pass


class SketchOperator:
    """Device sparse-sign embedding S in R^{d x n} (sketch.hpp:16-24)."""

    def __init__(self, ctx: Context, handle, d, n, zeta, seed):
        self.ctx, self.h, self.d, self.n, self.zeta, self.seed = ctx, handle, d, n, zeta, seed
        self._scale = 1.0 / math.sqrt(zeta)

    def layout_bytes_per_tile(self):
        """(header, entry) bytes per 128-column tile of the layout K2 streams."""
        h, e = C.c_int64(), C.c_int64()
        lib().rkmf_sketch_layout_info(self.h, C.byref(h), C.byref(e))
        return h.value, e.value

    @property
    def scale(self) -> float:
        return self._scale

    @scale.setter
    def scale(self, value: float) -> None:
        lib().rkmf_sketch_set_scale(self.h, float(value))
        self._scale = float(value)

    def export(self):
        """(rows int64[n*zeta], signs int8[n*zeta], scale) on the host."""
        rows = np.empty(self.n * self.zeta, np.int64)
        signs = np.empty(self.n * self.zeta, np.int8)
        sc = C.c_double()
        self.ctx.check(lib().rkmf_sketch_export(self.ctx.h, self.h, _ptr(rows), _ptr(signs),
                                                C.byref(sc)))
        return rows, signs, sc.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().rkmf_sketch_destroy(self.h)
        except Exception:
            pass


def make_sketch(d: int, n: int, zeta: int, seed: int, ctx: Optional[Context] = None) -> SketchOperator:
    """sketch::make_sketch (sketch.cpp:13-49), generated on the device."""
    ctx = ctx or Context.default()
    h = C.c_void_p()
    ctx.check(lib().rkmf_sketch_create(ctx.h, d, n, zeta, C.c_uint64(seed), C.byref(h)))
    return SketchOperator(ctx, h, d, n, zeta, seed)


def _dev(x, ctx: Context):
    import torch
    if _is_torch(x) and x.is_cuda:
        return x.to(torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, np.float64)).to(f"cuda:{ctx.device}")


def spmv(A: SparseMatrix, x):
    """z = A x (sparse.cpp:83-95); returns a CUDA tensor."""
    import torch
    xd = _dev(x, A.ctx)
    if xd.numel() != A.n_cols:
        raise ShapeError("shape: spmv expects len(x) == n_cols")
    y = torch.empty(A.n_rows, dtype=torch.float64, device=xd.device)
    A.ctx.check(lib().rkmf_spmv(A.ctx.h, A.h, xd.data_ptr(), y.data_ptr()))
    return y


def sketch_apply(S: SketchOperator, x):
    """y = S x (sketch.cpp:51-63); returns a CUDA tensor."""
    import torch
    xd = _dev(x, S.ctx)
    if xd.numel() != S.n:
        raise ShapeError("shape: sketch_apply expects len(x) == n")
    y = torch.empty(S.d, dtype=torch.float64, device=xd.device)
    S.ctx.check(lib().rkmf_sketch_apply(S.ctx.h, S.h, xd.data_ptr(), y.data_ptr()))
    return y


def spmv_sketch(A: SparseMatrix, S: SketchOperator, x):
    """(A x, S A x) from the fused kernel."""
    import torch
    xd = _dev(x, A.ctx)
    z = torch.empty(A.n_rows, dtype=torch.float64, device=xd.device)
    p = torch.empty(S.d, dtype=torch.float64, device=xd.device)
    A.ctx.check(lib().rkmf_spmv_sketch(A.ctx.h, A.h, S.h, xd.data_ptr(), z.data_ptr(),
                                       p.data_ptr()))
    return z, p


def kernel_bench(A: SparseMatrix, S: Optional[SketchOperator], x, mode: int = 1,
                 reps: int = 50) -> float:
    """Average device ms of one step-kernel launch (measurement only): mode 1 =
    fused SpMV+sketch (K2), 0 = SpMV alone, 2 = sketch of x alone."""
    import torch
    xd = _dev(x, A.ctx)
    z = torch.empty(A.n_rows, dtype=torch.float64, device=xd.device)
    p = torch.empty(S.d if S is not None else 1, dtype=torch.float64, device=xd.device)
    ms = C.c_double()
    A.ctx.check(lib().rkmf_kernel_bench(A.ctx.h, A.h, S.h if S is not None else None, mode,
                                        xd.data_ptr(), z.data_ptr(), p.data_ptr(), reps,
                                        C.byref(ms)))
    return ms.value


@dataclass
class KrylovDecomposition:
    """basis::KrylovDecomposition (basis.hpp:22-41), sketched-orthonormal kind."""
    W: object  # CUDA tensor n x cols
    U: object  # CUDA tensor d x cols
    Rbar: np.ndarray
    start_norm: float
    breakdown_at: Optional[int]
    counters: dict

    def m(self) -> int:
        return self.Rbar.shape[1]

    def Rm(self) -> np.ndarray:
        return self.Rbar[: self.m(), :]

    def subdiag(self) -> float:
        return float(self.Rbar[self.m(), self.m() - 1]) if self.Rbar.shape[0] > self.m() else 0.0


def randomized_arnoldi(A: SparseMatrix, S: SketchOperator, b, m: int) -> KrylovDecomposition:
    """basis::randomized_arnoldi (basis.cpp:92-142) on the device."""
    import torch
    bd = _dev(b, A.ctx)
    n = A.n_rows
    if bd.numel() != n:
        raise ShapeError("arnoldi: start vector length mismatch")
    W = torch.zeros((m + 1, n), dtype=torch.float64, device=bd.device)  # column-major n x (m+1)
    U = torch.zeros((m + 1, S.d), dtype=torch.float64, device=bd.device)
    R = np.zeros((m, m + 1))  # column-major (m+1) x m
    sn, mk, bk = C.c_double(), C.c_int64(), C.c_int64()
    ctr = np.zeros(5, np.int64)
    A.ctx.solves += 1
    A.ctx.check(lib().rkmf_randomized_arnoldi(A.ctx.h, A.h, S.h, bd.data_ptr(), m, W.data_ptr(),
                                              n, U.data_ptr(), _ptr(R), C.byref(sn), C.byref(mk),
                                              C.byref(bk), _ptr(ctr)))
    k = mk.value
    cols = k + 1 if bk.value == 0 else k
    Rbar = R.T[: (k + 1 if bk.value == 0 else k), :k].copy()
    return KrylovDecomposition(W=W[:cols].T, U=U[:cols].T, Rbar=Rbar, start_norm=sn.value,
                               breakdown_at=bk.value or None,
                               counters=dict(zip(["matvecs", "dot_n", "dot_d", "basis_updates",
                                                  "peak_basis_cols"], ctr.tolist())))


@dataclass
class FunctionSpec:
    """densefun::FunctionSpec (densefun.hpp:19-32): ExpNeg(t) and the new InvSqrt."""
    kind: int = FN_EXP_NEG
    t: float = 1.0

    @staticmethod
    def exp_neg(t: float) -> "FunctionSpec":
        if not (t >= 0.0):
            raise ParameterError("FunctionSpec: t must be >= 0")
        return FunctionSpec(FN_EXP_NEG, float(t))

    @staticmethod
    def inv_sqrt() -> "FunctionSpec":
        return FunctionSpec(FN_INV_SQRT, 1.0)


@dataclass
class RestartOptions:
    """restart::RestartOptions (restart.hpp:20-26) + device dense-f choice."""
    m_r: int = 20
    tol: float = 1e-10
    k_max: int = 100
    budget_total_m: int = 4000
    divergence_factor: float = 1e6
    dense_f: str = "auto"  # auto | full | quadrature
    quad_nodes: int = 0
    diagnostics: bool = False  # per-cycle kappa_W / leftmost Ritz (restart.cpp:101,103)

    def to_c(self) -> RestartOptionsC:
        mode = {"auto": DENSE_AUTO, "full": DENSE_FULL, "quadrature": DENSE_QUADRATURE}[self.dense_f]
        return RestartOptionsC(int(self.m_r), float(self.tol), int(self.k_max),
                               int(self.budget_total_m), float(self.divergence_factor), mode,
                               int(self.quad_nodes), int(bool(self.diagnostics)), 0)


@dataclass
class CycleRecord:
    """restart::CycleRecord (restart.hpp:28-40); times are device times."""
    cycle: int
    total_m: int
    total_matvecs: int
    update_norm: float
    error_vs_reference: Optional[float]
    kappa_W: float
    leftmost_ritz_re: float
    alpha_dev: float
    elapsed_ms: float
    build_ms: float
    funm_ms: float
    start_norm: float
    subdiag: float


@dataclass
class CycleInfo:
    """restart::CycleInfo (restart.hpp:42-54), host copies made for the
    observer: W is the cycle's basis block as built (n x w_cols, column 0 =
    start / alpha_k, one extra column when a next vector exists), R_accum the
    accumulated compression (None when not kept), update = y_k, f_hat the
    running approximation, alpha the global scale from cycle 1."""
    cycle: int
    W: np.ndarray
    m_k: int
    R_accum: Optional[np.ndarray]
    update: np.ndarray
    f_hat: np.ndarray
    alpha: float


def _observer_callback(fn):
    def cb(_user, pinfo):
        i = pinfo.contents
        n, wc, M = int(i.n), int(i.w_cols), int(i.total_m)
        W = np.ctypeslib.as_array(i.W, shape=(wc, n)).T.copy() if wc * n else np.zeros((n, wc))
        R = (np.ctypeslib.as_array(i.R_accum, shape=(M, M)).T.copy()
             if bool(i.R_accum) and M else None)
        y = np.ctypeslib.as_array(i.update, shape=(n,)).copy()
        f = np.ctypeslib.as_array(i.f_hat, shape=(n,)).copy()
        try:
            fn(CycleInfo(cycle=int(i.cycle), W=W, m_k=int(i.m_k), R_accum=R, update=y, f_hat=f,
                         alpha=float(i.alpha)))
        except Exception:  # noqa: BLE001 - an observer must not unwind through C
            import traceback
            traceback.print_exc()
    return _OBSERVER_CB(cb)


@dataclass
class RestartResult:
    """restart::RestartResult (restart.hpp:56-65)."""
    f_hat: object
    history: List[CycleRecord]
    converged: bool
    alpha: float
    cycles: int
    total_m: int
    counters: dict
    solve_ms: float
    quad_nodes: int = 0  # restart-quadrature nodes of the last cycle (0: FULL)
    _ctx: Context = field(repr=False, default=None)
    _R: Optional[np.ndarray] = field(repr=False, default=None)
    _solve_id: int = field(repr=False, default=-1)

    @property
    def R_accum(self) -> np.ndarray:
        """The accumulated compression (restart.cpp:61-70), read from the
        context's device buffer on first access. That buffer belongs to the
        context's latest solve: after another solve on the same context the
        property raises instead of returning the newer solve's matrix (pass
        keep_R_accum=True to restarted_krylov to copy it out eagerly)."""
        if self._R is None:
            if self._ctx is None or self._ctx.solves != self._solve_id:
                raise Error("R_accum: the context has run another solve since this result; "
                            "use restarted_krylov(..., keep_R_accum=True)")
            M = self.total_m
            R = np.zeros((M, M), order="F")
            tm = C.c_int64()
            self._ctx.check(lib().rkmf_last_r_accum(self._ctx.h, _ptr(R), M, C.byref(tm)))
            self._R = R if tm.value == M else None
        return self._R


def restarted_krylov(A: SparseMatrix, b, f: FunctionSpec, opts: RestartOptions = None,
                     S: SketchOperator = None, reference=None, out=None,
                     keep_R_accum: bool = False, observer=None) -> RestartResult:
    """restart::restarted_krylov (restart.hpp:74-79): the randomized builder with a
    SketchOperator S, the classical builder (CGS2 on device) with S = None.
    observer(CycleInfo) is the reference's test-only CycleObserver (device->host
    copies every cycle; not for timed runs).

    b may be a numpy array (host: the host<->device copies are part of the call)
    or a CUDA tensor (device-resident); f_hat comes back in the same residency
    (into `out` when given: a float64 array/tensor of length n).
    """
    opts = opts or RestartOptions()
    ctx = A.ctx
    # S is None selects the classical builder (restart.cpp:53-55, basis.cpp:34-77)
    on_dev = _is_torch(b) and b.is_cuda
    n = A.n_rows
    if on_dev:
        import torch
        bb = b.to(torch.float64).contiguous()
        fout = out if out is not None else torch.empty(n, dtype=torch.float64, device=bb.device)
        ref = None if reference is None else _dev(reference, ctx)
        bptr, fptr = bb.data_ptr(), fout.data_ptr()
    else:
        bb = np.ascontiguousarray(b, np.float64)
        fout = out if out is not None else np.zeros(n)
        if fout.dtype != np.float64 or not fout.flags["C_CONTIGUOUS"] or fout.size != n:
            raise ShapeError("restarted_krylov: out must be a contiguous float64 array of length n")
        ref = None if reference is None else np.ascontiguousarray(reference, np.float64)
        bptr, fptr = _ptr(bb), _ptr(fout)
    if len(bb) != n:
        raise ShapeError("arnoldi: start vector length mismatch")
    res = RestartResultC()
    cap = int(opts.k_max) + 1
    recs = (CycleRecordC * cap)()
    oc = opts.to_c()
    ctx.solves += 1
    cb = None
    if observer is not None:  # test-only CycleObserver (restart.hpp:53)
        cb = _observer_callback(observer)
        ctx.check(lib().rkmf_context_set_observer(ctx.h, cb, None))
    try:
        ctx.check(lib().rkmf_restarted_krylov(ctx.h, A.h, S.h if S is not None else None, bptr,
                                              1 if on_dev else 0, f.kind, f.t, C.byref(oc), fptr,
                                              1 if on_dev else 0, _ptr(ref), C.byref(res),
                                              C.cast(recs, C.c_void_p), cap))
    finally:
        if cb is not None:
            lib().rkmf_context_set_observer(ctx.h, _OBSERVER_CB(), None)
    hist = []
    for i in range(res.n_records):
        r = recs[i]
        d = {k: getattr(r, k) for k, _ in CycleRecordC._fields_}
        if math.isnan(d["error_vs_reference"]):
            d["error_vs_reference"] = None
        hist.append(CycleRecord(**d))
    out_res = RestartResult(f_hat=fout, history=hist, converged=bool(res.converged), alpha=res.alpha,
                         cycles=res.cycles, total_m=res.total_m,
                         counters=dict(matvecs=res.matvecs, dot_n=res.dot_n, dot_d=res.dot_d,
                                       basis_updates=res.basis_updates,
                                       peak_basis_cols=res.peak_basis_cols),
                         solve_ms=res.solve_ms, quad_nodes=res.quad_nodes, _ctx=ctx,
                         _solve_id=ctx.solves)
    if keep_R_accum:
        _ = out_res.R_accum
    return out_res


# ---- multi-GPU: row-block partition ----
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    if lib().rkmf_nccl_unique_id(buf) != RKMF_OK:
        raise DeviceError("ncclGetUniqueId failed")
    return buf.raw


def init_comm(ctx: Context, nranks: int, rank: int, unique_id: bytes) -> None:
    """One NCCL communicator per context (one process per GPU)."""
    buf = C.create_string_buffer(unique_id, 128)
    ctx.check(lib().rkmf_context_init_comm(ctx.h, nranks, rank, buf))
    ctx.nranks, ctx.rank = nranks, rank


_REDUCE_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
_A2A_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                      C.POINTER(C.c_int64))


class _HostComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum_f64", _REDUCE_CB),
                ("allreduce_max_f64", _REDUCE_CB), ("alltoallv_b64", _A2A_CB)]


def init_host_comm(ctx: Context, nranks: int, rank: int, allreduce, alltoallv) -> None:
    """Drive the partitioned solve through host callbacks (rkmf_host_comm).

    allreduce(buf: np.ndarray[float64], op: "sum" | "max") reduces in place;
    alltoallv(send: np.ndarray[int8], send_counts, recv: np.ndarray[int8],
    recv_counts) moves per-rank segments of 8-byte elements in rank order."""
    def red(op):
        def cb(_u, buf, count):
            try:
                allreduce(np.ctypeslib.as_array(buf, shape=(count,)), op)
                return 0
            except Exception:  # noqa: BLE001 - reported as a status code
                import traceback
                traceback.print_exc()
                return 1
        return _REDUCE_CB(cb)

    def a2a(_u, send, scnt, recv, rcnt):
        try:
            sc = np.ctypeslib.as_array(scnt, shape=(nranks,)).copy()
            rc = np.ctypeslib.as_array(rcnt, shape=(nranks,)).copy()
            sb = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_int8)),
                                       shape=(8 * max(int(sc.sum()), 1),))
            rb = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_int8)),
                                       shape=(8 * max(int(rc.sum()), 1),))
            alltoallv(sb, sc, rb, rc)
            return 0
        except Exception:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1

    hc = _HostComm(None, red("sum"), red("max"), _A2A_CB(a2a))
    ctx._host_comm = hc  # the callbacks must outlive the context's use of them
    ctx.check(lib().rkmf_context_init_host_comm(ctx.h, nranks, rank, C.byref(hc)))
    ctx.nranks, ctx.rank = nranks, rank


def partition_rows(row_ptr, nranks: int) -> np.ndarray:
    """nnz-balanced contiguous row blocks: row_starts[nranks+1] (host)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    out = np.empty(nranks + 1, np.int64)
    lib().rkmf_partition_rows(len(rp) - 1, _ptr(rp), nranks, _ptr(out))
    return out


def local_rows(row_ptr, col_idx, values, row_starts, rank):
    """Rows [row_starts[rank], row_starts[rank+1]) with local row pointers and
    global columns."""
    rb, re = int(row_starts[rank]), int(row_starts[rank + 1])
    lo, hi = int(row_ptr[rb]), int(row_ptr[re])
    rp = np.ascontiguousarray(row_ptr[rb:re + 1] - lo, np.int64)
    return rp, np.ascontiguousarray(col_idx[lo:hi], np.int32), np.ascontiguousarray(values[lo:hi])


def partition_halo(row_starts, rank: int, rp_local, col_global):
    """Halo plan of one rank (host): (halo_global, recv_counts, col_local)."""
    rs = np.ascontiguousarray(row_starts, np.int64)
    rp = np.ascontiguousarray(rp_local, np.int64)
    cg = np.ascontiguousarray(col_global, np.int32)
    P = len(rs) - 1
    nh = C.c_int64()
    lib().rkmf_partition_halo(P, rank, _ptr(rs), _ptr(rp), _ptr(cg), C.byref(nh), None, None,
                              None)
    halo = np.empty(nh.value, np.int64)
    rc = np.empty(P, np.int64)
    cl = np.empty(len(cg), np.int32)
    lib().rkmf_partition_halo(P, rank, _ptr(rs), _ptr(rp), _ptr(cg), C.byref(nh), _ptr(halo),
                              _ptr(rc), _ptr(cl))
    return halo, rc, cl


def partitioned_matrix(ctx: Context, n_global: int, row_starts, rp_local, col_global,
                       values) -> SparseMatrix:
    rs = np.ascontiguousarray(row_starts, np.int64)
    rp = np.ascontiguousarray(rp_local, np.int64)
    cg = np.ascontiguousarray(col_global, np.int32)
    v = np.ascontiguousarray(values, np.float64)
    h = C.c_void_p()
    ctx.check(lib().rkmf_matrix_create_partitioned(ctx.h, n_global, _ptr(rs), _ptr(rp), _ptr(cg),
                                                   _ptr(v), C.byref(h)))
    return SparseMatrix(ctx, h)


def partitioned_sketch(ctx: Context, d: int, n_global: int, zeta: int, seed: int, col_begin: int,
                       n_local: int) -> SketchOperator:
    h = C.c_void_p()
    ctx.check(lib().rkmf_sketch_create_partitioned(ctx.h, d, n_global, zeta, C.c_uint64(seed),
                                                   col_begin, n_local, C.byref(h)))
    return SketchOperator(ctx, h, d, n_local, zeta, seed)


# ---- convergence sweep (restart.cpp:124-305) and its CSV (rkmf_bench.cpp:172-186) ----
@dataclass
class MethodSpec:
    """restart::MethodSpec (restart.hpp:81-97) for the device sweep."""
    name: str
    m: int = 100
    d: int = 0
    zeta: int = 4
    tol: float = 1e-10
    k_max: int = 100
    seed: int = 0


def convergence_sweep(A: SparseMatrix, b, f: FunctionSpec, methods, reference=None,
                      with_timing: bool = False) -> list:
    """Rows (dicts with the SweepRecord fields) of every method in order."""
    bb = np.ascontiguousarray(b, np.float64)
    ref = None if reference is None else np.ascontiguousarray(reference, np.float64)
    ms = (MethodSpecC * max(len(methods), 1))()
    for i, m in enumerate(methods):
        ms[i] = MethodSpecC(m.name.encode()[:31], m.m, m.d, m.zeta, m.tol, m.k_max, m.seed)
    n = C.c_int64()
    A.ctx.check(lib().rkmf_convergence_sweep(A.ctx.h, A.h, _ptr(bb), f.kind, f.t, _ptr(ref), ms,
                                             len(methods), int(with_timing), None, 0,
                                             C.byref(n)))
    recs = (SweepRecordC * max(n.value, 1))()
    A.ctx.check(lib().rkmf_convergence_sweep(A.ctx.h, A.h, _ptr(bb), f.kind, f.t, _ptr(ref), ms,
                                             len(methods), int(with_timing), recs, n.value,
                                             C.byref(n)))
    rows = []
    for i in range(n.value):
        r = recs[i]
        rows.append({k: (getattr(r, k).decode() if t in (C.c_char * 32, C.c_char * 256)
                         else getattr(r, k)) for k, t in SweepRecordC._fields_})
    return rows


def write_sweep_csv(rows, path: str = "") -> None:
    """The CLI's CSV (fixed header, %.17g numbers); "" writes to stdout."""
    recs = (SweepRecordC * max(len(rows), 1))()
    for i, r in enumerate(rows):
        vals = dict(r)
        vals["method"] = vals["method"].encode()
        vals["note"] = vals["note"].encode()
        recs[i] = SweepRecordC(**vals)
    err = C.create_string_buffer(512)
    _io_check(lib().rkmf_sweep_write_csv(recs, len(rows), os.fsencode(path), err, 512), err)


# ---- Matrix Market / vector interchange: sparse.cpp:140-242 (host only) ----
def _io_check(code: int, err) -> None:
    if code != RKMF_OK:
        raise _CODE.get(code, Error)(err.value.decode(errors="replace"))


def load_matrix_market(path: str):
    """sparse::load_matrix_market: (row_ptr int64, col_idx int32, values, n_rows, n_cols)."""
    nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
    rp, ci, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
    err = C.create_string_buffer(1024)
    _io_check(lib().rkmf_mtx_load(os.fsencode(path), C.byref(nr), C.byref(nc), C.byref(nz),
                                  C.byref(rp), C.byref(ci), C.byref(v), err, 1024), err)
    try:
        n, k = nr.value, nz.value
        out = (np.ctypeslib.as_array(C.cast(rp, C.POINTER(C.c_int64)), (n + 1,)).copy(),
               np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_int32)), (max(k, 1),))[:k].copy(),
               np.ctypeslib.as_array(C.cast(v, C.POINTER(C.c_double)), (max(k, 1),))[:k].copy(),
               n, nc.value)
    finally:
        for p in (rp, ci, v):
            lib().rkmf_host_free(p)
    return out


def save_matrix_market(A, path: str) -> None:
    """sparse::save_matrix_market of a SparseMatrix (device) or a host CSR
    tuple (row_ptr, col_idx, values[, n_cols])."""
    if isinstance(A, SparseMatrix):
        A.save_mtx(path)
        return
    rp = np.ascontiguousarray(A[0], np.int64)
    ci = np.ascontiguousarray(A[1], np.int32)
    v = np.ascontiguousarray(A[2], np.float64)
    nc = int(A[3]) if len(A) > 3 else len(rp) - 1
    err = C.create_string_buffer(1024)
    _io_check(lib().rkmf_mtx_save(os.fsencode(path), len(rp) - 1, nc, _ptr(rp), _ptr(ci), _ptr(v),
                                  err, 1024), err)


def load_vector(path: str) -> np.ndarray:
    """sparse::load_vector (sparse.cpp:213-231)."""
    n, p = C.c_int64(), C.c_void_p()
    err = C.create_string_buffer(1024)
    _io_check(lib().rkmf_vector_load(os.fsencode(path), C.byref(n), C.byref(p), err, 1024), err)
    try:
        k = n.value
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), (max(k, 1),))[:k].copy()
    finally:
        lib().rkmf_host_free(p)


def save_vector(v, path: str) -> None:
    """sparse::save_vector (sparse.cpp:233-242), %.17g per line."""
    x = np.ascontiguousarray(v.cpu().numpy() if hasattr(v, "cpu") else v, np.float64)
    err = C.create_string_buffer(1024)
    _io_check(lib().rkmf_vector_save(os.fsencode(path), len(x), _ptr(x), err, 1024), err)


# ---- synthetic inputs (host; need only the shared library, not a GPU) ----
def _gen(fn, *args):
    n, nnz = C.c_int64(), C.c_int64()
    code = fn(*args, C.byref(n), C.byref(nnz), None, None, None)
    if code != RKMF_OK:
        raise ParameterError("generator: invalid parameters")
    rp = np.empty(n.value + 1, np.int64)
    ci = np.empty(nnz.value, np.int32)
    v = np.empty(nnz.value, np.float64)
    fn(*args, C.byref(n), C.byref(nnz), _ptr(rp), _ptr(ci), _ptr(v))
    return rp, ci, v


def gen_laplacian(dim: int, N: int):
    """2D 5-point / 3D 7-point Dirichlet Laplacian scaled by h^-2 (CSR arrays)."""
    return _gen(lib().rkmf_gen_laplacian, dim, N)


def gen_q1_hex(N: int, lognormal: bool = False, coef_seed: int = 1, dirichlet: bool = False):
    """Q1 hexahedral 27-point stiffness matrix on an N^3 node grid (CSR arrays)."""
    return _gen(lib().rkmf_gen_q1_hex, N, int(lognormal), C.c_uint64(coef_seed), int(dirichlet))


def gen_convdiff_upwind(N: int, peclet: float = 10.0, v=(1.0, 0.5, 0.25)):
    """3D upwind convection-diffusion, 7-point (CSR arrays)."""
    return _gen(lib().rkmf_gen_convdiff_upwind, N, float(peclet), float(v[0]), float(v[1]),
                float(v[2]))


def gen_gaussian_device(seed: int, i0: int, n: int, ctx: Optional[Context] = None):
    """gen_gaussian_range on the device: a float64 CUDA tensor."""
    import torch
    ctx = ctx or Context.default()
    out = torch.empty(n, dtype=torch.float64, device=f"cuda:{ctx.device}")
    ctx.check(lib().rkmf_gen_gaussian_device(ctx.h, C.c_uint64(seed), i0, n, out.data_ptr()))
    return out


def gen_gaussian_range(seed: int, i0: int, n: int) -> np.ndarray:
    """Entries [i0, i0 + n) of gen_gaussian(seed, .) (one rank's slice of b)."""
    out = np.empty(n, np.float64)
    if lib().rkmf_gen_gaussian_range(C.c_uint64(seed), i0, n, _ptr(out)) != RKMF_OK:
        raise ParameterError("gen_gaussian_range: bad range")
    return out


def gen_gaussian(seed: int, n: int) -> np.ndarray:
    """b[i] = N(0,1) draw of SplitMix64(derive(seed, i)) (rng.hpp:47-59)."""
    out = np.empty(n)
    lib().rkmf_gen_gaussian(C.c_uint64(seed), n, _ptr(out))
    return out


__all__ = ["Context", "SparseMatrix", "SketchOperator", "make_sketch", "spmv", "sketch_apply",
           "spmv_sketch", "randomized_arnoldi", "KrylovDecomposition", "FunctionSpec",
           "RestartOptions", "RestartResult", "CycleRecord", "CycleInfo", "restarted_krylov", "gen_laplacian",
           "gen_q1_hex", "gen_convdiff_upwind", "gen_gaussian", "load_matrix_market",
           "save_matrix_market", "load_vector", "save_vector", "Error", "ShapeError",
           "ParameterError", "ParseError", "NumericalError", "DeviceError", "build", "lib",
           "SYMBOLS"]
