"""The five BASELINE.json configurations as seeded synthetic problems.

Each config fixes the matrix generator, the function f, m, the sketch size
d = s, zeta = 8 and the relative tolerance. Shared by tests and bench.py so the
device path and the CPU oracle always see the same CSR, b, S and t.

Conventions (documented in DESIGN.md):
  * b[i] = N(0,1) from SplitMix64(derive(b_seed, i)) (rng.hpp:47-59), b_seed = 1.
  * S = make_sketch(d, n, 8, sketch_seed = 1) (sketch.cpp:13-49).
  * tol_abs = tol_rel * ||b||_2 (the reference's own convention,
    proj/tests/acceptance.cpp:358).
  * t = c / ||A||_2; ||A||_2 analytic for the Dirichlet Laplacians, else a
    fixed-seed, fixed-iteration power iteration (on A^T A when nonsymmetric),
    as the reference's acceptance test does (acceptance.cpp:429-437).
  * k_max = floor(budget_total_m / m) with the reference's budget 4000.

Two interchangeable generator backends build the same arrays bit-for-bit
(tests/test_generators.py): "product" (the library's host generators,
csrc/problems.cpp) and "oracle" (oracle/problems_oracle.cpp, test
infrastructure). bench.py's reference arm uses the oracle backend so that its
process never maps the product library.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np


CONFIGS = {
    "cfg1": dict(kind="lap2d", N=256, fn="exp_neg", c=100.0, m=30, d=120, zeta=8, tol_rel=1e-8),
    "cfg2": dict(kind="lap3d", N=128, fn="exp_neg", c=500.0, m=50, d=200, zeta=8, tol_rel=1e-8),
    "cfg3": dict(kind="q1", N=200, lognormal=True, dirichlet=True, fn="inv_sqrt", m=40, d=160,
                 zeta=8, tol_rel=1e-7),
    "cfg4": dict(kind="convdiff", N=256, peclet=10.0, v=(1.0, 0.5, 0.25), fn="exp_neg", c=200.0,
                 m=30, d=120, zeta=8, tol_rel=1e-8),
    "cfg5": dict(kind="q1", N=512, lognormal=False, dirichlet=False, fn="exp_neg", c=300.0, m=50,
                 d=200, zeta=8, tol_rel=1e-8),
}
BUDGET_TOTAL_M = 4000
B_SEED, SKETCH_SEED, COEF_SEED = 1, 1, 1
POWER_SEED, POWER_ITERS = 7, 60

# ||A||_2 estimates of the full-size configs whose t comes from the power
# iteration (60 fixed-seed iterations, power_norm2 / device_power_norm2),
# computed once and frozen so that every process (both bench arms, the
# device-generated problems) uses the same t without re-running a 117M- or
# 3.6G-nonzero power iteration at start-up. tests/test_generators.py and
# tests/test_gpu_fullsize.py recompute them.
NORM2_FROZEN = {
    ("cfg4", 256): 1046.860307424342,  # power_norm2 (A^T A), host scipy
    ("cfg5", 512): 0.007727342009466925,  # device_power_norm2 (tools/freeze_norms.py)
}
# ||b||_2 of the full-size cfg5 right-hand side (134M entries), so the
# row-partitioned runs and the one-GPU run use one tol without a global
# reduction at set-up (np.linalg.norm of gen_gaussian(B_SEED, 512^3)).
BNORM_FROZEN = {
    ("cfg5", 512): 11584.694751146742,
}


class _Gen:
    """The generator backend: the product library's host generators or the
    oracle's independent restatement (same arrays bit-for-bit)."""

    def __init__(self, backend: str):
        if backend not in ("product", "oracle"):
            raise ValueError(f"unknown generator backend {backend!r}")
        self.backend = backend

    def _mod(self):
        if self.backend == "product":
            import paper_2503_22631_b200 as m
            return m
        from oracle import oracle as m
        return m

    def laplacian(self, dim, N):
        return self._mod().gen_laplacian(dim, N)

    def q1_hex(self, N, lognormal, seed, dirichlet):
        return self._mod().gen_q1_hex(N, lognormal, seed, dirichlet)

    def convdiff(self, N, peclet, v):
        return self._mod().gen_convdiff_upwind(N, peclet, v)

    def gaussian(self, seed, n):
        m = self._mod()
        return m.gen_gaussian(seed, n) if self.backend == "product" else m.gaussian_vector(seed, n)


@dataclass
class Problem:
    name: str
    n: int
    nnz: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    b: np.ndarray
    fn: str
    t: float
    m: int
    d: int
    zeta: int
    tol: float  # absolute
    k_max: int
    norm2: float

    def scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr), shape=(self.n, self.n))


def lap_lambda_max(dim: int, N: int) -> float:
    h = 1.0 / (N + 1)
    return (4.0 * dim / (h * h)) * math.sin(N * math.pi / (2 * N + 2)) ** 2


def power_norm2(rp, ci, v, n, symmetric: bool, iters: int = POWER_ITERS, seed: int = POWER_SEED,
                backend: str = "product") -> float:
    """Deterministic power iteration for ||A||_2 (host, scipy)."""
    import scipy.sparse as sp
    A = sp.csr_matrix((v, ci, rp), shape=(n, n))
    x = _Gen(backend).gaussian(seed, n)
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = A @ x if symmetric else A.T @ (A @ x)
        lam = float(np.linalg.norm(y))
        x = y / lam
    return lam if symmetric else math.sqrt(lam)


def frozen_norm2(name: str, N: int) -> Optional[float]:
    return NORM2_FROZEN.get((name, int(N)))


def frozen_tol(name: str, N: int) -> Optional[float]:
    """tol_rel * ||b||_2 from BNORM_FROZEN, or None."""
    bn = BNORM_FROZEN.get((name, int(N)))
    return None if bn is None else CONFIGS[name]["tol_rel"] * bn


def build(name: str, N: Optional[int] = None, with_b: bool = True,
          backend: str = "product", frozen: bool = True) -> Problem:
    """Build config `name`; N overrides the grid size (scaled-down parity
    cases). backend: "product" or "oracle" generators (identical arrays).
    frozen: use NORM2_FROZEN for ||A||_2 where recorded."""
    cfg = dict(CONFIGS[name])
    N = int(N or cfg["N"])
    kind = cfg["kind"]
    G = _Gen(backend)
    fz = frozen_norm2(name, N) if frozen else None
    if kind == "lap2d":
        rp, ci, v = G.laplacian(2, N)
        norm2 = lap_lambda_max(2, N)
    elif kind == "lap3d":
        rp, ci, v = G.laplacian(3, N)
        norm2 = lap_lambda_max(3, N)
    elif kind == "q1":
        rp, ci, v = G.q1_hex(N, cfg["lognormal"], COEF_SEED, cfg["dirichlet"])
        norm2 = 0.0
        if cfg["fn"] == "exp_neg":
            norm2 = fz if fz is not None else power_norm2(rp, ci, v, len(rp) - 1, True,
                                                          backend=backend)
    elif kind == "convdiff":
        rp, ci, v = G.convdiff(N, cfg["peclet"], cfg["v"])
        norm2 = fz if fz is not None else power_norm2(rp, ci, v, len(rp) - 1, False,
                                                      backend=backend)
    else:
        raise ValueError(kind)
    n = len(rp) - 1
    b = G.gaussian(B_SEED, n) if with_b else None
    t = cfg["c"] / norm2 if cfg["fn"] == "exp_neg" else 1.0
    tol = cfg["tol_rel"] * (float(np.linalg.norm(b)) if with_b else math.sqrt(n))
    return Problem(name=name, n=n, nnz=int(rp[-1]), row_ptr=rp, col_idx=ci, values=v, b=b,
                   fn=cfg["fn"], t=t, m=cfg["m"], d=cfg["d"], zeta=cfg["zeta"], tol=tol,
                   k_max=BUDGET_TOTAL_M // cfg["m"], norm2=norm2)


def algorithmic_bytes_per_cycle(n: int, nnz: int, m: int, rp_bytes: int = 4) -> int:
    """B_cycle = sum_k B_step(k) + 8n + 16n + 8n(m+2).

    B_step(k) = 12 nnz + rp (n+1) + 8n (x) + 8n (z write) + 8n (k+1) (W read)
                + 8n (z read) + 8n (w_{k+1} write).
    Sketch metadata excluded (regenerable from the seed).
    """
    total = 0
    for k in range(m):
        total += 12 * nnz + rp_bytes * (n + 1) + 8 * n * 4 + 8 * n * (k + 1)
    total += 8 * n + 16 * n + 8 * n * (m + 2)
    return total


@dataclass
class Slab:
    """One rank's rows of the weak-scaling problem (bench.py --gpus N)."""
    name: str
    n_global: int
    row_starts: np.ndarray
    row_ptr: np.ndarray   # local row pointers
    col_idx: np.ndarray   # GLOBAL column indices (int32)
    values: np.ndarray
    b: np.ndarray         # local slice
    nnz: int              # local
    nnz_global: int
    fn: str
    t: float
    m: int
    d: int
    zeta: int
    tol: float
    k_max: int


def build_slab(world: int, rank: int, N: int = 128) -> Slab:
    """cfg2 weak-scaled: the 7-point Laplacian on an (N*world) x N x N interior
    grid (spacing h = 1/(N+1) in every direction, Dirichlet boundary
    eliminated, scaled by h^-2), lexicographic order (ix*N + iy)*N + iz, so
    rank r owns the x-slab ix in [rN, (r+1)N): exactly cfg2's rows and stencil
    per rank, with one N^2 halo plane to each neighbour. Only the rank's rows
    are generated. f = exp(-tA), t = 500 / lambda_max, m = 50, d = 200."""
    cfg = CONFIGS["cfg2"]
    Nx, plane = N * world, N * N
    n_global = Nx * plane
    h = 1.0 / (N + 1)
    s = 1.0 / (h * h)
    r0, r1 = rank * N * plane, (rank + 1) * N * plane
    rows = np.arange(r0, r1, dtype=np.int64)
    ix, iy, iz = rows // plane, (rows // N) % N, rows % N
    # neighbours in increasing column order: -x, -y, -z, self, +z, +y, +x
    offs = [-plane, -N, -1, 0, 1, N, plane]
    ok = [ix > 0, iy > 0, iz > 0, np.ones_like(ix, bool), iz < N - 1, iy < N - 1, ix < Nx - 1]
    cols = np.stack([rows + o for o in offs], axis=1)
    vals = np.where(np.arange(7) == 3, 6.0 * s, -s)[None, :].repeat(len(rows), 0)
    mask = np.stack(ok, axis=1)
    row_ptr = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(mask.sum(1), out=row_ptr[1:])
    col_idx = cols[mask].astype(np.int32)
    values = vals[mask].astype(np.float64)
    lam = lap_lambda_max(3, N) if world == 1 else (4.0 / (h * h)) * (
        math.sin(Nx * math.pi / (2 * Nx + 2)) ** 2 + 2 * math.sin(N * math.pi / (2 * N + 2)) ** 2)
    from . import gen_gaussian_range
    b = gen_gaussian_range(B_SEED, r0, r1 - r0)
    # ||b||_2 of the global vector without materialising it: sum of squares of
    # every rank's slice is deterministic, so compute it slab by slab
    ss = 0.0
    for q in range(world):
        ss += float(np.dot(*(2 * [gen_gaussian_range(B_SEED, q * N * plane, N * plane)])))
    # 7 per row minus one per missing neighbour: two boundary faces per axis
    nnz_global = 7 * n_global - 2 * (N * N + Nx * N + Nx * N)
    row_starts = np.arange(world + 1, dtype=np.int64) * N * plane
    return Slab(name="cfg2-slab", n_global=n_global, row_starts=row_starts, row_ptr=row_ptr,
                col_idx=col_idx, values=values, b=b, nnz=int(row_ptr[-1]),
                nnz_global=int(nnz_global), fn="exp_neg", t=cfg["c"] / lam, m=cfg["m"],
                d=cfg["d"], zeta=cfg["zeta"], tol=cfg["tol_rel"] * math.sqrt(ss),
                k_max=BUDGET_TOTAL_M // cfg["m"])


@dataclass
class DeviceProblem:
    """A BASELINE config generated in HBM (cfg5's 3.6e9 nonzeros never touch
    the host): the device matrix, the device b, and the solver parameters."""
    name: str
    n: int
    nnz: int
    A: object   # SparseMatrix
    b: object   # float64 CUDA tensor
    fn: str
    t: float
    m: int
    d: int
    zeta: int
    tol: float
    k_max: int
    norm2: float


def device_power_norm2(A, iters: int = 60, seed: int = 7) -> float:
    """||A||_2 of a symmetric device matrix by a fixed-seed power iteration
    (the host power_norm2 on the device: same start vector, same count)."""
    from . import gen_gaussian_device, spmv
    x = gen_gaussian_device(seed, 0, A.n_rows, A.ctx)
    x /= x.norm()
    lam = 0.0
    for _ in range(iters):
        y = spmv(A, x)
        lam = float(y.norm())
        x = y / lam
    return lam


def build_device(name: str, N: Optional[int] = None, ctx=None) -> DeviceProblem:
    """Config `name` generated in HBM (Laplacians, Q1, upwind
    convection-diffusion: the host generators' entries bit-for-bit, the
    lognormal Q1 coefficients to an ulp). tol uses the same ||b||_2 as build()
    (numpy on the host copy) or BNORM_FROZEN."""
    from . import Context, SparseMatrix, gen_gaussian_device
    cfg = dict(CONFIGS[name])
    N = int(N or cfg["N"])
    ctx = ctx or Context.default()
    kind = cfg["kind"]
    if kind == "lap2d":
        A = SparseMatrix.laplacian(2, N, ctx)
        norm2 = lap_lambda_max(2, N)
    elif kind == "lap3d":
        A = SparseMatrix.laplacian(3, N, ctx)
        norm2 = lap_lambda_max(3, N)
    elif kind == "q1":
        A = SparseMatrix.q1_hex(N, cfg["lognormal"], COEF_SEED, cfg["dirichlet"], ctx)
        norm2 = 0.0
        if cfg["fn"] == "exp_neg":
            norm2 = frozen_norm2(name, N) or device_power_norm2(A)
    elif kind == "convdiff":
        A = SparseMatrix.convdiff(N, cfg["peclet"], cfg["v"], ctx)
        norm2 = frozen_norm2(name, N)
        if norm2 is None:  # A^T A needs the transpose: build() on the host
            norm2 = build(name, N, with_b=False).norm2
    else:
        raise ValueError(f"{name}: no device generator for {kind}")
    b = gen_gaussian_device(B_SEED, 0, A.n_rows, ctx)
    t = cfg["c"] / norm2 if cfg["fn"] == "exp_neg" else 1.0
    tol = frozen_tol(name, N) or cfg["tol_rel"] * float(np.linalg.norm(b.cpu().numpy()))
    return DeviceProblem(name=name, n=A.n_rows, nnz=A.nnz, A=A, b=b, fn=cfg["fn"], t=t,
                         m=cfg["m"], d=cfg["d"], zeta=cfg["zeta"], tol=tol,
                         k_max=BUDGET_TOTAL_M // cfg["m"], norm2=norm2)
