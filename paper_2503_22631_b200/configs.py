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
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import gen_convdiff_upwind, gen_gaussian, gen_laplacian, gen_q1_hex

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


def power_norm2(rp, ci, v, n, symmetric: bool, iters: int = 60, seed: int = 7) -> float:
    """Deterministic power iteration for ||A||_2 (host, scipy)."""
    import scipy.sparse as sp
    A = sp.csr_matrix((v, ci, rp), shape=(n, n))
    x = gen_gaussian(seed, n)
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = A @ x if symmetric else A.T @ (A @ x)
        lam = float(np.linalg.norm(y))
        x = y / lam
    return lam if symmetric else math.sqrt(lam)


def build(name: str, N: Optional[int] = None, with_b: bool = True) -> Problem:
    """Build config `name`; N overrides the grid size (scaled-down parity cases)."""
    cfg = dict(CONFIGS[name])
    N = int(N or cfg["N"])
    kind = cfg["kind"]
    if kind == "lap2d":
        rp, ci, v = gen_laplacian(2, N)
        norm2 = lap_lambda_max(2, N)
    elif kind == "lap3d":
        rp, ci, v = gen_laplacian(3, N)
        norm2 = lap_lambda_max(3, N)
    elif kind == "q1":
        rp, ci, v = gen_q1_hex(N, cfg["lognormal"], COEF_SEED, cfg["dirichlet"])
        norm2 = power_norm2(rp, ci, v, len(rp) - 1, True) if cfg["fn"] == "exp_neg" else 0.0
    elif kind == "convdiff":
        rp, ci, v = gen_convdiff_upwind(N, cfg["peclet"], cfg["v"])
        norm2 = power_norm2(rp, ci, v, len(rp) - 1, False)
    else:
        raise ValueError(kind)
    n = len(rp) - 1
    b = gen_gaussian(B_SEED, n) if with_b else None
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
    """Config `name` generated on the device (Laplacians and Q1; cfg4's
    upwind operator has no device generator and uses build())."""
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
        norm2 = device_power_norm2(A) if cfg["fn"] == "exp_neg" else 0.0
    else:
        raise ValueError(f"{name}: no device generator for {kind}")
    b = gen_gaussian_device(B_SEED, 0, A.n_rows, ctx)
    t = cfg["c"] / norm2 if cfg["fn"] == "exp_neg" else 1.0
    return DeviceProblem(name=name, n=A.n_rows, nnz=A.nnz, A=A, b=b, fn=cfg["fn"], t=t,
                         m=cfg["m"], d=cfg["d"], zeta=cfg["zeta"],
                         tol=cfg["tol_rel"] * float(b.norm()), k_max=BUDGET_TOTAL_M // cfg["m"],
                         norm2=norm2)
