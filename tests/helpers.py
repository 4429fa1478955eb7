"""Seeded small test problems (restating the roles of proj/tests/oracles.hpp)."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def random_sparse(n: int, density: float, seed: int, shift: float = 0.0) -> sp.csr_matrix:
    """Random nonsymmetric sparse matrix with a full diagonal (oracles.hpp:127-160 role)."""
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=rng, format="csr",
                  data_rvs=lambda k: rng.standard_normal(k))
    A = (A + sp.diags(rng.standard_normal(n) + shift)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


def random_spd_tridiag(n: int, lo: float, hi: float, seed: int) -> sp.csr_matrix:
    """SPD tridiagonal with diagonal in [lo, hi] + 2 (oracles.hpp:162-175 role)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(lo, hi, n) + 2.0
    off = -np.ones(n - 1)
    A = sp.diags([off, d, off], [-1, 0, 1]).tocsr()
    A.sort_indices()
    return A


def random_vector(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


def conv_diff_2d(nx: int, ny: int, eps: float, vx: float, vy: float) -> sp.csr_matrix:
    """Centred 2D convection-diffusion (the reference's gen_conv_diff family,
    problems.cpp:292-377, here with the boundary eliminated)."""
    hx, hy = 1.0 / (nx + 1), 1.0 / (ny + 1)
    Tx = sp.diags([-(eps / hx**2 + vx / (2 * hx)) * np.ones(nx - 1), 2 * eps / hx**2 * np.ones(nx),
                   -(eps / hx**2 - vx / (2 * hx)) * np.ones(nx - 1)], [-1, 0, 1])
    Ty = sp.diags([-(eps / hy**2 + vy / (2 * hy)) * np.ones(ny - 1), 2 * eps / hy**2 * np.ones(ny),
                   -(eps / hy**2 - vy / (2 * hy)) * np.ones(ny - 1)], [-1, 0, 1])
    A = (sp.kron(Tx, sp.eye(ny)) + sp.kron(sp.eye(nx), Ty)).tocsr()
    A.sort_indices()
    return A


def dense_sketch(rows: np.ndarray, signs: np.ndarray, scale: float, d: int, n: int,
                 zeta: int) -> np.ndarray:
    """oracles.hpp:55-61: densified S."""
    S = np.zeros((d, n))
    for j in range(n):
        for k in range(zeta):
            S[rows[j * zeta + k], j] += scale * signs[j * zeta + k]
    return S


# ---- an independent, pure-Python restatement of SplitMix64 / make_sketch ----
M64 = (1 << 64) - 1


def sm64_next(state):
    state[0] = (state[0] + 0x9E3779B97F4A7C15) & M64
    z = state[0]
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def sm64_derive(seed: int, tag: int) -> int:
    st = [(seed ^ ((0xA0761D6478BD642F + tag * 0xE7037ED1A0B428DB) & M64)) & M64]
    return sm64_next(st)


def py_make_sketch(d: int, n: int, zeta: int, seed: int):
    """rng.hpp:17-63 + sketch.cpp:13-49 in pure Python (small n only)."""
    rows = np.empty(n * zeta, np.int64)
    signs = np.empty(n * zeta, np.int8)
    for j in range(n):
        st = [sm64_derive(seed, j)]
        chosen = []
        for i in range(d - zeta, d):
            bound = i + 1
            limit = (bound * (M64 // bound)) & M64
            while True:
                v = sm64_next(st)
                if v < limit:
                    break
            t = v % bound
            chosen.append(i if t in chosen else t)
        chosen.sort()
        for k in range(zeta):
            rows[j * zeta + k] = chosen[k]
            signs[j * zeta + k] = 1 if (sm64_next(st) & 1) else -1
    return rows, signs
