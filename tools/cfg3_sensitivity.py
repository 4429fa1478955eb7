"""cfg3's kind (lognormal Q1 with Dirichlet rows, z^{-1/2}, m = 40, d = 160,
tol 1e-7 relative) on an N^3 grid, CPU oracle only: how much the restart
process amplifies rounding, and whether the dense f(R_accum) is the cause.

1. the oracle's Denman-Beavers f(R_accum) e1 against a Schur-method sqrtm
   (scipy) and the trapezoid quadrature the device uses (numpy restatement)
   on the converged R_accum;
2. the oracle against itself with different summation orders (threads = 1,
   2, 8: the parallel reductions split differently): cycle counts and the
   relative difference of the converged f_hat;
3. the same at forced equal cycle counts;
4. b scaled by (1 + 2^-50) (no change in exact arithmetic: f(A) is linear),
   one cycle and converged, and the first cycle's kappa(W) and Rbar
   subdiagonal (the dense steps are well conditioned).

  python tools/cfg3_sensitivity.py [N]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sl  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def quad_invsqrt_e1(R, h, lmin, lmax):
    """(2/pi) sum_q h e^{u_q} (e^{2 u_q} I + R)^{-1} e1 (densef.cu invsqrt_nodes)."""
    M = R.shape[0]
    e1 = np.zeros(M)
    e1[0] = 1.0
    u0 = 0.5 * np.log(lmin / 4) - 38.0
    u1 = 0.5 * np.log(lmax * 4) + 38.0
    nq = int(np.ceil((u1 - u0) / h))
    acc = np.zeros(M)
    for i in range(nq):
        u = u0 + (i + 0.5) * h
        acc += (2 / np.pi) * h * np.exp(u) * np.linalg.solve(np.exp(2 * u) * np.eye(M) + R, e1)
    return acc, nq


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 56
    P = configs.build("cfg3", N, backend="oracle")
    S = O.make_sketch(P.d, P.n, P.zeta, 1)
    A = (P.row_ptr, P.col_idx, P.values)
    print(f"cfg3 kind N={N}: n={P.n} m={P.m} d={P.d} tol={P.tol:.3e}")
    runs = {}
    for th in (1, 2, 8):
        t0 = time.time()
        runs[th] = O.restarted_krylov(A, P.b, O.KIND_INV_SQRT, P.t, m_r=P.m, tol=P.tol,
                                      k_max=P.k_max, S=S, threads=th, want_R=(th == 1))
        o = runs[th]
        print(f"threads={th}: cycles={o.cycles} converged={o.converged} "
              f"last updates={[round(h['update_norm'], 9) for h in o.history][-3:]} "
              f"({time.time() - t0:.1f} s)", flush=True)
    for a in (2, 8):
        print(f"f_hat threads={a} vs threads=1: {rel(runs[a].f_hat, runs[1].f_hat):.3e}")
    R = runs[1].R_accum
    M = R.shape[0]
    e1 = np.zeros(M)
    e1[0] = 1.0
    ev = np.linalg.eigvals(R)
    Fs = np.linalg.solve(sl.sqrtm(R), e1)
    Fdb = O.funm(R, O.KIND_INV_SQRT, 0.0)[:, 0]
    Fq, nq = quad_invsqrt_e1(R, 0.25, np.abs(ev).min(), np.abs(ev).max())
    print(f"R_accum {M}x{M}: |lambda| in [{np.abs(ev).min():.3e}, {np.abs(ev).max():.3e}], "
          f"max |arg| {np.abs(np.angle(ev)).max():.3f}")
    print(f"f(R_accum) e1: Denman-Beavers vs Schur sqrtm {rel(Fdb, Fs):.2e}; "
          f"quadrature ({nq} nodes) vs Schur sqrtm {rel(Fq, Fs):.2e}")
    for k in (1, 3, 6, 10):
        r1 = O.restarted_krylov(A, P.b, O.KIND_INV_SQRT, P.t, m_r=P.m, tol=1e-30, k_max=k, S=S,
                                threads=1)
        r8 = O.restarted_krylov(A, P.b, O.KIND_INV_SQRT, P.t, m_r=P.m, tol=1e-30, k_max=k, S=S,
                                threads=8)
        print(f"forced {k} cycles: threads=8 vs threads=1 {rel(r8.f_hat, r1.f_hat):.3e}", flush=True)
    delta = 2.0 ** -50
    for k, tol in ((1, 1e-30), (P.k_max, P.tol)):
        a = O.restarted_krylov(A, P.b, O.KIND_INV_SQRT, P.t, m_r=P.m, tol=tol, k_max=k, S=S)
        b = O.restarted_krylov(A, P.b * (1 + delta), O.KIND_INV_SQRT, P.t, m_r=P.m, tol=tol,
                               k_max=k, S=S)
        print(f"b * (1 + 2^-50), k_max={k}: cycles {a.cycles} vs {b.cycles}, f_hat "
              f"{rel(b.f_hat / (1 + delta), a.f_hat):.3e}", flush=True)
    D = O.arnoldi_decomp(A, P.b, P.m, S)
    W = np.asarray(D.W)[:, :P.m]
    sub = np.abs(np.diag(np.asarray(D.Rbar), -1))
    print(f"cycle 1: kappa(W_m) {np.linalg.cond(W):.3f}, Rbar subdiagonal in "
          f"[{sub.min():.3e}, {sub.max():.3e}], ||A||_1 {O.norm1(A):.4f}")


if __name__ == "__main__":
    main()
