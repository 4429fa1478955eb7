"""cfg3 at full size (8M rows, lognormal Q1 with Dirichlet rows, z^{-1/2}, m =
40, d = 160): per-cycle update norm, kappa(W_m) and the Ritz values of the
cycle's compression H_k, to tell the method's behaviour from the quadrature's.

  python tools/cfg3_diagnose.py [cycles]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 16
P = configs.build_device("cfg3")
S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
f = rk.FunctionSpec.inv_sqrt()
print(f"cfg3: n={P.n} nnz={P.nnz} m={P.m} d={P.d} tol={P.tol:.3e}", flush=True)
ritz = []


def obs(info):
    M = info.R_accum.shape[0]
    H = info.R_accum[M - info.m_k:, M - info.m_k:]
    ritz.append(np.linalg.eigvals(H))


# fixed nodes: no branch-cut guard, so the iteration runs on
r = rk.restarted_krylov(P.A, P.b, f, rk.RestartOptions(m_r=P.m, tol=1e-30, k_max=cycles,
                                                       quad_nodes=512, diagnostics=True),
                        S, observer=obs)
print(f"{'cycle':>5} {'update_norm':>12} {'kappa_W':>10} {'min Re':>12} {'min |lam|':>11} "
      f"{'max arg/pi':>10} {'#Re<=0':>6}")
for h, lam in zip(r.history, ritz):
    print(f"{h.cycle:5d} {h.update_norm:12.4e} {h.kappa_W:10.3e} {lam.real.min():12.4e} "
          f"{np.abs(lam).min():11.4e} {np.abs(np.angle(lam)).max() / np.pi:10.4f} "
          f"{int((lam.real <= 0).sum()):6d}", flush=True)
try:
    r2 = rk.restarted_krylov(P.A, P.b, f, rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max), S)
    print(f"adaptive quadrature: converged={r2.converged} cycles={r2.cycles} nodes={r2.quad_nodes}")
except rk.NumericalError as e:
    print(f"adaptive quadrature: NumericalError: {e}")
