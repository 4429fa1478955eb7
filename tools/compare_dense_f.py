"""FULL f(R_accum) vs restart quadrature for exp(-tA):
solve time, dense-f time per cycle, agreement.

    python tools/compare_dense_f.py [cfg1 cfg2 cfg4] [--m M] [--kmax K]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["cfg1", "cfg2", "cfg4"])
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--tol", type=float, default=0.0)
args = ap.parse_args()
for name in args.configs:
    P = configs.build(name)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d if not args.m else 4 * args.m, P.n, P.zeta, configs.SKETCH_SEED)
    f = rk.FunctionSpec.exp_neg(P.t)
    b = torch.tensor(P.b, device="cuda")
    m = args.m or P.m
    tol = args.tol * float(np.linalg.norm(P.b)) if args.tol else P.tol
    res = {}
    for mode in ("full", "quadrature"):
        o = rk.RestartOptions(m_r=m, tol=tol, k_max=4000 // m, dense_f=mode)
        rk.restarted_krylov(A, b, f, o, S)
        r = min((rk.restarted_krylov(A, b, f, o, S) for _ in range(3)), key=lambda r: r.solve_ms)
        res[mode] = r
        fm = [h.funm_ms for h in r.history]
        print(f"{name} m={m} {mode:10s}: cycles={r.cycles} total_m={r.total_m} "
              f"solve_ms={r.solve_ms:.2f} dense_f_ms total={sum(fm):.2f} "
              f"last={fm[-1]:.3f}", flush=True)
    a, q = res["full"].f_hat.cpu().numpy(), res["quadrature"].f_hat.cpu().numpy()
    print(f"{name}: ||f_quad - f_full|| / ||f_full|| = {np.linalg.norm(a - q) / np.linalg.norm(a):.2e}",
          flush=True)
