"""The paper's restart vs restart-rand comparison on B200: the
same restarted f(A)b solve with the classical builder (S = None, CGS2 on
device) and the randomized builder (sketched Gram-Schmidt), same matrix, b,
m, tolerance.

    python tools/compare_builders.py [cfg2 cfg4 ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

for name in sys.argv[1:] or ["cfg2", "cfg4"]:
    P = configs.build(name)
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    b = torch.tensor(P.b, device="cuda")
    out = {}
    for label, sk in (("restart (classical)", None), ("restart-rand", S)):
        rk.restarted_krylov(A, b, f, opts, sk)  # warm-up
        best = None
        for _ in range(3):
            r = rk.restarted_krylov(A, b, f, opts, sk)
            best = r if best is None or r.solve_ms < best.solve_ms else best
        out[label] = best
        print(f"{name} {label:20s}: cycles={best.cycles} total_m={best.total_m} "
              f"solve_ms={best.solve_ms:.2f} vec/s={best.total_m / best.solve_ms * 1e3:.0f}",
              flush=True)
    fc = out["restart (classical)"].f_hat.cpu().numpy()
    fr = out["restart-rand"].f_hat.cpu().numpy()
    sp = out["restart (classical)"].solve_ms / out["restart-rand"].solve_ms
    print(f"{name}: restart-rand speed-up {sp:.2f}x; ||f_c - f_r|| / ||f_c|| = "
          f"{np.linalg.norm(fc - fr) / np.linalg.norm(fc):.2e}", flush=True)
