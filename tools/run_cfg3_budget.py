"""cfg3 (A^{-1/2} b on the lognormal Q1 matrix) at the reference's default
4000-vector budget and at 40000, with the update-norm history.

    python tools/run_cfg3_budget.py
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2503_22631_b200 as rk
from paper_2503_22631_b200 import configs
P = configs.build("cfg3")
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, 1)
b = torch.tensor(P.b, device="cuda")
for budget in (4000, 40000):
    r = rk.restarted_krylov(A, b, rk.FunctionSpec.inv_sqrt(),
                            rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=budget // P.m, budget_total_m=budget), S)
    un = [c.update_norm for c in r.history]
    print(budget, "cycles", r.cycles, "converged", r.converged, "solve_ms", round(r.solve_ms, 1),
          "tol", P.tol, "updates every 50:", ["%.2e" % u for u in un[::50]], "last", ["%.2e" % u for u in un[-5:]], flush=True)
