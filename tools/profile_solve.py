"""One device-resident solve of a BASELINE config, for ncu captures.

    python tools/profile_solve.py [cfg2] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
P = configs.build(name)
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
b = torch.tensor(P.b, device="cuda")
for _ in range(reps):
    r = rk.restarted_krylov(A, b, f, opts, S)
torch.cuda.synchronize()
print(f"{name}: cycles={r.cycles} total_m={r.total_m} solve_ms={r.solve_ms:.3f} "
      f"launches={A.ctx.launch_count}")
