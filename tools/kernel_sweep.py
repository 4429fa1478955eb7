"""Per-kernel device times of one device-resident solve (CUDA events around
every launch, rkmf_context_kernel_timing) for A/B runs of the env tunables:

    RKMF_PIPE_STAGES=3 python tools/kernel_sweep.py [cfg2] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P = configs.build(name)
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
b = torch.tensor(P.b, device="cuda")
ctx = A.ctx
r = rk.restarted_krylov(A, b, f, opts, S)  # warm-up
ctx.kernel_timing(True)
t = []
for _ in range(reps):
    r = rk.restarted_krylov(A, b, f, opts, S)
    t.append(r.solve_ms)
times = ctx.kernel_times()
ctx.kernel_timing(False)
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("RKMF_"))
per = {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in times.items() if v[1]}
print(f"[{env or 'default'}] {name} solve_ms={min(t):.3f} cycles={r.cycles} us/launch={per}")
