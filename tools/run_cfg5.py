"""cfg5 (Q1 27-point, 512^3 nodes, n = 134M, 3.6e9 nonzeros, int64 row
pointers) on ONE B200: matrix and b generated in HBM, device sketch, one
restarted f(A)b solve with per-cycle records.

    python tools/run_cfg5.py [N] [k_max]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t0 = time.perf_counter()
P = configs.build_device("cfg5", N)
torch.cuda.synchronize()
t1 = time.perf_counter()
S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cfg5 N={N}: n={P.n} nnz={P.nnz} norm2={P.norm2:.6e} t={P.t:.6e} gen+power={t1-t0:.1f}s "
      f"sketch={t2-t1:.1f}s mem={torch.cuda.memory_allocated()/1e9:.1f}GB(torch)", flush=True)
f = rk.FunctionSpec.exp_neg(P.t)
opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=kmax or P.k_max)
A = P.A
A.ctx.kernel_timing(True)
r = rk.restarted_krylov(A, P.b, f, opts, S)
kt = A.ctx.kernel_times()
free, total = torch.cuda.mem_get_info()
print(f"cycles={r.cycles} total_m={r.total_m} converged={r.converged} solve_ms={r.solve_ms:.1f} "
      f"vec/s={r.total_m / r.solve_ms * 1e3:.1f} device_free={free/1e9:.1f}/{total/1e9:.1f}GB",
      flush=True)
print("updates", [f"{h.update_norm:.2e}" for h in r.history])
print("kernel ms", {k: (round(v[0], 2), v[1]) for k, v in kt.items()})
nnz, n, m = P.nnz, P.n, P.m
alg = configs.algorithmic_bytes_per_cycle(n, nnz, m, rp_bytes=8)
print(f"alg GB/cycle={alg/1e9:.1f} achieved={alg * r.cycles / (r.solve_ms / 1e3) / 1e9:.0f} GB/s")
