"""Microbenchmark of the fused SpMV+sketch kernel alone (rkmf_spmv_sketch).

    python tools/bench_spmv.py [cfg2] [iters]
Prints per-launch device time and the algorithmic GB/s (12 nnz + 4 (n+1) +
8n x + 8n z; sketch metadata excluded).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
P = configs.build(name)
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, 1)
x = torch.tensor(P.b, device="cuda")
z = torch.empty_like(x)
p = torch.empty(P.d, dtype=torch.float64, device="cuda")
L = rk.lib()
ctx = A.ctx
for _ in range(5):
    L.rkmf_spmv_sketch(ctx.h, A.h, S.h, x.data_ptr(), z.data_ptr(), p.data_ptr())
# rkmf_spmv_sketch synchronises per call; time with host clock around a loop,
# and with CUDA events per call on the context stream (own stream)
import time  # noqa: E402
t0 = time.perf_counter()
for _ in range(iters):
    L.rkmf_spmv_sketch(ctx.h, A.h, S.h, x.data_ptr(), z.data_ptr(), p.data_ptr())
dt = (time.perf_counter() - t0) / iters
nb = 12 * P.nnz + 4 * (P.n + 1) + 16 * P.n
print(f"{name} env={os.environ.get('RKMF_PIPE_DEBUG','0')}/{os.environ.get('RKMF_PIPE_STAGES','auto')}"
      f"/{os.environ.get('RKMF_SPMV_PIPE','1')}: {dt*1e6:.1f} us/call (incl. sync) "
      f"{nb/dt/1e9:.0f} GB/s alg")
