"""Microbenchmark of the step kernels alone (rkmf_kernel_bench: CUDA events
around back-to-back launches on the context stream).

    RKMF_PIPE_DEBUG=1 python tools/bench_spmv.py [cfg2] [reps]
Algorithmic bytes: SpMV 12 nnz + 4 (n+1) + 8n x + 8n z;
sketch metadata excluded.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
P = configs.build(name)
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, 1)
x = torch.tensor(P.b, device="cuda")
rp = 8 if P.nnz >= 2**31 else 4
nb = 12 * P.nnz + rp * (P.n + 1) + 16 * P.n
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("RKMF_"))
out = []
for mode, label in ((1, "spmv+sketch"), (0, "spmv"), (2, "sketch-only")):
    ms = rk.kernel_bench(A, S, x, mode, reps)
    gbs = (nb if mode < 2 else 8 * P.n) / ms / 1e6
    out.append(f"{label} {ms*1e3:.1f} us ({gbs:.0f} GB/s alg)")
print(f"[{env or 'default'}] {name}: " + "; ".join(out))
