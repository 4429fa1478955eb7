"""Microbenchmark of the sketch-only kernel (rkmf_sketch_apply) on a BASELINE size."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
P = configs.build(name, with_b=True)
S = rk.make_sketch(P.d, P.n, P.zeta, 1)
x = torch.tensor(P.b, device="cuda")
p = torch.empty(P.d, dtype=torch.float64, device="cuda")
L = rk.lib()
ctx = S.ctx
for _ in range(5):
    L.rkmf_sketch_apply(ctx.h, S.h, x.data_ptr(), p.data_ptr())
t0 = time.perf_counter()
for _ in range(iters):
    L.rkmf_sketch_apply(ctx.h, S.h, x.data_ptr(), p.data_ptr())
dt = (time.perf_counter() - t0) / iters
nb = 8 * P.n + P.n * P.zeta + 2 * (P.d + 8) * ((P.n + 127) // 128)
print(f"{name} sketch_apply: {dt*1e6:.1f} us/call (incl. sync) {nb/dt/1e9:.0f} GB/s (z + metadata)")
