"""Device timeline of the per-step kernels inside one solve (globaltimer stamps).

    python tools/trace_steps.py [cfg2] [reps]

Arms rkmf_debug_trace, runs one device-resident solve, and prints per step
the phases (microseconds) of K2 (fused SpMV + sketch), K3 (sketched
Gram-Schmidt) and K4 (basis update), from the stamps of the last cycle.
The stamps are compiled only into the trace build of the library
(`make -C paper_2503_22631_b200/csrc trace`), which this script selects; use
it for the breakdown, not for the bench number.
"""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

os.environ.setdefault("RKMF_LIB_PATH", os.path.join(
    ROOT, "paper_2503_22631_b200", "_lib", "librkmf_b200_trace.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

SLOTS = 16
NAMES = {
    10: "K2 block 0 start", 0: "K2 block 0 past wait", 1: "K2 last sketch flush",
    2: "K3 start", 3: "K3 past wait", 4: "K3 p+U staged", 5: "K3 dots", 6: "K3 tri-solve",
    7: "K3 end", 11: "K4 block 0 start", 8: "K4 block 0 past wait", 9: "K4 last block end",
}

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
P = configs.build(name)
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
b = torch.tensor(P.b, device="cuda")
L = rk.lib()
L.rkmf_debug_trace.restype = C.c_int
L.rkmf_debug_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
for _ in range(reps):
    r = rk.restarted_krylov(A, b, f, opts, S)
torch.cuda.synchronize()
steps = P.m
opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=int(os.environ.get("TRACE_KMAX", P.k_max)))
assert L.rkmf_debug_trace(A.ctx.h, 1, None, steps) == 0
r = rk.restarted_krylov(A, b, f, opts, S)
out = np.zeros((steps, SLOTS), dtype=np.uint64)
assert L.rkmf_debug_trace(A.ctx.h, 0, out.ctypes.data, steps) == 0
print(f"{name}: cycles={r.cycles} solve_ms={r.solve_ms:.3f}")
t = out.astype(np.float64)
t[t == 0] = np.nan
order = [10, 0, 1, 2, 3, 4, 5, 6, 7, 11, 8, 9]
rows = []
for k in range(1, steps - 1):
    base = t[k, 0]
    rows.append([(t[k, s] - base) / 1e3 for s in order] + [(t[k + 1, 0] - base) / 1e3])
rows = np.array(rows)
print(f"{'stamp':28s} {'median us':>10s} {'min':>8s} {'max':>8s}   (relative to K2 block 0 past wait; last cycle)")
for j, s in enumerate(order):
    col = rows[:, j]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{NAMES[s]:28s} {np.median(col):10.2f} {col.min():8.2f} {col.max():8.2f}")
col = rows[:, -1]
col = col[~np.isnan(col)]
print(f"{'next K2 past wait':28s} {np.median(col):10.2f} {col.min():8.2f} {col.max():8.2f}")
