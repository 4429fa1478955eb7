"""K2 alone (back-to-back launches, CUDA events) and the whole solve on a
device-generated BASELINE config, for A/B runs of library variants
(RKMF_LIB_PATH) without the host generators.

    python tools/kbench.py [cfg4] [reps] [--solve] [--label NAME]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "cfg4"
reps = int(args[1]) if len(args) > 1 else 50
label = os.path.basename(os.environ.get("RKMF_LIB_PATH", "main"))
if "--label" in sys.argv:
    label = sys.argv[sys.argv.index("--label") + 1]
P = configs.build_device(name)
A = P.A
if os.environ.get("RKMF_FUSED") == "0":  # per-step kernels even for small matrices
    A.ctx.set_fused_cycle(False)
    label += "+steps"
if "--csrdict" in sys.argv:  # the CSR row dictionary instead of the diagonal copy
    A.set_diagonal_copy(False)
    label += f"+csrdict({A.set_row_dictionary(True)})"
S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED, A.ctx)
x = P.b.clone()
rk.kernel_bench(A, S, x, 1, 5)
ms = min(rk.kernel_bench(A, S, x, 1, reps) for _ in range(3))
line = f"{name} [{label}] K2 {ms * 1e3:.1f} us"
if "--solve" in sys.argv:
    f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    rk.restarted_krylov(A, P.b, f, opts, S)
    best = min(rk.restarted_krylov(A, P.b, f, opts, S).solve_ms for _ in range(3))
    r = rk.restarted_krylov(A, P.b, f, opts, S)
    line += f"; solve {best:.2f} ms ({r.total_m / best * 1e3:.0f} vec/s, {r.cycles} cycles)"
    A.ctx.kernel_timing(True)
    A.ctx.kernel_times(reset=True)
    rk.restarted_krylov(A, P.b, f, opts, S)
    kt = A.ctx.kernel_times(reset=True)
    A.ctx.kernel_timing(False)
    line += " [" + ", ".join(f"{c} {t:.2f}/{n}" for c, (t, n) in kt.items() if n) + "]"
print(line, flush=True)
