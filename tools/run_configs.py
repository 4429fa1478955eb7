"""Full-size device solves of BASELINE configs with the per-cycle record, for
DESIGN.md's table (and to check every config runs at its real size).

    python tools/run_configs.py cfg1 cfg3 cfg4
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg3", "cfg4"]:
    t0 = time.perf_counter()
    P = configs.build(name)
    t1 = time.perf_counter()
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    b = torch.tensor(P.b, device="cuda")
    r = rk.restarted_krylov(A, b, f, opts, S)
    r = rk.restarted_krylov(A, b, f, opts, S)
    print(f"{name}: n={P.n} nnz={P.nnz} gen={t1-t0:.1f}s upload+sketch={t2-t1:.2f}s "
          f"cycles={r.cycles} total_m={r.total_m} converged={r.converged} "
          f"solve_ms={r.solve_ms:.2f} vec/s={r.total_m/r.solve_ms*1e3:.0f} "
          f"funm_ms={[round(h.funm_ms, 2) for h in r.history][:8]} "
          f"upd={[f'{h.update_norm:.1e}' for h in r.history][:12]}", flush=True)
    del A, S, b
    torch.cuda.empty_cache()
