"""cfg3 (InvSqrt on the lognormal Q1 matrix, 200^3 nodes) at its BASELINE sketch
size d = 4m and larger (d = 0: the classical builder): does the restarted sketched FOM keep its Ritz values
off the branch cut (-inf, 0], and how many cycles does it need?

    python tools/cfg3_sketch_size.py [N] [d ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

args = [int(a) for a in sys.argv[1:]]
N = args[0] if args else 200
ds = args[1:] or [160, 320, 640]
P = configs.build_device("cfg3", N)
f = rk.FunctionSpec.inv_sqrt()
for d in ds:
    # d = 0: the classical builder (S == nullptr, orthonormal basis)
    S = rk.make_sketch(d, P.n, P.zeta, configs.SKETCH_SEED, P.A.ctx) if d else None
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=1000, budget_total_m=40000)
    try:
        r = rk.restarted_krylov(P.A, P.b, f, opts, S)
        un = [h.update_norm for h in r.history]
        print(f"N={N} m={P.m} d={d}: converged={r.converged} cycles={r.cycles} "
              f"solve_ms={r.solve_ms:.0f} nodes={getattr(r, 'quad_nodes', '?')} "
              f"last updates={[f'{u:.3g}' for u in un[-3:]]}", flush=True)
    except rk.NumericalError as e:
        print(f"N={N} m={P.m} d={d}: NumericalError: {e}", flush=True)
