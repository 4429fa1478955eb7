"""Device path vs the reference's own sources: the measured differences behind
tests/test_gpu_ref.py and tests/test_gpu_fullsize.py (run on the GPU box).

    python tools/ref_report.py > profiles/<tag>_ref_report.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def solve(P, diagnostics=True):
    A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
    S = rk.make_sketch(P.d, P.n, P.zeta, 1)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max, diagnostics=diagnostics)
    return rk.restarted_krylov(A, torch.tensor(P.b, device="cuda"), rk.FunctionSpec.exp_neg(P.t),
                               opts, S, keep_R_accum=True)


print("# device f_hat vs the reference's own sources (oracle/_ref), relative 2-norm")
print("config                 rows   cycles dev/ref   rel err f_hat   max|R_accum diff|/max|R|"
      "   max rel kappa_W diff")
if R.available():
    Rf = R.front()
    for name, N in (("cfg1", None), ("cfg2", 44), ("cfg4", 40), ("cfg5", 24)):
        P = configs.build(name) if N is None else configs.build(name, N)
        S = Rf.make_sketch(P.d, P.n, P.zeta, 1)
        q = Rf.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, 0, P.t, m_r=P.m, tol=P.tol,
                                k_max=P.k_max, S=S, want_R=True)
        r = solve(P)
        dk = max(abs(h.kappa_W - g["kappa_W"]) / g["kappa_W"] for h, g in zip(r.history, q.history))
        print(f"{name + (' full size' if N is None else f' N={N}'):20s} {P.n:8d}   {r.cycles}/{q.cycles}"
              f"            {rel(r.f_hat.cpu().numpy(), q.f_hat):.2e}        "
              f"{np.abs(np.asarray(r.R_accum) - q.R_accum).max() / np.abs(q.R_accum).max():.2e}"
              f"                   {dk:.2e}")
g = np.load(os.path.join(ROOT, "tests", "golden", "ref_fullsize.npz"))
print("\n# full BASELINE size, against the digest frozen from the reference's sources")
print("config      rows   cycles dev/ref   rel err at 8192 sample rows   rel err of S f_hat (d=256)"
      "   | ||f|| rel diff")
for name in ("cfg2", "cfg4"):
    P = configs.build(name)
    r = solve(P)
    f = r.f_hat.cpu().numpy()
    rows = np.sort(np.random.default_rng(2503).choice(P.n, 8192, replace=False))
    D = O.make_sketch(256, P.n, 8, 2503)
    print(f"{name:8s} {P.n:9d}   {r.cycles}/{int(g[f'{name}/meta'][1])}            "
          f"{rel(f[rows], g[f'{name}/f_samples']):.2e}                      "
          f"{rel(O.sketch_apply(D, f), g[f'{name}/f_digest']):.2e}                    "
          f"{abs(np.linalg.norm(f) - g[f'{name}/f_norm'][0]) / g[f'{name}/f_norm'][0]:.2e}")
