"""Freeze the REFERENCE'S OWN sources on BASELINE configs at full size.

    python tests/golden/make_ref_fullsize.py [cfg2 cfg4]

Runs restart::restarted_krylov of oracle/_ref (the reference's sources compiled
against the Eigen-API stand-in; single-threaded, minutes per config) on the
full-size BASELINE config and stores a compact digest in
tests/golden/ref_fullsize.npz, because f_hat itself (2.1M / 16.8M doubles)
is too large to commit: f_hat at 8,192 seeded sample rows, ||f_hat||_2, the
sparse-sign sketch S f_hat (d = 256, zeta = 8, seed 2503, through the
reference's own sketch_apply: every row of f_hat enters eight of its
entries), R_accum, the per-cycle update norms, kappa_W, leftmost Ritz values
and the counters. tests/test_gpu_fullsize.py holds the device solve to it.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_fullsize.npz")
DIGEST_D, DIGEST_ZETA, DIGEST_SEED, SAMPLES = 256, 8, 2503, 8192


def sample_rows(n):
    return np.sort(np.random.default_rng(DIGEST_SEED).choice(n, SAMPLES, replace=False))


def main():
    names = sys.argv[1:] or ["cfg2", "cfg4"]
    g = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    Rf = R.front()
    for name in names:
        P = configs.build(name)
        S = Rf.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
        t0 = time.time()
        r = Rf.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, 0, P.t, m_r=P.m, tol=P.tol,
                                k_max=P.k_max, S=S, want_R=True)
        print(f"{name}: n={P.n} cycles={r.cycles} converged={r.converged} "
              f"{time.time() - t0:.0f} s", flush=True)
        D = Rf.make_sketch(DIGEST_D, P.n, DIGEST_ZETA, DIGEST_SEED)
        g[f"{name}/meta"] = np.array([P.n, r.cycles, r.total_m, int(r.converged)], np.int64)
        g[f"{name}/f_samples"] = r.f_hat[sample_rows(P.n)]
        g[f"{name}/f_norm"] = np.array([np.linalg.norm(r.f_hat)])
        g[f"{name}/f_digest"] = Rf.sketch_apply(D, r.f_hat)
        g[f"{name}/R_accum"] = r.R_accum
        g[f"{name}/alpha"] = np.array([r.alpha])
        g[f"{name}/update_norm"] = np.array([h["update_norm"] for h in r.history])
        g[f"{name}/kappa_W"] = np.array([h["kappa_W"] for h in r.history])
        g[f"{name}/ritz_left"] = np.array([h["leftmost_ritz_re"] for h in r.history])
        g[f"{name}/counters"] = np.array(list(r.counters.values()), np.int64)
        np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
