"""Regenerate tests/golden/*.npz from the CPU oracle (run from the repo root).

The reference ships no golden vectors for this path: its
sketch is pinned only by determinism (test_sketch.cpp:55-62) and every solver
check is an identity or a tolerance. These fixtures freeze the oracle's
restatement so that (1) the independent pure-Python SplitMix64/make_sketch
restatement in tests/helpers.py, (2) the oracle and (3) the device path can be
checked against the same bytes. Inputs are the product generators (same CSR on
both sides).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    # SplitMix64 streams and derived seeds (rng.hpp:21-26, 56-59)
    np.savez_compressed(os.path.join(OUT, "splitmix.npz"),
                        stream_0=O.splitmix_stream(0, 64), stream_42=O.splitmix_stream(42, 64),
                        derive=np.array([O.splitmix_derive(s, t) for s in (0, 1, 77)
                                         for t in (0, 1, 2, 1000, 2**40)], np.uint64),
                        gauss_1=O.gaussian_vector(1, 257))
    # sketches (sketch.cpp:13-49) at the shapes the reference tests use and at
    # the BASELINE d/zeta
    sk = {}
    for (d, n, z, s) in [(40, 300, 5, 123), (24, 24, 24, 9), (60, 500, 4, 77), (30, 200, 1, 5),
                         (120, 4096, 8, 1), (200, 2000, 8, 1), (160, 1000, 8, 3)]:
        S = O.make_sketch(d, n, z, s)
        key = f"d{d}_n{n}_z{z}_s{s}"
        sk[key + "_rows"] = S.rows.astype(np.int16)
        sk[key + "_signs"] = S.signs
    np.savez_compressed(os.path.join(OUT, "sketch.npz"), **sk)
    # restart histories on scaled-down configs
    hist = {}
    for name, N in [("cfg1", 32), ("cfg2", 12), ("cfg4", 10)]:
        P = configs.build(name, N)
        S = O.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED)
        r = O.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, O.KIND_EXP_NEG, P.t,
                               m_r=P.m, tol=P.tol, k_max=P.k_max, S=S)
        hist[f"{name}_N{N}_f"] = r.f_hat
        hist[f"{name}_N{N}_update_norm"] = np.array([h["update_norm"] for h in r.history])
        hist[f"{name}_N{N}_start_norm"] = np.array([h["start_norm"] for h in r.history])
        hist[f"{name}_N{N}_meta"] = np.array([r.cycles, r.total_m, int(r.converged)], np.int64)
        hist[f"{name}_N{N}_t"] = np.array([P.t])
    np.savez_compressed(os.path.join(OUT, "restart.npz"), **hist)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
