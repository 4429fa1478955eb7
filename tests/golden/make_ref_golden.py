"""Freeze outputs of the REFERENCE'S OWN sources as tests/golden/ref_pin.npz.

Run in the build container (where /root/reference is mounted) from the repo
root, after `make -C oracle ref`:

    python tests/golden/make_ref_golden.py

`oracle/_ref/librkmf_ref.so` is the reference's restart.cpp, basis.cpp,
sketch.cpp, sparse.cpp, densefun.cpp, approximants.cpp and leastsq.cpp compiled
unmodified against the Eigen-API stand-in (oracle/eigen_standin; Eigen is
absent from the image). The fixture holds, per case of tests/ref_cases.py:
the sketch, S b, one randomized-Arnoldi decomposition (U, Rbar, the last basis
vector), restarted_krylov with the randomized and the classical builder
(f_hat, R_accum, per-cycle update norms, kappa_W, leftmost Ritz value,
counters), and funm. tests/test_ref_pin.py holds the oracle to these bytes
(bit for bit in its contraction-free build), so the pin survives where the
library and /root/reference are absent.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402
from tests import ref_cases  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    assert R.build() and R.available(), "oracle/_ref is not built (needs /root/reference)"
    g = {}
    for name in ref_cases.CASES:
        P = ref_cases.build(name, O)
        S = R.make_sketch(P["d"], P["n"], P["zeta"], P["seed"])
        g[f"{name}/sketch_rows"] = S.rows.astype(np.int16)
        g[f"{name}/sketch_signs"] = S.signs
        g[f"{name}/Sb"] = R.sketch_apply(S, P["b"])
        g[f"{name}/Ab"] = R.spmv(P["A"], P["b"])
        g[f"{name}/norm1"] = np.array([R.norm1(P["A"])])
        dec = R.arnoldi_decomp(P["A"], P["b"], P["m"], S)
        g[f"{name}/dec_U"] = dec.U
        g[f"{name}/dec_Rbar"] = dec.Rbar
        g[f"{name}/dec_w_last"] = dec.W[:, -1].copy()
        g[f"{name}/dec_start_norm"] = np.array([dec.start_norm])
        g[f"{name}/dec_counters"] = np.array(list(dec.counters.values()), np.int64)
        for tag, Sk in (("rand", S), ("classical", None)):
            r = R.restarted_krylov(P["A"], P["b"], O.KIND_EXP_NEG, P["t"], m_r=P["m"],
                                   tol=P["tol"], k_max=P["k_max"], S=Sk, want_R=True)
            g[f"{name}/{tag}_f"] = r.f_hat
            g[f"{name}/{tag}_R_accum"] = r.R_accum
            g[f"{name}/{tag}_update_norm"] = np.array([h["update_norm"] for h in r.history])
            g[f"{name}/{tag}_kappa_W"] = np.array([h["kappa_W"] for h in r.history])
            g[f"{name}/{tag}_ritz_left"] = np.array([h["leftmost_ritz_re"] for h in r.history])
            g[f"{name}/{tag}_alpha_dev"] = np.array([h["alpha_dev"] for h in r.history])
            g[f"{name}/{tag}_meta"] = np.array([r.cycles, r.total_m, int(r.converged)], np.int64)
            g[f"{name}/{tag}_alpha"] = np.array([r.alpha])
            g[f"{name}/{tag}_counters"] = np.array(list(r.counters.values()), np.int64)
    X = ref_cases.dense_f_input()
    g["funm/X"] = X
    for t in (0.05, 0.7, 3.0):
        g[f"funm/F_t{t}"] = R.funm(X, O.KIND_EXP_NEG, t)
    g["rng/below_1000"] = R.splitmix_below(99, 1000, 256)
    g["rng/below_big"] = R.splitmix_below(7, (1 << 63) + 12345, 64)
    np.savez_compressed(os.path.join(OUT, "ref_pin.npz"), **g)
    print("wrote ref_pin.npz:", len(g), "arrays,", os.path.getsize(os.path.join(OUT, "ref_pin.npz")), "bytes")


if __name__ == "__main__":
    main()
