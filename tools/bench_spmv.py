"""Microbenchmark of the fused SpMV + sketch (K2) alone, per matrix stream
(rkmf_kernel_bench: CUDA events around back-to-back launches on the context
stream), plus the whole solve per stream.

    python tools/bench_spmv.py [cfg2] [reps] [--solve]

Streams: the diagonal copy with its row dictionary (one byte per row), the
diagonal copy (8 bytes per slot), the CSR arrays. Algorithmic bytes
(SURVEY.md §8(d)): SpMV 12 nnz + 4 (n+1) + 8n x + 8n z; sketch metadata
excluded. Streamed bytes: what each stream actually reads and writes.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_22631_b200 as rk  # noqa: E402
from paper_2503_22631_b200 import configs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "cfg2"
reps = int(args[1]) if len(args) > 1 else 100
solve = "--solve" in sys.argv
P = configs.build(name)
A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values)
S = rk.make_sketch(P.d, P.n, P.zeta, 1)
x = torch.tensor(P.b, device="cuda")
rp = 8 if P.nnz >= 2**31 else 4
nb = 12 * P.nnz + rp * (P.n + 1) + 16 * P.n
tiles = (P.n + 127) // 128
sk = tiles * sum(S.layout_bytes_per_tile())  # sketch tile layout
nd, nt = A.ndiag, A.ntuples
streams = []
if nt:
    streams.append(("dict", 16 * P.n + tiles * 128 + sk))
if nd:
    streams.append(("dia", 16 * P.n + tiles * 128 * 8 * nd + sk))
streams.append(("csr", nb + sk))
b = torch.tensor(P.b, device="cuda")
f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
for label, sb in streams:
    if label == "dia":
        A.set_row_dictionary(False)
    if label == "csr":
        A.set_diagonal_copy(False)
    ms = rk.kernel_bench(A, S, x, 1, reps)
    line = (f"{name} K2 [{label}] {ms * 1e3:.1f} us: {nb / ms / 1e6:.0f} GB/s alg, "
            f"{sb / ms / 1e6:.0f} GB/s streamed ({sb / 1e6:.1f} MB)")
    if solve:
        rk.restarted_krylov(A, b, f, opts, S)
        best = min(rk.restarted_krylov(A, b, f, opts, S).solve_ms for _ in range(3))
        r = rk.restarted_krylov(A, b, f, opts, S)
        line += f"; solve {best:.2f} ms ({r.total_m / best * 1e3:.0f} vec/s, {r.cycles} cycles)"
        A.ctx.kernel_timing(True)
        A.ctx.kernel_times(reset=True)
        rk.restarted_krylov(A, b, f, opts, S)
        kt = A.ctx.kernel_times(reset=True)
        A.ctx.kernel_timing(False)
        line += " [" + ", ".join(f"{c} {ms:.2f}/{n}" for c, (ms, n) in kt.items() if n) + "]"
    print(line, flush=True)
print(f"{name}: ndiag={nd} ntuples={nt} n={P.n}")
