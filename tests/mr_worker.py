"""One rank of a row-partitioned restarted_krylov solve (launched by
tests/test_multirank_gpu.py under torch.distributed.run). All ranks share
cuda:0 and talk through the engine's host transport over gloo, so the
multi-rank code path (partitioned matrix and sketch, halo exchange, sketch
allreduce, replicated Gram-Schmidt, distributed norms) runs on one GPU with no
kernel ever waiting on another rank.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tests/mr_worker.py OUT.npz cfg2 24 [transport]
"""
import os
import sys
from datetime import timedelta

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out, name, N = sys.argv[1], sys.argv[2], int(sys.argv[3])
    transport = sys.argv[4] if len(sys.argv) > 4 else "host"
    classical = len(sys.argv) > 5 and sys.argv[5] == "classical"
    dist.init_process_group("gloo", timeout=timedelta(seconds=300))
    rank, world = dist.get_rank(), dist.get_world_size()
    import paper_2503_22631_b200 as rk
    from paper_2503_22631_b200 import configs
    from paper_2503_22631_b200 import distributed as D
    P = configs.build(name, N)
    ctx = D.make_context(0, world, rank, transport)
    part = D.partition(ctx, P.row_ptr, P.col_idx, P.values, P.b, P.d, P.zeta,
                       configs.SKETCH_SEED, world, rank)
    f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    r = rk.restarted_krylov(part.A, part.b, f, opts, None) if classical else D.solve(part, f, opts)
    fg = D.gather_f(r.f_hat, part.row_starts)
    # the partitioned sketch is the global sketch's column range (bit-exact)
    rows, signs, _ = part.S.export()
    srows = [None] * world
    dist.all_gather_object(srows, (part.row_begin, rows, signs))
    norm1 = part.A.norm1
    nd = [None] * world  # diagonal copy on every rank (halo diagonals included)
    dist.all_gather_object(nd, part.A.ndiag)
    if rank == 0:
        rr = np.concatenate([x[1] for x in sorted(srows, key=lambda t: t[0])])
        ss = np.concatenate([x[2] for x in sorted(srows, key=lambda t: t[0])])
        np.savez(out, f=fg, cycles=r.cycles, converged=r.converged, total_m=r.total_m,
                 updates=np.array([h.update_norm for h in r.history]),
                 matvecs=r.counters["matvecs"], norm1=norm1, row_starts=part.row_starts,
                 sketch_rows=rr, sketch_signs=ss, ndiag=np.array(nd))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
