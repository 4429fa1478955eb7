"""One rank of the cfg5-kind partitioned solve with the Q1 rows generated in
HBM (rkmf_matrix_gen_q1_hex_partitioned) beside the same rows built on the
host and uploaded through rkmf_matrix_create_partitioned (launched by
tests/test_multirank_gpu.py; ranks share cuda:0 over the host transport).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tests/mr_q1_worker.py OUT.npz N
"""
import os
import sys
from datetime import timedelta

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out, N = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo", timeout=timedelta(seconds=300))
    rank, world = dist.get_rank(), dist.get_world_size()
    import paper_2503_22631_b200 as rk
    from paper_2503_22631_b200 import configs
    from paper_2503_22631_b200 import distributed as D
    P = configs.build("cfg5", N)
    ctx = D.make_context(0, world, rank, "host")
    plane = N * N
    rs = np.array([plane * (N * q // world) for q in range(world + 1)], np.int64)
    host = D.partition(ctx, P.row_ptr, P.col_idx, P.values, P.b, P.d, P.zeta,
                       configs.SKETCH_SEED, world, rank, row_starts=rs)
    Adev = rk.SparseMatrix.q1_hex_partitioned(ctx, N, rs, False, configs.COEF_SEED, False)
    same_csr = all(np.array_equal(a, b) for a, b in zip(Adev.export(), host.A.export()))
    rb, re = int(rs[rank]), int(rs[rank + 1])
    bdev = rk.gen_gaussian_device(configs.B_SEED, rb, re - rb, ctx)
    f = rk.FunctionSpec.exp_neg(P.t)
    opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    r_host = D.solve(host, f, opts)
    r_dev = rk.restarted_krylov(Adev, host.b, f, opts, host.S)
    same_f = bool(np.array_equal(r_dev.f_hat, r_host.f_hat))
    # the device N(0,1) draws go through CUDA's log/cos: equal to the host's
    # to an ulp or so
    bd = bdev.cpu().numpy()
    b_close = bool(np.abs(bd - host.b).max() <= 4e-16 * np.abs(host.b).max())
    flags = [None] * world
    dist.all_gather_object(flags, (same_csr, same_f, Adev.norm1 == host.A.norm1, b_close))
    fg = D.gather_f(r_dev.f_hat, rs)
    if rank == 0:
        np.savez(out, flags=np.array(flags), f=fg, cycles=r_dev.cycles,
                 converged=r_dev.converged, comm=str(ctx.comm_info()))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
