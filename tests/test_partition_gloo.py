"""Host logic of the row-partitioned (multi-GPU) path, on the CPU.

* partition_rows / partition_halo (partition.cpp) on the BASELINE stencils and
  on irregular matrices;
* one Krylov step's communication pattern over a real 2- and 3-rank gloo group,
  driven by the same callbacks the engine's host transport calls
  (distributed.gloo_allreduce / gloo_alltoallv): the halo-request exchange that
  builds the send lists (comm.cu step 2), the per-step halo exchange, the local
  SpMV over [owned | halo] columns, the sketch-partial allreduce and the
  norm1 column-sum return path. Local arithmetic uses the CPU oracle, and the
  result must equal the oracle's global SpMV / sketch / norm1.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _csr(name, N):
    from paper_2503_22631_b200 import configs
    P = configs.build(name, N)
    return P


@pytest.mark.parametrize("name,N", [("cfg1", 40), ("cfg2", 12), ("cfg3", 7), ("cfg4", 10)])
@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_partition_rows_and_halo(rk, name, N, P):
    prob = _csr(name, N)
    rp, ci = prob.row_ptr, prob.col_idx
    rs = rk.partition_rows(rp, P)
    n = prob.n
    assert rs[0] == 0 and rs[-1] == n and np.all(np.diff(rs) >= 0)
    nnz = rp[-1]
    maxrow = int(np.max(np.diff(rp)))
    for r in range(1, P):  # boundary r: first row whose nnz prefix reaches floor(r nnz / P)
        target = nnz * r // P
        assert rp[rs[r]] >= target
        assert rs[r] == 0 or rp[rs[r] - 1] < target
    per = np.diff(rp[rs])
    assert per.max() - per.min() <= 2 * maxrow + 1
    for q in range(P):
        lrp, lcg, _ = rk.local_rows(rp, ci, prob.values, rs, q)
        halo, rc, cl = rk.partition_halo(rs, q, lrp, lcg)
        rb, re = rs[q], rs[q + 1]
        off = (lcg < rb) | (lcg >= re)
        assert np.array_equal(halo, np.unique(lcg[off]))
        assert rc.sum() == len(halo) and rc[q] == 0
        owners = np.searchsorted(rs, halo, side="right") - 1
        assert np.array_equal(np.bincount(owners, minlength=P), rc)
        ext = np.concatenate([np.arange(rb, re), halo])  # local column -> global column
        assert np.array_equal(ext[cl], lcg)


def test_partition_irregular(rk):
    from tests.helpers import random_sparse
    A = random_sparse(300, 0.05, 3)
    A.indices = A.indices.astype(np.int32)
    for P in (2, 4, 7):
        rs = rk.partition_rows(A.indptr.astype(np.int64), P)
        assert rs[-1] == 300
        for q in range(P):
            lrp, lcg, _ = rk.local_rows(A.indptr.astype(np.int64), A.indices, A.data, rs, q)
            halo, rc, cl = rk.partition_halo(rs, q, lrp, lcg)
            ext = np.concatenate([np.arange(rs[q], rs[q + 1]), halo])
            assert np.array_equal(ext[cl], lcg)


def _rank_main(rank, world, port, name, N, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from datetime import timedelta
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=timedelta(seconds=120))
    try:
        import paper_2503_22631_b200 as rk
        from oracle import oracle as O
        from paper_2503_22631_b200 import configs
        from paper_2503_22631_b200.distributed import gloo_allreduce, gloo_alltoallv
        prob = configs.build(name, N)
        rs = rk.partition_rows(prob.row_ptr, world)
        rb, re = int(rs[rank]), int(rs[rank + 1])
        nl = re - rb
        lrp, lcg, lv = rk.local_rows(prob.row_ptr, prob.col_idx, prob.values, rs, rank)
        halo, rcnt, cl = rk.partition_halo(rs, rank, lrp, lcg)

        def exchange(segs, rcounts, dtype):
            """segs[q] goes to rank q; returns what each rank sent here (the
            callback's contract: contiguous segments in rank order)."""
            sc = np.array([0 if q == rank else len(segs[q]) for q in range(world)], np.int64)
            rc = np.array([0 if q == rank else rcounts[q] for q in range(world)], np.int64)
            send = np.concatenate([np.asarray(segs[q], dtype) for q in range(world) if q != rank]
                                  + [np.zeros(0, dtype)])
            recv = np.zeros(max(int(rc.sum()), 1), dtype)
            gloo_alltoallv(send.view(np.int8), sc, recv.view(np.int8), rc)
            o = np.concatenate([[0], np.cumsum(rc)])
            return [recv[o[q]:o[q + 1]] for q in range(world)]

        # requests -> owners: how many each rank needs from me, then which
        roff = np.concatenate([[0], np.cumsum(rcnt)])
        got = exchange([[rcnt[q]] for q in range(world)], [1] * world, np.int64)
        scnt = np.array([0 if q == rank else int(got[q][0]) for q in range(world)], np.int64)
        reqs = exchange([halo[roff[q]:roff[q + 1]] for q in range(world)], scnt, np.int64)
        want = np.concatenate(reqs)
        assert np.all((want >= rb) & (want < re))
        send_idx = want - rb
        soff = np.concatenate([[0], np.cumsum(scnt)])
        # one step: halo exchange of x, local SpMV on [owned | halo], sketch partial
        x = O.gaussian_vector(5, prob.n)
        xl = x[rb:re].copy()
        hv = exchange([xl[send_idx[soff[q]:soff[q + 1]]] for q in range(world)], rcnt,
                      np.float64)
        ext = np.concatenate([xl] + hv)
        import scipy.sparse as sp
        Al = sp.csr_matrix((lv, cl, lrp), shape=(nl, nl + len(halo)))
        zl = O.spmv(Al, ext)
        Sg = O.make_sketch(prob.d, prob.n, prob.zeta, 1)
        Sl = O.Sketch(prob.d, nl, prob.zeta, 1, Sg.rows[rb * prob.zeta:re * prob.zeta].copy(),
                      Sg.signs[rb * prob.zeta:re * prob.zeta].copy(), Sg.scale)
        p = O.sketch_apply(Sl, zl)
        gloo_allreduce(p, "sum")
        # norm1: column sums, halo parts back to their owners, max
        cs = np.zeros(nl + len(halo))
        np.add.at(cs, cl, np.abs(lv))
        back = exchange([cs[nl + roff[q]:nl + roff[q + 1]] for q in range(world)], scnt,
                        np.float64)
        np.add.at(cs, send_idx, np.concatenate(back))
        mx = np.array([cs[:nl].max() if nl else 0.0])
        gloo_allreduce(mx, "max")
        zall = [None] * world
        dist.all_gather_object(zall, (rb, zl))
        if rank == 0:
            z = np.zeros(prob.n)
            for b0, zz in zall:
                z[b0:b0 + len(zz)] = zz
            np.savez(os.path.join(out_dir, "res.npz"), z=z, p=p, norm1=mx[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,N,world", [("cfg2", 10, 2), ("cfg4", 9, 3), ("cfg1", 30, 2)])
def test_gloo_step_matches_global(tmp_path, oracle, name, N, world):
    import torch.multiprocessing as mp
    from paper_2503_22631_b200 import configs
    mp.spawn(_rank_main, args=(world, _free_port(), name, N, str(tmp_path)), nprocs=world,
             join=True)
    r = np.load(tmp_path / "res.npz")
    prob = configs.build(name, N)
    A = (prob.row_ptr, prob.col_idx, prob.values)
    x = oracle.gaussian_vector(5, prob.n)
    z = oracle.spmv(A, x)
    S = oracle.make_sketch(prob.d, prob.n, prob.zeta, 1)
    assert np.linalg.norm(r["z"] - z) <= 1e-14 * np.linalg.norm(z)
    p = oracle.sketch_apply(S, z)
    assert np.linalg.norm(r["p"] - p) <= 1e-13 * np.linalg.norm(p)
    assert float(r["norm1"]) == pytest.approx(oracle.norm1(A), rel=1e-14)
