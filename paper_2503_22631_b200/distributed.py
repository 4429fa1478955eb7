"""Row-partitioned (multi-rank) solve: one process per GPU.

The reference is single-process; this is the B200 build's domain
decomposition. Rank r owns the contiguous, nnz-balanced rows
[row_starts[r], row_starts[r+1]) of A, of b, of every basis vector and of
f_hat; its sketch is the same column range of the global make_sketch(d, n, zeta,
seed). The engine exchanges halo values and sums the d sketch partials every
Krylov step, and replicates the sketch-space Gram-Schmidt on every rank.

Two transports:
  * "nccl": one NCCL communicator per context (the product path on an
    NVLink/NVSwitch box; the unique id is broadcast over torch.distributed).
  * "host": the engine stages the same collectives through pinned host memory
    into callbacks served by torch.distributed (gloo). It runs where fewer GPUs
    than ranks exist (the ranks never wait on each other inside a kernel), and
    it is how an MPI/gloo host stack would drive the solver.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (Context, FunctionSpec, RestartOptions, RestartResult, SketchOperator, SparseMatrix,
               init_comm, init_host_comm, local_rows, nccl_unique_id, partition_rows,
               partitioned_matrix, partitioned_sketch, restarted_krylov)


def gloo_allreduce(buf: np.ndarray, op: str) -> None:
    """In-place allreduce of a host float64 array over torch.distributed."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(buf)
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)


def gloo_alltoallv(send: np.ndarray, send_counts, recv: np.ndarray, recv_counts) -> None:
    """Personalised exchange of 8-byte elements (segments in rank order) with
    point-to-point isend/irecv, which gloo supports."""
    import torch
    import torch.distributed as dist
    me, P = dist.get_rank(), dist.get_world_size()
    sc = np.asarray(send_counts, np.int64)
    rc = np.asarray(recv_counts, np.int64)
    so = np.concatenate([[0], np.cumsum(sc)]) * 8
    ro = np.concatenate([[0], np.cumsum(rc)]) * 8
    st = torch.from_numpy(send.view(np.uint8))
    rt = torch.from_numpy(recv.view(np.uint8))
    reqs = []
    for q in range(P):
        if q == me:
            continue
        if rc[q] > 0:
            reqs.append(dist.irecv(rt[ro[q]:ro[q + 1]], src=q))
        if sc[q] > 0:
            reqs.append(dist.isend(st[so[q]:so[q + 1]].clone(), dst=q))
    for r in reqs:
        r.wait()


def make_context(device: int, nranks: int, rank: int, transport: str) -> Context:
    """A context with a communicator over the current torch.distributed group."""
    ctx = Context(device)
    if nranks == 1:
        return ctx
    if transport == "nccl":
        import torch
        import torch.distributed as dist
        uid = nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(np.frombuffer(uid, np.uint8).copy())
        if dist.get_backend() == "nccl":  # a pure-NCCL group moves CUDA tensors only
            t = t.cuda(device)
        dist.broadcast(t, src=0)
        init_comm(ctx, nranks, rank, bytes(t.cpu().numpy().tobytes()))
    elif transport == "host":
        init_host_comm(ctx, nranks, rank, gloo_allreduce, gloo_alltoallv)
    else:
        raise ValueError(f"unknown transport {transport!r}")
    return ctx


@dataclass
class RankPart:
    ctx: Context
    row_starts: np.ndarray
    row_begin: int
    n_local: int
    A: SparseMatrix
    S: SketchOperator
    b: np.ndarray  # local slice (host)


def partition(ctx: Context, row_ptr, col_idx, values, b, d: int, zeta: int, seed: int,
              nranks: int, rank: int, row_starts=None) -> RankPart:
    """This rank's share of A (global CSR on the host), b and S."""
    n = len(row_ptr) - 1
    rs = partition_rows(row_ptr, nranks) if row_starts is None else np.asarray(row_starts,
                                                                               np.int64)
    rp, cg, v = local_rows(row_ptr, col_idx, values, rs, rank)
    A = partitioned_matrix(ctx, n, rs, rp, cg, v)
    rb, re = int(rs[rank]), int(rs[rank + 1])
    S = partitioned_sketch(ctx, d, n, zeta, seed, rb, re - rb)
    return RankPart(ctx=ctx, row_starts=rs, row_begin=rb, n_local=re - rb, A=A, S=S,
                    b=np.ascontiguousarray(b[rb:re]))


def partition_local(ctx: Context, n_global: int, row_starts, row_ptr_local, col_global,
                    values_local, b_local, d: int, zeta: int, seed: int, rank: int) -> RankPart:
    """This rank's objects from rows generated locally (global column ids)."""
    rs = np.asarray(row_starts, np.int64)
    A = partitioned_matrix(ctx, n_global, rs, row_ptr_local, col_global, values_local)
    rb, re = int(rs[rank]), int(rs[rank + 1])
    S = partitioned_sketch(ctx, d, n_global, zeta, seed, rb, re - rb)
    return RankPart(ctx=ctx, row_starts=rs, row_begin=rb, n_local=re - rb, A=A, S=S,
                    b=np.ascontiguousarray(b_local, np.float64))


def solve(part: RankPart, f: FunctionSpec, opts: RestartOptions, b_local=None,
          reference_local=None) -> RestartResult:
    """restarted_krylov on this rank's rows; f_hat is the rank's slice."""
    b = part.b if b_local is None else b_local
    return restarted_krylov(part.A, b, f, opts, part.S, reference=reference_local)


def gather_f(f_local: np.ndarray, row_starts) -> np.ndarray:
    """Assemble the global f_hat on every rank (host, torch.distributed)."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size()
    rs = np.asarray(row_starts, np.int64)
    width = int(np.max(np.diff(rs)))
    buf = torch.zeros(width, dtype=torch.float64)
    buf[:len(f_local)] = torch.from_numpy(np.asarray(f_local, np.float64))
    out = [torch.zeros(width, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(out, buf)
    return np.concatenate([out[q].numpy()[:rs[q + 1] - rs[q]] for q in range(P)])
