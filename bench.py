#!/usr/bin/env python
"""bench.py — restarted randomized-Arnoldi f(A)b on B200.

One "step" = one full restarted f(A)b solve of the workload (default BASELINE
configs[1] = cfg2: 3D 7-point Laplacian 128^3, exp(-tA)b, m=50, s=200, zeta=8,
tol 1e-8 relative) with A, S and b resident in HBM. The metric is Krylov basis
vectors per second (sum of m_k over cycles / solve time), whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg1..cfg5]

N > 1 (torchrun, one rank per GPU): one row-partitioned solve over all ranks
(weak scaling: each rank owns a cfg2-sized x-slab of a 128N x 128 x 128 grid;
halo send/recv + sketch allreduce over NCCL every Krylov step).
`--impl reference` times the CPU restatement of the reference solver (the
reference itself cannot be built here: Eigen3 is absent) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Krylov basis vectors/sec (restarted randomized-Arnoldi f(A)b)"
UNIT = "basis_vectors/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload_desc(P, name):
    return {"workload": f"{name}: BASELINE configs[{int(name[-1]) - 1}]", "matrix_rows": P.n,
            "nnz": P.nnz, "function": P.fn, "t": P.t, "m": P.m, "sketch_d": P.d,
            "zeta": P.zeta, "tol_abs": P.tol, "tol_rel": P.tol / float(sum(P.b * P.b)) ** 0.5,
            "k_max": P.k_max, "b_seed": 1, "sketch_seed": 1,
            "l2_policy": "inputs larger than L2 (CSR + basis W exceed 126 MB)"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def class_bytes(w, total_m, cycles):
    """Algorithmic bytes per solve (per rank) for each kernel class (SURVEY.md
    §8(d) terms)."""
    n, nnz, m = w.n, w.nnz, w.m
    rp = 4 if nnz < 2**31 - 1 else 8
    steps = total_m
    spmv = steps * (12 * nnz + rp * (n + 1) + 8 * n + 8 * n)
    upd = 0
    for _ in range(cycles):
        for k in range(m - 1):
            upd += 8 * n * (k + 1) + 8 * n + 8 * n
    final = cycles * (8 * n * m + 8 * n + 16 * n + 8 * n)
    start = (cycles + 1) * 8 * n
    return {"spmv_sketch": spmv, "basis_update": upd, "final_update": final,
            "start_sketch_init": start}


_ORACLE_SKETCH = {}


def cpu_baseline_sample(P, threads: int, cycles: int = 1, m_r: int | None = None):
    """Oracle port on the host: `cycles` full restart cycles of the workload."""
    from oracle import oracle as O
    key = (P.d, P.n, P.zeta)
    if key not in _ORACLE_SKETCH:
        _ORACLE_SKETCH[key] = O.make_sketch(P.d, P.n, P.zeta, 1)
    S = _ORACLE_SKETCH[key]
    kind = O.KIND_EXP_NEG if P.fn == "exp_neg" else O.KIND_INV_SQRT
    t0 = time.perf_counter()
    r = O.restarted_krylov((P.row_ptr, P.col_idx, P.values), P.b, kind, P.t, m_r=m_r or P.m,
                           tol=1e-300, k_max=cycles, S=S, threads=threads)
    dt = time.perf_counter() - t0
    return r.total_m / dt, dt, r


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from paper_2503_22631_b200 import configs
    P = configs.build(args.config)
    threads = os.cpu_count() or 1
    vals = []
    for _ in range(args.warmup):  # cache/page warm-up: short 5-vector cycles
        cpu_baseline_sample(P, threads, 1, m_r=5)
    for _ in range(args.steps):
        v, dt, r = cpu_baseline_sample(P, threads, 1)
        vals.append((r.total_m, dt))
    tot_m = sum(v[0] for v in vals)
    tot_t = sum(v[1] for v in vals)
    value = tot_m / tot_t
    sample = (f"one restart cycle (m={P.m} basis vectors, incl. per-cycle validate/norm1 and the "
              f"full dense f) of {args.config} per step, oracle port, {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / len(vals), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(P, args.config),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": "the reference (Eigen-based C++) is not buildable in this image; its CPU "
                    "path is the Eigen-free restatement in oracle/ (DESIGN.md)"}
    print(json.dumps(line), flush=True)
    return 0


class Workload:
    """What one rank solves: the device objects plus the sizes the byte model
    and the JSON line need."""


def setup_single(args, ctx, dev):
    import torch

    import paper_2503_22631_b200 as rk
    from paper_2503_22631_b200 import configs
    P = configs.build(args.config)
    w = Workload()
    w.P, w.n, w.nnz, w.m = P, P.n, P.nnz, P.m
    w.A = rk.SparseMatrix.from_csr(P.row_ptr, P.col_idx, P.values, ctx=ctx)
    w.S = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED, ctx=ctx)
    w.f = rk.FunctionSpec.exp_neg(P.t) if P.fn == "exp_neg" else rk.FunctionSpec.inv_sqrt()
    w.opts = rk.RestartOptions(m_r=P.m, tol=P.tol, k_max=P.k_max)
    w.b_host = P.b
    w.b_dev = torch.tensor(P.b, device=dev)
    w.config = dict(workload_desc(P, args.config), parallelism="single",
                    matrix_stream=(f"diagonal copy, {w.A.ndiag} diagonals (uploaded as CSR)"
                                   if w.A.ndiag else "CSR"))
    return w


def setup_partitioned(args, ctx_device, world, rank, dev):
    """Weak scaling: rank r owns an x-slab of cfg2's size (configs.build_slab);
    one distributed solve over all ranks (halo exchange + sketch allreduce)."""
    import torch

    import paper_2503_22631_b200 as rk
    from paper_2503_22631_b200 import configs
    from paper_2503_22631_b200 import distributed as D
    transport = os.environ.get("RKMF_BENCH_TRANSPORT", "nccl")
    ctx = D.make_context(ctx_device, world, rank, transport)
    Sl = configs.build_slab(world, rank)
    part = D.partition_local(ctx, Sl.n_global, Sl.row_starts, Sl.row_ptr, Sl.col_idx, Sl.values,
                             Sl.b, Sl.d, Sl.zeta, configs.SKETCH_SEED, rank)
    w = Workload()
    w.ctx, w.P, w.n, w.nnz, w.m = ctx, None, part.n_local, Sl.nnz, Sl.m
    w.A, w.S = part.A, part.S
    w.f = rk.FunctionSpec.exp_neg(Sl.t)
    w.opts = rk.RestartOptions(m_r=Sl.m, tol=Sl.tol, k_max=Sl.k_max)
    w.b_host = part.b
    w.b_dev = torch.tensor(part.b, device=dev)
    w.config = {"workload": f"cfg2 weak-scaled: 3D 7-point Laplacian {128 * world}x128x128, "
                            f"one {128}^3 x-slab (cfg2's rows) per GPU",
                "matrix_rows": Sl.n_global, "nnz": Sl.nnz_global, "rows_per_gpu": part.n_local,
                "function": "exp_neg", "t": Sl.t, "m": Sl.m, "sketch_d": Sl.d, "zeta": Sl.zeta,
                "tol_abs": Sl.tol, "k_max": Sl.k_max, "b_seed": 1, "sketch_seed": 1,
                "l2_policy": "inputs larger than L2 (CSR + basis W exceed 126 MB)",
                "parallelism": f"row-partitioned x{world} ({transport}: halo send/recv + "
                               f"sketch allreduce per Krylov step)",
                "unit_note": "basis vectors counted per rank slab (value = world x m_k / s)",
                "matrix_stream": (f"diagonal copy, {part.A.ndiag} diagonals" if part.A.ndiag
                                  else "CSR")}
    return w


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2503_22631_b200 as rk

    rank, world, local = env_rank()
    if os.environ.get("RKMF_BENCH_ONE_GPU"):  # functional runs of N ranks on one GPU
        local = 0                             # (with RKMF_BENCH_TRANSPORT=host); not timing
    torch.cuda.set_device(local)
    if world > 1 and os.environ.get("RKMF_BENCH_ONE_GPU"):
        dist.init_process_group("gloo")  # NCCL refuses two ranks on one device
    elif world > 1:
        # CPU tensors (host transport, timing reductions) over gloo, CUDA over NCCL
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        w = setup_partitioned(args, local, world, rank, dev)
        ctx = w.ctx
    else:
        ctx = rk.Context.default(local)
        w = setup_single(args, ctx, dev)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream)
    A, S, f, opts, b_dev = w.A, w.S, w.f, w.opts, w.b_dev

    for _ in range(args.warmup):
        res = rk.restarted_krylov(A, b_dev, f, opts, S)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- timed region: device-resident inputs ----
    launches0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        total_m = 0
        for _ in range(args.steps):
            res = rk.restarted_krylov(A, b_dev, f, opts, S)
            total_m += res.total_m
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    gpu_launches = ctx.launch_count - launches0
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64)  # max over ranks (CPU tensor: gloo)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * total_m / (max_ms / 1e3)

    # ---- setup (once per matrix, outside both timed regions, reported):
    #      CSR upload from pinned host memory + validation, device sketch ----
    setup = None
    A2, S2 = A, S
    if world == 1:
        from paper_2503_22631_b200 import configs
        P = w.P
        rp_h = torch.from_numpy(P.row_ptr).pin_memory()
        ci_h = torch.from_numpy(P.col_idx).pin_memory()
        v_h = torch.from_numpy(P.values).pin_memory()
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        A2 = rk.SparseMatrix.from_csr(rp_h.numpy(), ci_h.numpy(), v_h.numpy(), ctx=ctx)
        s1 = time.perf_counter()
        S2 = rk.make_sketch(P.d, P.n, P.zeta, configs.SKETCH_SEED, ctx=ctx)
        torch.cuda.synchronize()
        s2 = time.perf_counter()
        setup = {"matrix_upload_validate_s": s1 - s0, "sketch_generate_s": s2 - s1,
                 "h2d_bytes": 8 * (P.n + 1) + 12 * P.nnz}

    # ---- e2e: the reference-facing call with HOST vectors: every step copies
    #      b host->device (pinned) and f device->host inside the timed region ----
    b_h = torch.from_numpy(w.b_host).pin_memory()
    f_h = torch.empty(w.n, dtype=torch.float64).pin_memory()
    e2e_steps = max(1, args.steps)
    rk.restarted_krylov(A2, b_h.numpy(), f, opts, S2, out=f_h.numpy())  # warm-up
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e2e_m = 0
    for _ in range(e2e_steps):
        r2 = rk.restarted_krylov(A2, b_h.numpy(), f, opts, S2, out=f_h.numpy())
        e2e_m += r2.total_m
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - w0
    del A2, S2
    et = torch.tensor([e2e_s], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_m / float(et.item())
    h2d = 8 * w.n
    d2h = 8 * w.n

    # ---- per-kernel breakdown (separate diagnostic solve, events per launch;
    #      every rank runs it so the collectives match) ----
    ctx.kernel_timing(True)
    ctx.kernel_times(reset=True)
    rb = rk.restarted_krylov(A, b_dev, f, opts, S)
    kt = ctx.kernel_times(reset=True)
    ctx.kernel_timing(False)
    if rank == 0:
        cb = class_bytes(w, rb.total_m, rb.cycles)
        peak, peak_src = measured_peaks()
        kernels = {}
        for cls, (kms, cnt) in kt.items():
            ent = {"ms": kms, "launches": cnt}
            if cls in cb and kms > 0:
                gbs = cb[cls] / (kms / 1e3) / 1e9
                ent.update({"alg_bytes": cb[cls], "achieved_gbs": gbs, "frac": gbs / peak})
            kernels[cls] = ent
        dom = max((c for c in cb if kernels[c]["ms"] > 0), key=lambda c: kernels[c]["ms"])
        dk = kernels[dom]
        cyc_bytes = sum(cb.values())
        traffic = None  # per-launch DRAM bytes of the committed ncu --set full capture
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
                tj = json.load(fh)
            if world == 1 and args.config == "cfg2" and dom in tj:
                traffic = tj[dom]["bytes"]
        except Exception:
            pass
        roofline = {"bound": "hbm", "kernel": dom, "achieved": dk["achieved_gbs"],
                    "peak": peak, "unit": "GB/s", "frac": dk["frac"],
                    "traffic": traffic, "alg_bytes_per_launch": dk["alg_bytes"] / dk["launches"],
                    "avg_launch_ms": dk["ms"] / dk["launches"], "peak_source": peak_src,
                    "whole_solve_gbs": cyc_bytes / (max_ms / args.steps / 1e3) / 1e9,
                    "per_kernel_frac": {c: kernels[c]["frac"] for c in cb
                                        if "frac" in kernels[c]}}
        cpu = None
        if world == 1:
            cv, cdt, cr = cpu_baseline_sample(w.P, 1, 1)
            cpu = {"value": cv, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"one restart cycle (m={w.m}) of {args.config}, single thread, "
                             f"{cdt:.1f} s"}
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded generators, BASELINE.json shapes)",
               "config": w.config,
               "solve": {"cycles": res.cycles, "total_m": res.total_m,
                         "converged": res.converged,
                         "solve_ms": max_ms / args.steps,
                         "update_norms": [h.update_norm for h in res.history],
                         "dense_f_ms": [h.funm_ms for h in rb.history]},
               "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu,
               "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h,
                       "note": "restarted_krylov(A, b_host, ...) per step with A and S "
                               "resident; setup reported separately",
                       "ms_per_step": 1e3 * float(et.item()) / e2e_steps},
               "setup": setup,
               "gpu_launches": gpu_launches, "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: W >= 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
