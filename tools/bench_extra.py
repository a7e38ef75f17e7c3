"""SURVEY.md §8(f) workloads of bench.py (not driver workloads): device CG on
C2's operator, the reference bench's ISTA scenario, Sparse CSR fwd/bwd.

    python bench.py --workload cg|ista|sparse [--steps K] [--warmup W]
"""

from __future__ import annotations

import time

import numpy as np

from bench import ClockSampler, _dist_env, _peaks


# ------------------------------------------------- solver leg ----
def run_solver(args):
    """--workload cg: conjugate gradients on the normal equations of C2's
    operator (Circulant 2^20, 64 right-hand sides, complex128 as the
    reference's cg_solve computes), fixed iteration count.  One step = one CG
    iteration over all 64 columns: A p and A^H (A p) through the compiled plan
    plus the fused step kernels, replayed from a CUDA graph."""
    import torch
    import torch.distributed as dist

    import paper_1710_09578_b200 as sm
    from paper_1710_09578_b200 import configs, solvers

    rank, world, local = _dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    w = configs.make(2)
    op = sm.Circulant(w.params["c"])
    K = w.ncols
    rhs = torch.from_numpy(np.ascontiguousarray(w.X)).to(f"cuda:{dev}").to(torch.complex128)
    del w.X
    opts_w = sm.SolveOptions(max_iterations=args.warmup, relative_tolerance=1e-300)
    sm.cg_solve(op, rhs, opts_w)  # warm-up: plans, workspaces, graph capture path
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    opts = sm.SolveOptions(max_iterations=args.steps, relative_tolerance=1e-300)
    stream = torch.cuda.current_stream(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        rep = sm.cg_solve(op, rhs, opts)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=f"cuda:{dev}", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_it = float(t.item()) / args.steps
    n = 1 << 20
    e = 16
    # per iteration: two 3-pass c128 convolutions (read+write of the block per
    # pass + spectrum) and the step kernels (p.ap reduce 2 blocks, x/r update
    # 4 read + 2 write, p update 2 read + 1 write)
    conv = 3 * 2 * n * K * e + n * e
    step_bytes = (2 + 6 + 3) * n * K * e
    it_bytes = 2 * conv + step_bytes
    peak, peak_src = _peaks()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import linop_oracle as orc

        its = 4
        t0 = time.perf_counter()
        orc.cg_solve(orc.circulant(configs.make(2, ncols=1).params["c"]), np.asarray(rhs[:, :1].cpu()),
                     max_iterations=its, tol=1e-300)
        dt = time.perf_counter() - t0
        cpu = {"value": its / dt, "unit": "column-iterations/s", "cores": 1, "kind": "port",
               "sample": f"1 of {K} columns, {its} iterations, numpy oracle of solvers.py:75-106 ({dt:.2f} s)"}
    if rank == 0:
        line = {
            "metric": "CG column-iterations/s (normal equations)", "value": world * K / (ms_it / 1e3),
            "unit": "column-iterations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_it, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (seeded numpy, C2 operator and block, SURVEY.md §8d)",
            "config": {"workload": "cg_solve(Circulant(2^20), 2^20x64 complex128, normal equations)",
                       "step": "one CG iteration over all 64 columns (A p, A^H A p, fused step kernels)",
                       "l2": "inputs larger than L2", "graph": solvers.last_loop_mode},
            "roofline": {"bound": "hbm", "kernel": "whole iteration", "achieved": it_bytes / (ms_it / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": it_bytes / (ms_it / 1e3) / 1e9 / peak,
                         "traffic": None, "bytes_per_launch": it_bytes, "peak_source": peak_src},
            "iterations_run": int(np.max(rep.iterations)),
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _ista_problem(size: int, seed: int = 1710):
    """The reference bench's ISTA scenario (pkg/src/linopkit/bench.py:142-162)
    restated: Partial(Hadamard(log2 m), rows) . Circulant(c), m = 2 size,
    size/16-sparse truth; returns (operator factors, b, lam) in numpy."""
    rng = np.random.default_rng([seed, size])
    m = 2 * size
    rows = rng.choice(m, size=size, replace=False)
    c = rng.standard_normal(m) / np.sqrt(m)
    xt = np.zeros(m)
    sup = rng.choice(m, size=max(1, size // 16), replace=False)
    xt[sup] = rng.standard_normal(sup.size) + np.sign(rng.standard_normal(sup.size))
    return rows, c, xt


def run_ista(args):
    """--workload ista: the reference bench's ISTA scenario at size 2^20
    (Partial(Hadamard(21), 2^20 rows) . Circulant(2^21), float64), a fixed step
    size, `--steps` ISTA iterations on the device (one CUDA graph replayed).
    value = ISTA iterations per second."""
    import torch

    import paper_1710_09578_b200 as sm
    from paper_1710_09578_b200 import solvers

    torch.cuda.set_device(0)
    size = 1 << 20
    rows, c, xt = _ista_problem(size)
    order = int(np.log2(2 * size))
    op = sm.Product(sm.Partial(sm.Hadamard(order), row_indices=rows), sm.Circulant(c))
    b = op.forward(xt)
    lam = 0.02 * float(np.abs(op.backward(b)).max())
    top = sm.power_iteration(op, mode="singular", tol=1e-6, max_iter=50, seed=0).value
    alpha = 1.0 / (1.01 * top ** 2)
    bd = torch.from_numpy(b).cuda()
    sm.ista(op, bd, sm.IstaOptions(lam=lam, steps=max(1, args.warmup), step_size=alpha))  # warm-up + capture
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        res = sm.ista(op, bd, sm.IstaOptions(lam=lam, steps=args.steps, step_size=alpha))
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_it = ev0.elapsed_time(ev1) / args.steps
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import linop_oracle as orc

        oo = orc.product(orc.partial(orc.hadamard(order), rows), orc.circulant(c))
        its = 2
        t0 = time.perf_counter()
        orc.ista(oo, b, lam, steps=its, step_size=alpha)
        dt = time.perf_counter() - t0
        cpu = {"value": its / dt, "unit": "iterations/s", "cores": 1, "kind": "port",
               "sample": f"{its} ISTA iterations (+1 residual), numpy oracle of solvers.py:163-194 ({dt:.2f} s)"}
    line = {
        "metric": "ISTA iterations/s (reference bench ista scenario)", "value": 1e3 / ms_it,
        "unit": "iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_it,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, reference bench.py:142-162 shapes)",
        "config": {"workload": "ista(Partial(Hadamard(21), 2^20 rows) . Circulant(2^21)), size 2^20",
                   "step": "one ISTA iteration: forward, residual, backward, soft-threshold update",
                   "graph": solvers.last_loop_mode},
        "final_objective": float(res.objective_trace[-1]),
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_sparse(args):
    """--workload sparse: Sparse (CSR) forward + backward of a 2^20 x 2^20
    float64 operator with 16 random nonzeros per row (duplicates summed) on a
    2^20 x 64 block — SURVEY.md §8(f) row 3 at scale.  HBM roofline: CSR
    arrays once per direction, one x row (K values) gathered per nonzero, y
    written once."""
    import torch

    import paper_1710_09578_b200 as sm

    torch.cuda.set_device(0)
    n, per_row, K = 1 << 20, 16, 64
    rng = np.random.default_rng(1710_3)
    rows = np.repeat(np.arange(n), per_row)
    cols = rng.integers(0, n, n * per_row)
    vals = rng.standard_normal(n * per_row)
    S = sm.Sparse.__new__(sm.Sparse)  # bulk constructor: arrays instead of a triplet list
    sm.Sparse._from_arrays(S, n, n, rows, cols, vals)
    X = torch.from_numpy(rng.standard_normal((n, K))).cuda()

    def step():
        return S.backward(S.forward(X))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    nnz = S.nnz
    # compulsory bytes per direction: CSR arrays, x and y once each (the
    # gathered x rows mostly hit L2 here; counting one DRAM row per nonzero
    # instead gives the `gather_model` upper bound)
    per_dir = nnz * (8 + 8) + (n + 1) * 8 + 2 * n * K * 8
    gather_dir = nnz * (8 + 8) + (n + 1) * 8 + nnz * K * 8 + n * K * 8
    peak, peak_src = _peaks()
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import linop_oracle as orc

        cols_s = 2
        tri = list(zip(rows.tolist(), cols.tolist(), vals.tolist()))
        oo = orc.sparse(n, n, tri)
        xs = X[:, :cols_s].cpu().numpy()
        t0 = time.perf_counter()
        orc.apply(oo, orc.apply(oo, xs, 0), 1)
        dt = time.perf_counter() - t0
        cpu = {"value": 2 * cols_s / dt, "unit": "columns/s", "cores": 1, "kind": "port",
               "sample": f"{cols_s} of {K} columns, forward then backward, numpy CSR oracle ({dt:.2f} s)"}
    line = {
        "metric": "Sparse fwd/bwd columns/s", "value": 2 * K / (ms / 1e3), "unit": "columns/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform CSR)",
        "config": {"workload": f"Sparse({n}x{n}, nnz {nnz}) on {n}x{K} float64",
                   "step": "forward + backward (conjugate-transposed CSR)"},
        "roofline": {"bound": "hbm", "kernel": "csr_kernel", "achieved": 2 * per_dir / (ms / 1e3) / 1e9,
                     "peak": peak, "unit": "GB/s", "frac": 2 * per_dir / (ms / 1e3) / 1e9 / peak, "traffic": None,
                     "bytes_per_launch": per_dir, "peak_source": peak_src,
                     "gather_model_GBps": 2 * gather_dir / (ms / 1e3) / 1e9},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


