"""Benchmark of the structured-transform hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl reference]

Metric: forward/backward column throughput of one transform (columns/s) —
one step = forward A·X then backward A^H·Y over the whole (rows, K) block of
the workload, so value = 2K / step time (column-transforms per second, both
directions counted).  Default workload: BASELINE config C2 (Circulant 2^20,
64 complex64 columns) = configs[1]; c1..c5 select the others.

Device timing: inputs resident in HBM, W untimed warm-up steps, then exactly
K steps bracketed by barrier + cuda.synchronize, CUDA events on the launching
stream, max over ranks.  Working sets exceed the 126 MB L2 for c2..c5; c1 is
L2-flushed between steps (a 256 MB write).  Multi-GPU (torchrun): one process
per GPU, every rank transforms its own full K-column block (weak scaling,
column sharding, no collective on the data path; NCCL only for the barrier and
the max-over-ranks timing reduction).

Extra keys: e2e (the same metric through the public API with pinned HOST
buffers, H2D+D2H inside the timed region), roofline (dominant kernel,
algorithmic bytes per launch / its CUDA-event duration vs MEASURED_PEAKS.json),
cpu_baseline (the CPU oracle — a numpy port of the reference algorithm — on a
bounded sample on the host), gpu_launches, clocks.

--impl reference: times the reference algorithm's CPU implementation (the
oracle port; the reference is pure Python and cannot be installed on the GPU
box) with all host cores (one process per column), rank 0 only.

SURVEY.md §8(f) rows, one JSON line each (not driver workloads):
  --workload cg      device CG on C2's operator (normal equations, 64 rhs)
  --workload ista    the reference bench's ISTA scenario at size 2^20
  --workload sparse  Sparse (CSR) fwd + bwd, 2^20 x 2^20 with 16.8 M nonzeros
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd/bwd columns/s and achieved HBM GB/s per transform vs B200 HBM peak"
UNIT = "columns/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "cg", "ista", "sparse"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _workload_config(cfg: int):
    from paper_1710_09578_b200 import configs

    names = {1: "C1 Hadamard(10) 1024x16 float64", 2: "C2 Circulant(2^20) 2^20x64 complex64",
             3: "C3 Toeplitz(3000x3000) 3000x4096 float32",
             4: "C4 Kron(Hadamard(6),Fourier(128),Circulant(256)) 2^21x32 complex64",
             5: "C5 Diag(d1)·Fourier(1000003)·Diag(d2)·Sum(Hpad,LowRank32) 1000003x128 complex128"}
    dtypes = {1: "f64", 2: "c64", 3: "f32", 4: "c64", 5: "c128"}
    return names[cfg], dtypes[cfg], configs


# --------------------------------------------------------------- CPU legs ----
def _oracle_op(cfg, w):
    from oracle import linop_oracle as orc

    p = w.params
    if cfg == 1:
        return orc.hadamard(p["order"])
    if cfg == 2:
        return orc.circulant(p["c"])
    if cfg == 3:
        return orc.toeplitz(p["col"], p["row_rest"])
    if cfg == 4:
        return orc.kron(orc.hadamard(p["h_order"]), orc.fourier(p["f_n"]), orc.circulant(p["c"]))
    return orc.chain_c5(p["N"], p["d1"], p["d2"], p["U"], p["V"])


# columns per CPU sample so one sample is ~10-30 s of single-core numpy work
_SAMPLE_COLS = {1: 16, 2: 8, 3: 512, 4: 8, 5: 4}

_POOL_STATE = {}


def _pool_init(cfg):
    from paper_1710_09578_b200 import configs

    w = configs.make(cfg, ncols=1)
    _POOL_STATE["w"] = w
    _POOL_STATE["op"] = _oracle_op(cfg, w)
    _POOL_STATE["cfg"] = cfg


def _pool_column(j):
    from oracle import linop_oracle as orc

    w, op = _POOL_STATE["w"], _POOL_STATE["op"]
    x = w.X[:, :1]
    t0 = time.perf_counter()
    y = orc.apply(op, x, 0)
    orc.apply(op, y, 1)
    return time.perf_counter() - t0


def cpu_baseline(cfg: int, cols: int | None = None):
    """Single-core oracle (numpy port of the reference algorithm) on `cols` columns."""
    from oracle import linop_oracle as orc
    from paper_1710_09578_b200 import configs

    cols = cols or _SAMPLE_COLS[cfg]
    w = configs.make(cfg, ncols=cols)
    op = _oracle_op(cfg, w)
    orc.apply(op, w.X[:, :1], 0)  # warm the lru-cached plans (reference bench.py:263-270)
    t0 = time.perf_counter()
    y = orc.apply(op, w.X, 0)
    orc.apply(op, y, 1)
    dt = time.perf_counter() - t0
    return {"value": 2 * cols / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{cols} of {_full_cols(cfg)} columns, forward then backward, "
                      f"numpy oracle single-threaded ({dt:.2f} s)"}


def _full_cols(cfg):
    return {1: 16, 2: 64, 3: 4096, 4: 32, 5: 128}[cfg]


def run_reference(args, cfg):
    """--impl reference: the reference algorithm's CPU path with all host cores."""
    import multiprocessing as mp

    rank, world, _ = _dist_env()
    if rank != 0:
        return
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    name, dtype, _ = _workload_config(cfg)
    per_step = max(1, min(ncpu, _full_cols(cfg)))
    ctx = mp.get_context("fork")
    with ctx.Pool(per_step, initializer=_pool_init, initargs=(cfg,)) as pool:
        pool.map(_pool_column, range(per_step))  # warm-up: plans + page-in
        for _ in range(max(0, args.warmup - 1)):
            pool.map(_pool_column, range(per_step))
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_pool_column, range(per_step))
        dt = time.perf_counter() - t0
    value = 2 * per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (seeded numpy, SURVEY.md §8d)",
        "config": {"workload": name, "columns_per_step": 2 * per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": per_step, "kind": "port",
                         "sample": f"{per_step} columns per step (one process per column), forward+backward, "
                                   f"numpy port of the reference algorithm (oracle/linop_oracle.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU leg -----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return self
        # the timed region starts only once the sampler is producing lines
        # (short regions, e.g. 20 steps of C2 = 27 ms, still get samples)
        t0 = time.time()
        while time.time() - t0 < 5.0:
            if self.path.exists() and self.path.stat().st_size > 0:
                break
            time.sleep(0.01)
        self.skip = self.path.read_text().count("\n") if self.path.exists() else 0
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return None
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.path.read_text().splitlines()
        # samples taken after the timed region began (keep the last pre-region
        # sample when the region was shorter than the sampling interval)
        lines = lines[max(0, getattr(self, "skip", 0) - 1):]
        for line in lines:
            f = [t.strip() for t in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        self.path.unlink(missing_ok=True)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _pass_bytes(cfg: int, label: str, ncols: int) -> int | None:
    """Algorithmic HBM bytes of one launch of the labelled pass (SURVEY.md §8d
    units: each operand block read or written once, vectors once).  Labels are
    smat_apply_profiled's: kernel_length[_spec][_tw|_twin][_msk]."""
    K = ncols
    if cfg == 1:
        return 2 * 1024 * K * 8
    if cfg == 2:
        n = 1 << 20
        return 2 * n * K * 8 + (n * 8 if "_spec" in label else 0)
    if cfg == 3:
        return None  # compute-bound (single tile pass per column pair), no HBM roofline
    if cfg == 4:
        return 2 * (1 << 21) * K * 8
    if cfg == 5:
        n = configs_c5_n()
        M = 1 << (2 * n - 1).bit_length()
        P = 1 << max(0, (n - 1).bit_length())
        e = 16
        if label.startswith("wht_"):
            return (n + P) * K * e
        if label == "lowrank_contract":
            return n * K * e + n * 32 * e
        if label == "lowrank_expand":
            return n * 32 * e + 2 * n * K * e
        if "_spec" in label:
            return 2 * M * K * e + M * e
        if label.startswith("fft_c128_"):  # Bluestein outer passes: n-row side, M-row side, chirp
            return n * K * e + M * K * e + n * e
    return None


def configs_c5_n():
    from paper_1710_09578_b200 import configs
    return configs.C5_N


def _traffic(workload: str, kernel: str):
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(workload, {}).get(kernel)
    except (ValueError, AttributeError):
        return None


def run_native(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1710_09578_b200 as sm
    from paper_1710_09578_b200 import configs

    rank, world, local = _dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    name, dtype, _ = _workload_config(cfg)
    w = configs.make(cfg)
    op = configs.operator(cfg, w)
    K = w.ncols
    X = torch.from_numpy(np.ascontiguousarray(w.X)).to(f"cuda:{dev}")
    del w.X
    stream = torch.cuda.current_stream(dev)

    flush = None
    if cfg == 1:  # working set < L2: flush between timed steps
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    def step():
        if flush is not None:
            flush.fill_(1)
        y = op.forward(X)
        return op.backward(y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if flush is not None:  # subtract the flush writes, timed separately
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            flush.fill_(1)
        f1.record(stream)
        torch.cuda.synchronize()
        ms -= f0.elapsed_time(f1)
    t = torch.tensor([ms], device=f"cuda:{dev}", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * 2 * K / (ms_step / 1e3)

    # per-launch durations (CUDA events on the launching stream) for the roofline
    plan = op.plan_for(w_dtype(cfg), dev)
    pcode = plan.dtype_code
    xcode = pcode
    Y = op.forward(X)
    launches = {0: plan.launches(0, K), 1: plan.launches(1, K)}
    prof = []
    for _ in range(max(3, min(args.steps, 10))):
        prof += [("fwd",) + p for p in plan.apply_profiled(0, X, xcode, Y, K, stream.cuda_stream)]
        Z = torch.empty_like(X)
        prof += [("bwd",) + p for p in plan.apply_profiled(1, Y, xcode, Z, K, stream.cuda_stream)]
    by_kernel = {}
    for d, lab, t_ms in prof:
        by_kernel.setdefault(lab, []).append(t_ms)
    total = sum(sum(v) for v in by_kernel.values())
    peak, peak_src = _peaks()
    # per-pass breakdown, and the roofline of the dominant kernel: the kernel
    # family (precision + length, e.g. fft_c64_1024, all its fused variants)
    # with the largest share of the step; achieved = its algorithmic bytes per
    # launch over its mean launch time
    passes = {}
    for lab, ts in by_kernel.items():
        pb = _pass_bytes(cfg, lab, K)
        avg = float(np.mean(ts))
        passes[lab] = {"launches_per_step": len(ts) / max(3, min(args.steps, 10)), "avg_ms": avg,
                       "bytes_per_launch": pb, "GB/s": (pb / (avg / 1e3) / 1e9) if pb else None}

    def family(lab):
        parts = lab.split("_")
        return "_".join(parts[:3]) if lab.startswith("fft_") else lab

    fams = {}
    for lab, ts in by_kernel.items():
        fams.setdefault(family(lab), []).append(lab)
    dom = max(fams, key=lambda f: sum(sum(by_kernel[l]) for l in fams[f]))
    dom_t = sum(sum(by_kernel[l]) for l in fams[dom])
    dom_n = sum(len(by_kernel[l]) for l in fams[dom])
    roofline = None
    if all(_pass_bytes(cfg, l, K) is not None for l in fams[dom]):
        dom_b = sum(_pass_bytes(cfg, l, K) * len(by_kernel[l]) for l in fams[dom])
        pb = dom_b / dom_n
        dom_avg_ms = dom_t / dom_n
        achieved = pb / (dom_avg_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "variants": sorted(fams[dom]), "achieved": achieved,
                    "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": _traffic(args.workload, dom),
                    "bytes_per_launch": pb, "avg_launch_ms": dom_avg_ms,
                    "share_of_step": dom_t / total if total else None,
                    "peak_source": peak_src,
                    # the north star's "~8 TB/s" nominal B200 HBM3e peak
                    "frac_vs_nominal_8000": achieved / 8000.0}
    if cfg == 3:
        # FP32-bound config: algorithmic FFT flops of the
        # length-8192 embedding with real-pair packing, whole step, against the
        # nominal FP32 FFMA peak
        flops = 2 * configs.c3_flops_per_direction(K)
        achieved = flops / (ms_step / 1e3) / 1e12
        fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
        roofline = {"bound": "fp32", "kernel": "all fft_c64 passes of the step", "variants": sorted(by_kernel),
                    "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                    "traffic": None, "flops_per_step": flops,
                    "peak_source": "nominal FP32 FFMA: 148 SMs x 128 lanes x 2 flops x 1965 MHz"}
    alg = configs.algorithmic_bytes(cfg, K)
    transform_gbs = 2 * alg / (ms_step / 1e3) / 1e9

    # end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        e_steps = max(3, min(args.steps, 5))
        # two untimed steps in the timed loop's exact pattern, so the pinned
        # host caching allocator holds every output block the loop cycles through
        for _ in range(2):
            yh = op.forward(Xh)
            zh = op.backward(yh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            yh = op.forward(Xh)
            zh = op.backward(yh)
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], device=f"cuda:{dev}", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        bytes_in = Xh.numel() * Xh.element_size() + yh.numel() * yh.element_size()
        bytes_out = yh.numel() * yh.element_size() + zh.numel() * zh.element_size()
        e2e = {"value": world * 2 * K * e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(bytes_in),
               "d2h_bytes_per_step": int(bytes_out), "steps": e_steps,
               "path": "op.forward/op.backward on pinned CPU tensors (smat_apply_host, chunked H2D/compute/D2H)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic (seeded numpy, SURVEY.md §8d)",
            "config": {"workload": name, "columns_per_step": 2 * K, "global_columns": world * K,
                       "parallelism": f"column-sharded x{world} (no data-path collective)",
                       "l2": "inputs larger than L2" if cfg != 1 else "L2 flushed between steps (256 MB write)",
                       "step": "forward + backward over the whole block"},
            "transform_gbs": transform_gbs,
            "algorithmic_bytes_per_direction": alg,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(args.steps * (launches[0] + launches[1])),
            "launches_per_step": {"forward": launches[0], "backward": launches[1]},
            "kernels_ms_per_step": {k: float(np.sum(v)) / max(3, min(args.steps, 10)) for k, v in by_kernel.items()},
            "passes": passes,
            "plan": plan.describe(),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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


def w_dtype(cfg):
    return {1: np.float64, 2: np.complex64, 3: np.float32, 4: np.complex64, 5: np.complex128}[cfg]


def main():
    args = _args()
    if args.workload == "cg":
        run_solver(args)
        return
    if args.workload == "ista":
        run_ista(args)
        return
    if args.workload == "sparse":
        run_sparse(args)
        return
    cfg = int(args.workload[1])
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_native(args, cfg)


if __name__ == "__main__":
    main()
