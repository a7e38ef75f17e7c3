"""Benchmark of the structured-transform hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl reference]

Metric (BASELINE.json): forward/backward column throughput of one transform
(columns/s) — one step = forward A·X then backward A^H·Y over the whole
(rows, K) block of the workload, value = 2K / step time, with the achieved
HBM GB/s and roofline fractions beside it.  Default workload: C5, the largest
single-GPU configuration and the one at the reference's own arithmetic width
(Diag·Fourier(1,000,003)·Diag·Sum(Hpad, LowRank32), 1,000,003 x 128
complex128); c1..c4 select the other BASELINE configs, whose device numbers
also appear under `per_config` of the default line.

Multi-GPU: the named block is split into contiguous column
slices, one per GPU (strong scaling, no collective on the data path).
`--gpus N` without a torchrun environment launches the N ranks itself
(torch.distributed.run, 127.0.0.1); NCCL carries only the barrier and the
max-over-ranks timing reduction.  value = 2K / max-over-ranks step time.

Device timing: inputs resident in HBM, W untimed warm-up steps, every rank's
step captured in one CUDA graph and replayed; exactly K steps bracketed by
barrier + cuda.synchronize, CUDA events on the launching stream.  Working
sets exceed the 126 MB L2 for c2..c5; c1 is L2-flushed between steps.

Parity gate: before printing, at least 8 columns (including the first and the
last) of the timed step's outputs are compared with the CPU oracle (north
star: relative L2 <= 1e-12 complex128 / float64, <= 1e-5 complex64 / float32,
int32 and C1 float64 bit-exact).  A failing check prints no value and exits 1.

Extra keys: roofline (dominant kernel: algorithmic bytes per launch / its
CUDA-event duration vs MEASURED_PEAKS.json; step-level HBM fraction; FP64
fraction vs the box's measured DFMA / DMMA peak), e2e (the same metric through
op.forward / op.backward on pinned HOST buffers, copies inside the timed
region), cpu_baseline (single-core oracle port on a bounded sample),
gpu_launches, clocks, parity, per_config.

--impl reference: the UNMODIFIED reference package (baseline/_ref/linopkit,
installed with pip --no-deps from /root/reference) on the host cores, one
process per sampled column, rank 0 only.

--workload cg|ista|sparse: SURVEY.md §8(f) workloads (tools/bench_extra.py).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd/bwd columns/s and achieved HBM GB/s per transform vs B200 HBM peak"
UNIT = "columns/s"
NAMES = {1: "C1 Hadamard(10) 1024x16 float64", 2: "C2 Circulant(2^20) 2^20x64 complex64",
         3: "C3 Toeplitz(3000x3000) 3000x4096 float32",
         4: "C4 Kron(Hadamard(6),Fourier(128),Circulant(256)) 2^21x32 complex64",
         5: "C5 Diag(d1)·Fourier(1000003)·Diag(d2)·Sum(Hpad,LowRank32) 1000003x128 complex128"}
DTYPES = {1: "f64", 2: "c64", 3: "f32", 4: "c64", 5: "c128"}
TOL = {1: 0.0, 2: 1e-5, 3: 1e-5, 4: 1e-5, 5: 1e-12}
FULL_COLS = {1: 16, 2: 64, 3: 4096, 4: 32, 5: 128}


def _args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "cg", "ista", "sparse"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly instead of a CUDA graph")
    ap.add_argument("--parity-cols", type=int, default=8)
    return ap.parse_args(argv)


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------- launcher -----
def _launch_ranks(args) -> int:
    """--gpus N outside torchrun: start N ranks on this node ourselves."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# --------------------------------------------------------------- oracle -----
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


def parity_columns(K: int, want: int) -> list[int]:
    """At least `want` global columns (all of a block of at most 16 columns),
    always including the first and the last, the rest evenly spaced."""
    if K <= max(want, 16):
        return list(range(K))
    cols = {0, K - 1}
    for c in np.linspace(0, K - 1, num=want).astype(int).tolist():
        if len(cols) >= want:
            break
        cols.add(int(c))
    return sorted(cols)


def rank_parity(cfg, w, a, b, want, fetch):
    """This rank's share of the parity gate: the checked global columns inside
    its slice [a, b), fetched (local indices -> (y, z) host arrays) and
    compared with the oracle; None when it owns none of them."""
    mine = [c for c in parity_columns(w.ncols, want) if a <= c < b]
    if not mine:
        return None
    y, z = fetch([c - a for c in mine])
    return check_parity(cfg, w, _oracle_op(cfg, w), np.ascontiguousarray(w.X[:, mine]), y, z, mine)


def reduce_over_ranks(ms, par, cfg, world, device):
    """Slowest rank's timed-region milliseconds and the combined parity report
    (max errors over ranks; passes only if every rank's columns pass)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(ms)], device=device, dtype=torch.float64)
    ok = torch.tensor([1 if (par is None or par["pass"]) else 0], device=device, dtype=torch.int32)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        gathered = [None] * world
        dist.all_gather_object(gathered, par)
        pars = [p for p in gathered if p]
    else:
        pars = [par] if par else []
    parity = {"columns": sorted(c for p in pars for c in p["columns"]), "tol": TOL[cfg], "pass": bool(ok.item()),
              "oracle": "oracle/linop_oracle.py (pinned to the reference's outputs, tests/golden)"}
    for k in ("rel_l2_fwd", "rel_l2_bwd", "max_col_rel_l2_fwd", "max_col_rel_l2_bwd", "ref_metric_fwd",
              "ref_metric_bwd"):
        parity[k] = max((p[k] for p in pars), default=None)
    return float(t.item()), parity


def check_parity(cfg, w, oop, x_cols, y_cols, z_cols, cols):
    """North-star metrics of the checked columns: relative L2 (block and max
    per column) and the reference's max|err| / (1 + max|ref|)."""
    from oracle import linop_oracle as orc

    tol = TOL[cfg]
    ry = orc.apply(oop, x_cols, 0)
    rz = orc.apply(oop, ry, 1)
    out = {"columns": [int(c) for c in cols], "tol": tol}
    ok = True
    for name, got, ref in (("fwd", y_cols, ry), ("bwd", z_cols, rz)):
        got = np.asarray(got, dtype=np.complex128 if np.iscomplexobj(got) or np.iscomplexobj(ref) else np.float64)
        num = np.linalg.norm(got - ref, axis=0)
        den = np.linalg.norm(ref, axis=0)
        den[den == 0] = 1.0
        blk = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))
        col = float(np.max(num / den))
        refm = float(np.max(np.abs(got - ref)) / (1.0 + np.max(np.abs(ref))))
        out[f"rel_l2_{name}"] = blk
        out[f"max_col_rel_l2_{name}"] = col
        out[f"ref_metric_{name}"] = refm
        if tol == 0.0:
            ok &= bool(np.array_equal(got, ref))
        else:
            ok &= blk <= tol and col <= tol
    out["pass"] = bool(ok)
    return out


# --------------------------------------------------------------- CPU legs ---
def cpu_baseline(cfg: int, cols: int = 4):
    """Single-core oracle (numpy port of the reference algorithm) on `cols` columns."""
    from oracle import linop_oracle as orc
    from paper_1710_09578_b200 import configs

    cols = min(cols, FULL_COLS[cfg]) if cfg != 3 else 512
    w = configs.make(cfg, ncols=cols)
    op = _oracle_op(cfg, w)
    orc.apply(op, w.X[:, :1], 0)  # warm the lru-cached plans (reference bench.py:263-270)
    t0 = time.perf_counter()
    y = orc.apply(op, w.X, 0)
    orc.apply(op, y, 1)
    dt = time.perf_counter() - t0
    return {"value": 2 * cols / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{cols} of {FULL_COLS[cfg]} columns, forward then backward, numpy port of the "
                      f"reference algorithm (oracle/linop_oracle.py), single-threaded ({dt:.2f} s)"}


_REF = {}


def _ref_module():
    """The unmodified reference package: baseline/_ref (pip --target install of
    /root/reference, git-ignored, travels to the GPU box with the repo)."""
    for p in (ROOT / "baseline" / "_ref",):
        if (p / "linopkit" / "__init__.py").exists():
            sys.path.insert(0, str(p))
            try:
                import linopkit  # noqa: F401

                return linopkit, str(p)
            except Exception as e:  # pragma: no cover - environment dependent
                _log(f"reference import from {p} failed: {e}")
            finally:
                sys.path.remove(str(p))
    return None, None


def reference_op(lk, cfg, w):
    """The config's operator through the reference's own public API (the
    Sum / LowRank vehicle of SURVEY.md §8c for C5)."""
    p = w.params
    if cfg == 1:
        return lk.Hadamard(p["order"])
    if cfg == 2:
        return lk.Circulant(p["c"])
    if cfg == 3:
        return lk.Toeplitz(p["col"], p["row_rest"])
    if cfg == 4:
        return lk.Kron(lk.Hadamard(p["h_order"]), lk.Fourier(p["f_n"]), lk.Circulant(p["c"]))
    N = p["N"]
    idx = np.arange(N)
    hpad = lk.Partial(lk.Hadamard((N - 1).bit_length()), idx, idx)
    lr = lk.Product(lk.Dense(p["U"]), lk.Dense(np.ascontiguousarray(p["V"].conj().T)))
    s = lk.Product(lk.Blocks([[hpad, lr]]), lk.Blocks([[lk.Identity(N)], [lk.Identity(N)]]))
    return lk.Product(lk.Diagonal(p["d1"]), lk.Fourier(N), lk.Diagonal(p["d2"]), s)


def _ref_column(j):
    op, X, apply = _REF["op"], _REF["X"], _REF["apply"]
    x = np.ascontiguousarray(X[:, j % X.shape[1]])
    t0 = time.perf_counter()
    apply(op, apply(op, x, 0), 1)
    return time.perf_counter() - t0


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU path with all host threads."""
    import multiprocessing as mp

    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    from paper_1710_09578_b200 import configs

    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    per_step = max(1, min(ncpu, FULL_COLS[cfg]))
    lk, where = _ref_module()
    w = configs.make(cfg, ncols=per_step)
    if lk is not None:
        _REF["op"] = reference_op(lk, cfg, w)
        _REF["apply"] = lambda op, x, d: op.forward(x) if d == 0 else op.backward(x)
        kind, what = "reference", f"linopkit (unmodified, {where})"
    else:
        from oracle import linop_oracle as orc

        _REF["op"] = _oracle_op(cfg, w)
        _REF["apply"] = orc.apply
        kind, what = "port", "oracle port (reference package not importable)"
    _REF["X"] = w.X
    # one column per process; the operator is built once and shared copy-on-write
    with mp.get_context("fork").Pool(per_step) as pool:
        for _ in range(max(1, args.warmup)):
            pool.map(_ref_column, range(per_step))  # plan caches, page-in
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_ref_column, range(per_step))
        dt = time.perf_counter() - t0
    value = 2 * per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPES[cfg],
        "data": "synthetic (seeded numpy, SURVEY.md §8d)",
        "config": {"workload": NAMES[cfg], "global_columns": FULL_COLS[cfg], "columns_per_step": per_step,
                   "step": "forward + backward of each sampled column, one host process per column"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": per_step, "kind": kind,
                         "sample": f"{per_step} of {FULL_COLS[cfg]} columns per step (one process per column, "
                                   f"{per_step} of {ncpu} host threads), forward + backward through {what}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------- GPU helpers -----
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
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(workload: str, kernel: str):
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    try:
        per = json.loads(p.read_text()).get(workload, {})
    except (ValueError, AttributeError):
        return None
    if kernel in per:
        return per[kernel]
    # (the launch lists name a kernel family by precision and length; the
    # bench label adds the pass variant: fft_c128_2048 -> fft_c128_2048_spec)
    fam = [k for k in per if kernel.startswith(k + "_")]
    return per[max(fam, key=len)] if fam else None


def pass_bytes(cfg: int, label: str, K: int) -> int | None:
    """Algorithmic HBM bytes of one launch of the labelled pass (SURVEY.md §8d
    units: every operand block read or written once, parameters once)."""
    from paper_1710_09578_b200 import configs

    if cfg == 1:
        return 2 * 1024 * K * 8
    if cfg == 2:
        n = 1 << 20
        return 2 * n * K * 8 + (n * 8 if "_spec" in label else 0)
    if cfg == 3:
        return None
    if cfg == 4:
        return 2 * (1 << 21) * K * 8
    n = configs.C5_N
    M = 1 << (2 * n - 1).bit_length()
    P = 1 << max(0, (n - 1).bit_length())
    e = 16
    if label == "wht_lowrank_a":  # user side (n rows) + T1 (P rows) + V (n x 32)
        return (n + P) * K * e + n * 32 * e
    if label == "wht_lowrank_b":  # T1 + T2 (P rows each) + U~ (P x 32)
        return 2 * P * K * e + P * 32 * e
    if label.startswith("wht_"):
        return 2 * P * K * e
    if label == "lowrank_finalize":
        return None
    if "_spec" in label:
        return 2 * M * K * e + M * e
    if label.startswith("fft_c128_"):  # Bluestein outer passes: n-row or P-row side, M-row side, chirp
        return P * K * e + M * K * e + n * e
    return None


def _graph_step(step, enabled: bool):
    """Capture one step into a CUDA graph (returns (replay, outputs, mode))."""
    import torch

    if not enabled:
        return step, None, "eager"
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
            step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            outs = step()
        g.replay()
        torch.cuda.synchronize()
        return g.replay, outs, "cuda_graph"
    except Exception as e:  # pragma: no cover - capture failure falls back to eager launches
        _log(f"graph capture failed ({e}); eager launches")
        torch.cuda.synchronize()
        return step, None, "eager"


def measure_config(cfg, w, op, X, dev, args, steps, warmup, graph=True, clocks=False):
    """Device timing of fwd + bwd on the resident block X; returns a dict with
    the step time, per-launch profile and the outputs of the timed step."""
    import torch
    import torch.distributed as dist

    rank, world, _ = _dist_env()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}") if cfg == 1 else None
    outs = {}

    def step():
        y = op.forward(X)
        z = op.backward(y)
        outs["y"], outs["z"] = y, z
        return y, z

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    run, gouts, mode = _graph_step(step, graph)
    if gouts is not None:
        outs["y"], outs["z"] = gouts
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(dev) if clocks else None
    if sampler:
        sampler.__enter__()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1)
        run()
    ev1.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1)
    if flush is not None:  # subtract the flush writes, timed separately
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(steps):
            flush.fill_(1)
        f1.record(stream)
        torch.cuda.synchronize()
        ms -= f0.elapsed_time(f1)
    return {"ms": ms, "mode": mode, "y": outs["y"], "z": outs["z"], "clocks": sampler.summary() if sampler else None}


def kernel_profile(cfg, op, X, dev, K, reps=3):
    """Per-launch durations (CUDA events on the launching stream) of `reps`
    eager fwd + bwd applies: {label: [ms, ...]}."""
    import torch

    plan = op.plan_for(w_dtype(cfg), dev)
    stream = torch.cuda.current_stream(dev)
    Y = op.forward(X)
    Z = torch.empty_like(X)
    by = {}
    for _ in range(reps):
        for lab, t in plan.apply_profiled(0, X, plan.dtype_code, Y, K, stream.cuda_stream):
            by.setdefault(lab, []).append(t)
        for lab, t in plan.apply_profiled(1, Y, plan.dtype_code, Z, K, stream.cuda_stream):
            by.setdefault(lab, []).append(t)
    return plan, by


def roofline_of(cfg, workload, by, K, ms_step, reps, peak, peak_src, fp64_peak=None):
    """Dominant single kernel (largest share of the step) and the step-level fractions."""
    from paper_1710_09578_b200 import configs

    total = sum(sum(v) for v in by.values())
    passes = {}
    for lab, ts in by.items():
        pb = pass_bytes(cfg, lab, K)
        avg = float(np.mean(ts))
        passes[lab] = {"launches_per_step": len(ts) / reps, "avg_ms": avg, "bytes_per_launch": pb,
                       "GB/s": (pb / (avg / 1e3) / 1e9) if pb else None,
                       "frac": (pb / (avg / 1e3) / 1e9 / peak) if pb else None,
                       "share_of_step": sum(ts) / total if total else None}
    alg = configs.algorithmic_bytes(cfg, K)
    step_gbs = 2 * alg / (ms_step / 1e3) / 1e9
    rf = {"bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": peak_src,
          "step_level": {"achieved": step_gbs, "frac": step_gbs / peak, "bytes_per_step": 2 * alg,
                         "definition": "algorithmic bytes of the minimal-pass plan (SURVEY.md §8d) per step / "
                                       "device step time"}}
    cands = [l for l in by if pass_bytes(cfg, l, K)]
    if cands:
        dom = max(cands, key=lambda l: sum(by[l]))
        rf.update({"kernel": dom, "achieved": passes[dom]["GB/s"], "frac": passes[dom]["frac"],
                   "traffic": _traffic(workload, dom), "bytes_per_launch": passes[dom]["bytes_per_launch"],
                   "avg_launch_ms": passes[dom]["avg_ms"], "share_of_step": passes[dom]["share_of_step"],
                   "frac_vs_nominal_8000": passes[dom]["GB/s"] / 8000.0})
    else:
        rf.update({"kernel": None, "achieved": step_gbs, "frac": step_gbs / peak, "traffic": None})
    if cfg == 3 and fp64_peak is not None:
        fl = 2 * configs.c3_flops_per_direction(K)
        ach = fl / (ms_step / 1e3) / 1e12
        rf["fp32"] = {"achieved": ach, "peak": fp64_peak["ffma2_fp32"], "unit": "TFLOP/s",
                      "frac": ach / fp64_peak["ffma2_fp32"], "flops_per_step": fl,
                      "peak_source": "measured FFMA2 (smat_probe_peak kind 3, this box)"}
    if cfg == 5 and fp64_peak is not None:
        fl = 2 * configs.c5_flops_per_direction(K)
        ach = fl / (ms_step / 1e3) / 1e12
        pk = max(fp64_peak["dfma_fp64"], fp64_peak["dmma_fp64"])
        rf["fp64"] = {"achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "flops_per_step": fl,
                      "peak_source": "measured max(DFMA, DMMA) FP64 peak of this box (smat_probe_peak; "
                                     "the two share one pipe)",
                      "definition": "algorithmic FP64 flops per step (SURVEY.md §8d: FFT 5 M log2 M x2, "
                                    "rank-32 halves 8 n r x2, FWHT 2 P log2 P, diagonals) / device step time"}
    return rf, passes


def w_dtype(cfg):
    return {1: np.float64, 2: np.complex64, 3: np.float32, 4: np.complex64, 5: np.complex128}[cfg]


def probe_peaks(dev):
    from paper_1710_09578_b200 import _native

    names = ["dfma_fp64", "dmma_fp64", "dfma_plus_dmma_fp64", "ffma2_fp32"]
    return {n: _native.probe_peak(k, dev) for k, n in enumerate(names)}


# ------------------------------------------------------------- GPU leg ------
def run_native(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1710_09578_b200 import configs, sharding

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.cuda.current_device()
    peak, peak_src = _peaks()
    w = configs.make(cfg)
    op = configs.operator(cfg, w)
    K = w.ncols
    a, b = sharding.column_slices(K, world)[rank]
    Kl = b - a
    Xh_local = np.ascontiguousarray(w.X[:, a:b])
    X = torch.from_numpy(Xh_local).to(f"cuda:{dev}")

    m = measure_config(cfg, w, op, X, dev, args, args.steps, args.warmup, graph=not args.no_graph, clocks=True)

    # parity gate on the outputs of the timed step (this rank's checked columns)
    par = rank_parity(cfg, w, a, b, args.parity_cols, lambda loc: (m["y"][:, loc].cpu().numpy(),
                                                                   m["z"][:, loc].cpu().numpy()))
    ms_max, parity = reduce_over_ranks(m["ms"], par, cfg, world, f"cuda:{dev}")
    ms_step = ms_max / args.steps
    value = 2 * K / (ms_step / 1e3)

    # per-launch profile and rooflines (eager, events on the launching stream)
    # (before the FP64 / FP32 peak probes: their power draw would carry into
    # the FP64-heavy passes profiled right after them)
    reps = 5
    plan, by = kernel_profile(cfg, op, X, dev, Kl, reps)
    fp_peaks = probe_peaks(dev) if rank == 0 else None
    rf, passes = roofline_of(cfg, args.workload, by, Kl, ms_step * 1.0, reps, peak, peak_src, fp_peaks)
    launches = plan.launches(0, Kl) + plan.launches(1, Kl)

    # end to end through the public API with pinned HOST buffers
    e2e = None
    if not args.no_e2e:
        # this rank's column slice as a strided view of the whole pinned host
        # block: the host path stages it with pitched copies (ABI ldx), no
        # host-side repacking inside or outside the timed region
        Xh = torch.from_numpy(np.ascontiguousarray(w.X)).pin_memory()[:, a:b]
        e_steps = max(3, min(int(args.steps), 10))
        for _ in range(3):  # the pinned caching allocator holds the blocks the loop cycles through
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
        bi = torch.tensor([Xh.numel() * Xh.element_size() + yh.numel() * yh.element_size()], device=f"cuda:{dev}",
                          dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dist.all_reduce(bi, op=dist.ReduceOp.SUM)
        dt = float(tt.item())
        nb = int(bi.item())
        e2e = {"value": 2 * K * e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
               "steps": e_steps,
               "path": "op.forward / op.backward on pinned CPU tensors (smat_apply_host: chunked pitched H2D, "
                       "device passes, D2H on three streams)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)

    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config:
        per_config = {}
        for c2 in (1, 2, 3, 4, 5):
            if c2 == cfg:
                continue
            try:
                per_config[f"c{c2}"] = _per_config(c2, dev, peak, peak_src, fp_peaks, not args.no_graph)
            except Exception as e:  # pragma: no cover - report, never hide the headline
                per_config[f"c{c2}"] = {"error": repr(e)}
            torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value if parity["pass"] else None, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPES[cfg],
            "data": "synthetic (seeded numpy, SURVEY.md §8d)",
            "config": {"workload": NAMES[cfg], "global_columns": K,
                       "columns_per_rank": [e - s for s, e in sharding.column_slices(K, world)],
                       "parallelism": f"column slices x{world} (strong scaling, no data-path collective)",
                       "l2": "inputs larger than L2" if cfg != 1 else "L2 flushed between steps (256 MB write)",
                       "step": "forward + backward over the whole block", "launch": m["mode"]},
            "transform_gbs": rf["step_level"]["achieved"],
            "roofline": rf,
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(args.steps * launches),
            "launches_per_step": launches,
            "passes": passes,
            "measured_peaks_tflops": fp_peaks,
            "per_config": per_config,
            "plan": plan.describe(),
            "clocks": m["clocks"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if parity["pass"] else 1


def _per_config(cfg, dev, peak, peak_src, fp_peaks, graph):
    """Device-only line of another config: ms/step, roofline, parity of two columns."""
    import torch

    from paper_1710_09578_b200 import configs

    w = configs.make(cfg)
    op = configs.operator(cfg, w)
    K = w.ncols
    X = torch.from_numpy(np.ascontiguousarray(w.X)).to(f"cuda:{dev}")
    m = measure_config(cfg, w, op, X, dev, None, 10, 3, graph=graph)
    ms_step = m["ms"] / 10
    cols = [0, K - 1]
    par = check_parity(cfg, w, _oracle_op(cfg, w), np.ascontiguousarray(w.X[:, cols]),
                       m["y"][:, cols].cpu().numpy(), m["z"][:, cols].cpu().numpy(), cols)
    plan, by = kernel_profile(cfg, op, X, dev, K, 3)
    rf, _ = roofline_of(cfg, f"c{cfg}", by, K, ms_step, 3, peak, peak_src, fp_peaks)
    return {"workload": NAMES[cfg], "dtype": DTYPES[cfg], "ms_per_step": ms_step, "value": 2 * K / (ms_step / 1e3),
            "unit": UNIT, "roofline": rf, "parity": par, "launch": m["mode"],
            "kernels_ms_per_step": {k: float(np.sum(v)) / 3 for k, v in by.items()}}


def main():
    args = _args()
    if args.workload in ("cg", "ista", "sparse"):
        sys.path.insert(0, str(ROOT / "tools"))
        import bench_extra

        {"cg": bench_extra.run_solver, "ista": bench_extra.run_ista, "sparse": bench_extra.run_sparse}[
            args.workload](args)
        return 0
    cfg = int(args.workload[1])
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _launch_ranks(args)
    return run_native(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
