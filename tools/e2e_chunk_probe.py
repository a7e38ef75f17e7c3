"""C5 host-path time (pinned host block in, pinned host block out) against the
column chunk width of smat_apply_host: python tools/e2e_chunk_probe.py [cfg]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from paper_1710_09578_b200 import configs
import bench


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w = configs.make(cfg)
op = configs.operator(cfg, w)
xh = torch.from_numpy(np.ascontiguousarray(w.X)).pin_memory()
out = torch.empty_like(xh).pin_memory()
K = xh.shape[1]
plan = op.plan_for(bench.w_dtype(cfg), 0)
code = plan.dtype_code
for cc in (0, 64, 32, 16, 8, 4):
    if cc > K:
        continue
    f = timeit(lambda: plan.apply_host(0, xh.data_ptr(), code, out.data_ptr(), K, cc))
    b = timeit(lambda: plan.apply_host(1, xh.data_ptr(), code, out.data_ptr(), K, cc))
    print(f"cfg {cfg} chunk {cc:3d} columns: forward {f:7.2f} ms  backward {b:7.2f} ms  -> {2 * K / (f + b) * 1e3:8.1f} columns/s")
