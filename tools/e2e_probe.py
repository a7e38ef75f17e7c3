"""Where the e2e (host-buffer) time of C2 goes: the public op.forward on a
pinned tensor vs the bare smat_apply_host call on preallocated pinned buffers
vs the device-only apply."""

import time

import numpy as np
import torch

import paper_1710_09578_b200 as sm
from paper_1710_09578_b200 import configs


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    w = configs.make(2)
    op = configs.operator(2, w)
    xh = torch.from_numpy(np.ascontiguousarray(w.X)).pin_memory()
    K = xh.shape[1]
    print(f"op.forward(pinned) : {timeit(lambda: op.forward(xh)):.2f} ms")
    out = torch.empty_like(xh).pin_memory()
    plan = op.plan_for(np.complex64, 0)
    code = plan.dtype_code
    print(f"apply_host (whole) : {timeit(lambda: plan.apply_host(0, xh.data_ptr(), code, out.data_ptr(), K, 0)):.2f} ms")
    for cc in (32, 16, 8):
        print(f"apply_host chunk {cc:2d}: "
              f"{timeit(lambda: plan.apply_host(0, xh.data_ptr(), code, out.data_ptr(), K, cc)):.2f} ms")
    def step():
        yh = op.forward(xh)
        return op.backward(yh)

    print(f"bench e2e step (fwd+bwd) : {timeit(step):.2f} ms")

    def step_fwd_only():
        return op.forward(xh)

    print(f"fwd only (new pinned out): {timeit(step_fwd_only):.2f} ms")
    yh = op.forward(xh)
    print(f"bwd only on pinned yh    : {timeit(lambda: op.backward(yh)):.2f} ms")
    print(f"yh pinned: {yh.is_pinned()}  dtype {yh.dtype}")
    xd = xh.cuda()
    print(f"device forward     : {timeit(lambda: op.forward(xd)):.2f} ms")
    yd = torch.empty_like(xd)
    print(f"H2D copy_          : {timeit(lambda: xd.copy_(xh, non_blocking=True)):.2f} ms")
    print(f"D2H copy_          : {timeit(lambda: out.copy_(yd, non_blocking=True)):.2f} ms")


if __name__ == "__main__":
    main()
