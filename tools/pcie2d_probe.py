"""Pitched (2-D) host<->device copies on this box: a (rows, 512 B) pinned
row-major block copied as column chunks of W bytes per row with
cudaMemcpy2DAsync, one chunk per stream, H2D alone and H2D + D2H overlapped —
whether column-chunked host transfers can pipeline against the transform."""

import time

import torch
from cuda.bindings import runtime as rt


def main():
    n = 512 << 20
    rows, pitch = n // 512, 512
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
    D2H = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
    for w in (64, 128, 256, 512):
        def run(both):
            for k, c0 in enumerate(range(0, pitch, w)):
                s = streams[k % 4].cuda_stream
                rt.cudaMemcpy2DAsync(d.data_ptr() + c0, pitch, h.data_ptr() + c0, pitch, w, rows, H2D, s)
                if both:
                    rt.cudaMemcpy2DAsync(h2.data_ptr() + c0, pitch, d2.data_ptr() + c0, pitch, w, rows, D2H, s)
            torch.cuda.synchronize()
        for both in (False, True):
            run(both)
            t0 = time.perf_counter()
            for _ in range(3):
                run(both)
            dt = (time.perf_counter() - t0) / 3
            print(f"W={w:4d} B rows {'H2D+D2H' if both else 'H2D    '}: {(2 if both else 1) * n / dt / 1e9:6.1f} GB/s total")


if __name__ == "__main__":
    main()
