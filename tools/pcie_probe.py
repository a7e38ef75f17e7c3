"""Host<->device copy bandwidth on this box (pinned memory): contiguous H2D /
D2H, both directions at once, and column-chunk (2-D, strided host rows)
copies — the numbers that bound bench.py's e2e line."""

import time

import torch


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


def main():
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    print(f"H2D contiguous 512 MiB: {bw(lambda: d.copy_(h, non_blocking=True), n):.1f} GB/s")
    print(f"D2H contiguous 512 MiB: {bw(lambda: h.copy_(d, non_blocking=True), n):.1f} GB/s")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    print(f"H2D + D2H concurrently: {bw(both, 2 * n):.1f} GB/s total")
    # column chunks of a (rows, 512 B) row-major block: 2-D copies, W bytes per row
    rows = n // 512
    hv = h.view(rows, 512)
    dv = d.view(rows, 512)
    for w in (64, 128, 256):
        def cols():
            for c0 in range(0, 512, w):
                dv[:, c0:c0 + w].copy_(hv[:, c0:c0 + w], non_blocking=True)
        print(f"H2D as {512 // w} column chunks of {w} B rows: {bw(cols, n, reps=2):.1f} GB/s")


if __name__ == "__main__":
    main()
