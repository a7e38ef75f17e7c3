"""Multi-process (gloo, world size 2) test of the column-sharding host logic.

The device path cannot run on the CPU-only build container; each rank applies
the CPU oracle to its column slice instead, which exercises exactly the same
partition / gather / max-over-ranks logic bench.py uses with NCCL on GPUs.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1710_09578_b200 import sharding


def test_column_slices_partition():
    for k in (1, 2, 7, 16, 64, 4096):
        for w in (1, 2, 3, 4, 8):
            s = sharding.column_slices(k, w)
            assert len(s) == w and s[0][0] == 0 and s[-1][1] == k
            assert all(a <= b for a, b in s) and all(s[i][1] == s[i + 1][0] for i in range(w - 1))
            widths = [b - a for a, b in s]
            assert max(widths) - min(widths) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import linop_oracle as orc

        rng = np.random.default_rng(0)  # same block on every rank
        c = rng.standard_normal(64) + 1j * rng.standard_normal(64)
        x = rng.standard_normal((64, 7)) + 1j * rng.standard_normal((64, 7))
        op = orc.circulant(c)
        local = sharding.shard_apply(lambda a: orc.apply(op, a, 0), x, rank, world)
        full = sharding.gather_columns(local)
        ref = orc.apply(op, x, 0)
        ok = bool(np.allclose(full, ref, rtol=1e-12, atol=1e-12))
        tmax = sharding.max_over_ranks(float(rank + 1))
        q.put((rank, ok, tmax, local.shape[1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_shard_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    res.sort()
    assert all(ok for _, ok, _, _ in res)
    assert all(t == 2.0 for _, _, t, _ in res)  # max over ranks
    assert sorted(w for *_, w in res) == [3, 4]  # 7 columns split 4 + 3


class _NumpyLocalOps:
    """CPU stand-in for the device local steps of rowshard.sharded_dft (the
    gloo test checks the all-to-all bookkeeping; the device steps are checked
    on the GPU in tests/test_gpu_extra.py)."""

    def fft_rows(self, x, a, n, inverse):
        import torch

        arr = x.numpy().reshape(a, n, -1)
        f = np.fft.ifft(arr, axis=1) * n if inverse else np.fft.fft(arr, axis=1)
        return torch.from_numpy(np.ascontiguousarray(f.reshape(a * n, -1)))

    def scale_rows(self, x, w, key):
        import torch

        return x * torch.from_numpy(w)[:, None]


def _rowshard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1710_09578_b200 import rowshard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        nt, k = 1 << 10, 3
        x = rng.standard_normal((nt, k)) + 1j * rng.standard_normal((nt, k))
        xl = torch.from_numpy(np.ascontiguousarray(rowshard.local_rows(x, rank, world)))
        ops = _NumpyLocalOps()
        y = rowshard.sharded_dft(xl, nt, ops=ops).numpy()
        ok_f = bool(np.allclose(y, rowshard.local_rows(np.fft.fft(x, axis=0), rank, world), atol=1e-9))
        z = rowshard.sharded_dft(torch.from_numpy(y), nt, inverse=True, ops=ops).numpy()
        ok_i = bool(np.allclose(z, rowshard.local_rows(x, rank, world), atol=1e-12))
        q.put((rank, ok_f, ok_i))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_row_sharded_dft():
    """Row-sharded four-step DFT (rowshard.py, §8(f) row 4): three
    all-to-alls over gloo with world size 2 reproduce np.fft on the gathered
    column, forward and inverse."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rowshard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    assert all(f and i for _, f, i in res), res


def test_rowshard_split_lengths():
    from paper_1710_09578_b200 import rowshard

    assert rowshard.split_lengths(1 << 10, 2) == (32, 32)
    assert rowshard.split_lengths(1 << 21, 8) == (2048, 1024)
    with pytest.raises(ValueError):
        rowshard.split_lengths(1000, 2)
    with pytest.raises(ValueError):
        rowshard.split_lengths(16, 8)  # 4 x 4 does not split over 8 ranks
    x = np.arange(24).reshape(12, 2)
    assert np.array_equal(rowshard.local_rows(x, 1, 3), x[4:8])


def _bench_worker(rank, world, port, q):
    """One rank of bench.py's multi-GPU path with the device steps replaced by
    the CPU oracle: the same column slice, the same parity share and the same
    max-over-ranks / parity reduction the native arm runs over NCCL."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import linop_oracle as orc
        from paper_1710_09578_b200 import configs

        w = configs.make(2, n=4096)  # C2's seeded draw at a small length, all 64 columns
        K = w.ncols
        a, b = sharding.column_slices(K, world)[rank]
        oop = bench._oracle_op(2, w)
        y = orc.apply(oop, w.X[:, a:b], 0)
        z = orc.apply(oop, y, 1)
        par = bench.rank_parity(2, w, a, b, 8, lambda loc: (y[:, loc], z[:, loc]))
        ms, parity = bench.reduce_over_ranks(10.0 + rank, par, 2, world, "cpu")
        q.put((rank, (a, b), ms, parity))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_world2_bench_shard_parity_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=170) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    import bench

    assert [r[1] for r in res] == [(0, 32), (32, 64)]            # strong scaling: the named block split
    assert all(r[2] == 11.0 for r in res)                          # slowest rank's time on every rank
    for _, _, _, parity in res:
        assert parity["pass"] and parity["columns"] == bench.parity_columns(64, 8)
        assert 0 in parity["columns"] and 63 in parity["columns"]  # first and last column checked
        assert parity["rel_l2_fwd"] == 0.0
