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
