"""Row-sharded long transforms across GPUs.

For a column too long for one GPU, the rows of the (Nt, K) block are split
into G contiguous slices, one per rank, and the DFT runs as a distributed
four-step decomposition Nt = N1 * N2 (n = n1 + N1 n2, k = k2 + N2 k1):

1. all-to-all: rank g trades its n2-slice (all n1) for an n1-slice (all n2);
2. local length-N2 FFTs over n2 for each local n1, then the four-step twiddle
   W_Nt^(n1 k2) — one Kron(Identity, Fourier) device plan plus a Diagonal;
3. all-to-all: n1-slices for k2-slices;
4. local length-N1 FFTs over n1 for each local k2;
5. all-to-all back to the natural row order (rank g holds output rows
   [g Nt / G, (g+1) Nt / G)).

No reference counterpart exists (the reference is single-process numpy);
the result equals ``kernels.dft`` of the gathered block (inverse: the
reference's conj-forward-conj / Nt).  The collective is
``torch.distributed.all_to_all_single`` — NCCL over NVLink on GPUs, gloo on
the CPU test; the local steps are pluggable (``DeviceLocalOps``: compiled
plans on CUDA tensors; tests inject a numpy implementation to check the
index bookkeeping with gloo on CPU).
"""

from __future__ import annotations

import numpy as np


def split_lengths(nt: int, world: int) -> tuple[int, int]:
    """(N1, N2) with N1 * N2 = nt, both divisible by `world` (powers of two:
    N1 the larger half of the exponent)."""
    if nt < 1 or nt & (nt - 1):
        raise ValueError(f"row-sharded DFT needs a power-of-two length, got {nt}")
    lg = nt.bit_length() - 1
    n1 = 1 << ((lg + 1) // 2)
    n2 = nt // n1
    if n1 % world or n2 % world:
        raise ValueError(f"length {nt} = {n1} x {n2} does not split over {world} ranks")
    return n1, n2


class DeviceLocalOps:
    """Local steps on the device: batched FFTs through compiled plans, the
    twiddle as a Diagonal plan (plans cached per shape / twiddle slice)."""

    def __init__(self):
        self._ops = {}

    def fft_rows(self, x, a: int, n: int, inverse: bool):
        """x: (a*n, K) CUDA tensor = a blocks of n rows; transform each block."""
        import paper_1710_09578_b200 as sm

        key = ("F", a, n)
        op = self._ops.get(key)
        if op is None:
            op = sm.Fourier(n) if a == 1 else sm.Kron(sm.Identity(a), sm.Fourier(n))
            self._ops[key] = op
        return op.backward(x) if inverse else op.forward(x)

    def scale_rows(self, x, w: np.ndarray, key):
        import paper_1710_09578_b200 as sm

        op = self._ops.get(("D", key))
        if op is None:
            op = sm.Diagonal(w)
            self._ops[("D", key)] = op
        return op.forward(x)


def _alltoall(t, group):
    """all_to_all_single along dim 0 (equal splits); identity for one rank."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    src = t.contiguous()
    if src.is_complex():  # (collectives move the (re, im) pairs as reals)
        src = torch.view_as_real(src)
    out = torch.empty_like(src)
    dist.all_to_all_single(out, src, group=group)
    return torch.view_as_complex(out) if t.is_complex() else out


def _rank_world(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def sharded_dft(x_local, nt: int, inverse: bool = False, group=None, ops=None):
    """DFT of a row-sharded (nt, K) block: x_local holds rows
    [g nt / G, (g+1) nt / G) of rank g; returns the same rows of dft(x)
    (or of the normalised inverse).  x_local: complex torch tensor.

    (The local re-layouts around each all-to-all are torch permute copies;
    folding them into the FFT passes' strided views is the next step.)"""
    g, world = _rank_world(group)
    ops = ops or DeviceLocalOps()
    n1, n2 = split_lengths(nt, world)
    a1, a2 = n1 // world, n2 // world
    squeeze = x_local.dim() == 1
    x = x_local[:, None] if squeeze else x_local
    k = x.shape[1]
    if x.shape[0] * world != nt:
        raise ValueError(f"local block has {x.shape[0]} rows, expected {nt // world}")
    # 1. (n2 slice, all n1) -> (all n2, n1 slice): layout (n1_local, n2, K)
    send = x.reshape(a2, world, a1, k).permute(1, 0, 2, 3).contiguous()
    recv = _alltoall(send, group)
    t = recv.reshape(n2, a1, k).permute(1, 0, 2).contiguous().reshape(a1 * n2, k)
    # 2. length-N2 FFTs over n2, four-step twiddle W^(+-n1 k2)
    t = ops.fft_rows(t, a1, n2, inverse)
    n1_idx = g * a1 + np.arange(a1)
    sgn = 1.0 if inverse else -1.0
    tw = np.exp(sgn * 2j * np.pi * np.outer(n1_idx, np.arange(n2)) / nt).reshape(-1)
    t = ops.scale_rows(t, tw, (nt, g, world, inverse))
    # 3. (n1 slice, all k2) -> (k2 slice, all n1): layout (k2_local, n1, K)
    send = t.reshape(a1, world, a2, k).permute(1, 0, 2, 3).contiguous()
    recv = _alltoall(send, group)
    t = recv.reshape(n1, a2, k).permute(1, 0, 2).contiguous().reshape(a2 * n1, k)
    # 4. length-N1 FFTs over n1: element (k2_local, k1) = X[k2 + N2 k1]
    t = ops.fft_rows(t, a2, n1, inverse)
    # 5. back to natural order: rank h holds k1 in its slice, all k2
    send = t.reshape(a2, world, a1, k).permute(1, 0, 2, 3).contiguous()
    recv = _alltoall(send, group)
    y = recv.reshape(n2, a1, k).permute(1, 0, 2).contiguous().reshape(a1 * n2, k)
    if inverse:
        y = y / nt
    return y[:, 0] if squeeze else y


def local_rows(x, rank: int, world: int):
    """Rank's contiguous row slice of an (nt, K) block."""
    n = x.shape[0] // world
    return x[rank * n:(rank + 1) * n]


__all__ = ["DeviceLocalOps", "local_rows", "sharded_dft", "split_lengths"]
