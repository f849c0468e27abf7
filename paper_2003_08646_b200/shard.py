"""Batch sharding across GPUs.

The lance_gemm path shards over the batch with no exchange on the data path.
GEMM rows are image-major (engines.hpp:199-200), so a contiguous batch slice is
a contiguous row block of every position GEMM and of y. Two parity modes:

* per-shard (default, no collective): each rank runs an independent
  ``lance_gemm`` on its slice. This is bit-exact against the reference run on
  that slice.
* global: after the range pass, one 128-byte all-reduce of the 16 (min, max)
  pairs (as one MAX over [-min, max]) reproduces the full-batch PerPosition
  fit (engines.hpp:157-165, fit_params quant.hpp:54-72). Every rank then
  quantises with those params (``LanceConv.forward(params=...)``). This is
  bit-exact against a single full-batch reference call.

Only ``torch.distributed`` plumbing lives here; the compute is the C ABI.
"""
from __future__ import annotations

import numpy as np

from .api import QuantParams


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of a batch of n images for `rank` of `world`
    (the first n % world ranks get one extra image)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def params_from_minmax(lo: np.ndarray, hi: np.ndarray, bits: int) -> list[QuantParams]:
    """fit_params (quant.hpp:54-72) from per-position ranges: scale = (hi-lo)/(2^b-1)
    in fp32 with IEEE division; -0 canonicalised to +0 as the reference's matmul
    accumulation never produces -0 (matrix.hpp:75-84)."""
    lo = np.asarray(lo, np.float32) + np.float32(0.0)
    hi = np.asarray(hi, np.float32) + np.float32(0.0)
    if np.isnan(lo).any() or np.isnan(hi).any():
        raise ValueError("fit_params: NaN in values")
    top = np.float32((1 << bits) - 1)
    out = []
    for a, b in zip(lo, hi):
        scale = np.float32(np.float32(b - a) / top)
        out.append(QuantParams(bits, float(a), float(b), float(scale)))
    return out


def allreduce_minmax(lo, hi, group=None):
    """Global (min, max) per position across ranks: one all-reduce of 32 floats
    (MAX over [-lo, hi]; -(-x) is exact). Works with any torch.distributed
    backend (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    lo_t = torch.as_tensor(np.asarray(lo, np.float32))
    hi_t = torch.as_tensor(np.asarray(hi, np.float32))
    buf = torch.cat([-lo_t, hi_t])
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=group)
    buf = buf.cpu().numpy()
    return -buf[:16], buf[16:]


def gather_batch(y_local, n_total: int, group=None):
    """All-gather of every rank's output slice along the batch (verification
    only, outside any timed region). Returns the full [N, ...] array on every
    rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.as_tensor(np.ascontiguousarray(y_local))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    sizes = [shard_range(n_total, world, r) for r in range(world)]
    shape = tuple(t.shape[1:])
    parts = [torch.empty((b - a,) + shape, dtype=t.dtype, device=t.device) for a, b in sizes]
    dist.all_gather(parts, t, group=group)
    return torch.cat(parts).cpu().numpy()
