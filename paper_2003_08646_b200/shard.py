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
    """Global (min, max) per position across ranks: one all-reduce of 2 x P floats
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
    n = lo_t.numel()  # 16 positions, or 36 for F(4x4)
    return -buf[:n], buf[n:]


def scatter_batch(x_full, n_total: int, shape_tail, src: int = 0, group=None):
    """Scatter of a full batch held by rank `src` into contiguous per-rank
    slices (verification only, outside any timed region).  x_full: the
    [N, ...] array on `src` (ignored elsewhere); returns this rank's slice.
    NCCL over NVLink on GPUs, gloo on CPU."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cuda = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if cuda else torch.device("cpu")
    spans = [shard_range(n_total, world, r) for r in range(world)]
    a, b = spans[rank]
    out = torch.empty((b - a,) + tuple(shape_tail), dtype=torch.float32, device=dev)
    if rank == src:
        full = torch.as_tensor(np.ascontiguousarray(x_full, dtype=np.float32)).to(dev)
        for r, (ra, rb) in enumerate(spans):
            if r == src:
                out.copy_(full[ra:rb])
            else:
                dist.send(full[ra:rb].contiguous(), dst=r, group=group)
    else:
        dist.recv(out, src=src, group=group)
    return out


def gather_batch(y_local, n_total: int, group=None):
    """All-gather of every rank's output slice along the batch (verification
    only, outside any timed region). Returns the full [N, ...] array on every
    rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = y_local if isinstance(y_local, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(y_local))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    else:
        t = t.cpu()
    sizes = [shard_range(n_total, world, r) for r in range(world)]
    shape = tuple(t.shape[1:])
    # Uneven shards: every rank contributes a slice padded to the largest one
    # (all_gather needs equal sizes), trimmed again after the exchange.
    mx = max(b - a for a, b in sizes)
    if t.shape[0] < mx:
        t = torch.cat([t, torch.zeros((mx - t.shape[0],) + shape, dtype=t.dtype, device=t.device)])
    parts = [torch.empty((mx,) + shape, dtype=t.dtype, device=t.device) for _ in sizes]
    dist.all_gather(parts, t.contiguous(), group=group)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, sizes)]).cpu().numpy()


def allreduce_ranges(buf, group=None):
    """Element-wise MAX all-reduce of a ``LanceConv.ranges`` buffer
    [-t_min, t_max, nan] across the batch shards: the global PerPosition fit
    of engines.hpp:157-165.  With NCCL the buffer stays on the device (one
    2P+1-float ncclAllReduce on the current stream, no host round trip);
    gloo reduces a host copy."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        dist.all_reduce(buf, op=dist.ReduceOp.MAX, group=group)
        return buf
    host = buf.cpu()
    dist.all_reduce(host, op=dist.ReduceOp.MAX, group=group)
    buf.copy_(host)
    return buf


def global_forward(conv, x, y=None, group=None, stream=None):
    """One shard's forward in the global-fit mode: K0 on the shard ->
    all-reduce of the ranges -> on-device re-fit -> K1 -> K3/K4.  Every rank
    of `group` must call it with its own slice; the result is bitwise the
    shard's rows of one full-batch lance_gemm."""
    r = conv.ranges(x, stream=stream)
    allreduce_ranges(r, group)
    return conv.forward(x, y, stream=stream, ranges=r)


def verify_sharded(x_full, w, spec, cfg, group=None, tile_m: int = 2):
    """Multi-GPU full-batch parity check of one layer (north star: NCCL only
    scatters inputs and gathers outputs for verification).  Rank 0 holds x
    [N,H,W,C] and w; x is scattered, every rank runs its slice in the
    global-fit mode (``global_forward``: K0 -> MAX all-reduce of the 2P+1
    range floats on the device -> re-fit -> K1 -> GEMM), and the gathered
    output is returned on every rank.  It must equal one full-batch
    lance_gemm call bitwise.  w must be given on every rank (with NCCL rank
    0's copy is broadcast)."""
    import torch
    import torch.distributed as dist

    from .api import ConvSpec, LanceConv

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    a, b = shard_range(spec.n, world, rank)
    xs = scatter_batch(x_full, spec.n, (spec.h, spec.w, spec.c), group=group)
    wt = torch.as_tensor(np.ascontiguousarray(w, dtype=np.float32)).cuda()
    if dist.get_backend(group) == "nccl":  # rank 0's filters everywhere
        dist.broadcast(wt, src=0, group=group)
    conv = LanceConv(ConvSpec(b - a, spec.c, spec.h, spec.w, spec.k, spec.pad), cfg,
                     device=torch.cuda.current_device(), tile_m=tile_m)
    conv.set_filters(wt)
    y = global_forward(conv, xs.cuda(), group=group)
    conv.sync()
    out = gather_batch(y, spec.n, group)
    conv.close()
    return out
