"""Multi-GPU path, CPU side: world_size-2 gloo process
groups exercise the batch-shard plumbing of paper_2003_08646_b200.shard.

The device compute is stood in for by the oracle (test infrastructure) so the
tests run without a GPU. They check:
  * per-shard mode: every rank's slice is an independent lance_gemm, and the
    gathered batch equals the per-slice reference calls;
  * global mode: the 128-byte MAX all-reduce of per-shard (min, max) pairs
    reproduces the full-batch PerPosition fit, and quantising every shard with
    those params gives the full-batch reference output bitwise.
The same flow runs on one GPU through the C ABI in
tests/test_gpu_parity.py::test_global_params_across_shards.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import Oracle, Spec
from paper_2003_08646_b200 import shard
from tests.golden_cases import make_inputs

SPEC = Spec(6, 16, 10, 10, 12, 1)  # N = 6 images -> 3 per rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        x, w = make_inputs(o.uniform, SPEC, "relu", 31)
        a, b = shard.shard_range(SPEC.n, world, rank)
        sspec = Spec(b - a, SPEC.c, SPEC.h, SPEC.w, SPEC.k, SPEC.pad)
        xs = x[a:b]
        # per-shard mode: independent lance_gemm on the slice
        y_local = o.lance_gemm(sspec, xs, w)
        y_all = shard.gather_batch(y_local, SPEC.n)
        # global mode: per-shard ranges -> all-reduce -> full-batch params
        _, dump = o.lance_gemm(sspec, xs, w, dump=True)
        v = dump["v"]
        lo, hi = v.min(axis=(1, 2)), v.max(axis=(1, 2))
        glo, ghi = shard.allreduce_minmax(lo, hi)
        params = shard.params_from_minmax(glo, ghi, 8)
        arr = np.array([[q.bits, q.t_min, q.t_max, q.scale] for q in params], np.float32)
        y_glob = o.lance_gemm(sspec, xs, w, in_params=arr)
        y_glob_all = shard.gather_batch(y_glob, SPEC.n)
        if rank == 0:
            results["y_all"] = y_all
            results["y_glob_all"] = y_glob_all
            results["params"] = arr
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (1, 5, 6, 256):
        for world in (1, 2, 3, 8):
            if world > n:
                continue
            spans = [shard.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_params_from_minmax_matches_fit_params():
    o = Oracle()
    vals = o.uniform(5, 4000).reshape(16, 250) * np.float32(3.7)
    ps = shard.params_from_minmax(vals.min(axis=1), vals.max(axis=1), 8)
    for p, row in zip(ps, vals):
        ref = o.fit_params(row, 8)
        assert (p.t_min, p.t_max, p.scale) == (ref.t_min, ref.t_max, ref.scale)


def test_gloo_world2_per_shard_and_global_parity():
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    o = Oracle()
    x, w = make_inputs(o.uniform, SPEC, "relu", 31)
    # per-shard mode == the reference run on each slice
    expect = np.concatenate([o.lance_gemm(Spec(b - a, SPEC.c, SPEC.h, SPEC.w, SPEC.k, SPEC.pad),
                                          x[a:b], w)
                             for a, b in (shard.shard_range(SPEC.n, 2, r) for r in range(2))])
    assert np.array_equal(results["y_all"].view(np.uint32), expect.view(np.uint32))
    # global mode == one full-batch reference call, bitwise (params and y)
    y_full, dump = o.lance_gemm(SPEC, x, w, dump=True)
    assert np.array_equal(results["params"], dump["params_a"])
    assert np.array_equal(results["y_glob_all"].view(np.uint32), y_full.view(np.uint32))
    # and the per-shard mode really differs from the full batch (batch coupling)
    assert not np.array_equal(results["y_all"], y_full)


def _scatter_worker(rank, world, port, results):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, tail = 7, (3, 4, 5)
        full = np.arange(n * 60, dtype=np.float32).reshape((n,) + tail) if rank == 0 else None
        part = shard.scatter_batch(full, n, tail)
        a, b = shard.shard_range(n, world, rank)
        ok = np.array_equal(part.numpy(), np.arange(n * 60, dtype=np.float32).reshape((n,) + tail)[a:b])
        back = shard.gather_batch(part, n)
        lo = np.linspace(-1, 0, 36).astype(np.float32) - rank
        hi = np.linspace(0, 1, 36).astype(np.float32) + rank
        glo, ghi = shard.allreduce_minmax(lo, hi)  # 36 positions (F(4x4))
        if rank == 0:
            results["ok"] = ok
            results["back"] = back
            results["glo"], results["ghi"] = glo, ghi
    finally:
        dist.destroy_process_group()


def test_gloo_world3_scatter_gather_and_36_position_allreduce():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_scatter_worker, args=(3, _free_port(), results), nprocs=3, join=True)
    assert results["ok"]
    assert np.array_equal(results["back"], np.arange(7 * 60, dtype=np.float32).reshape(7, 3, 4, 5))
    assert np.array_equal(results["glo"], np.linspace(-1, 0, 36).astype(np.float32) - 2)
    assert np.array_equal(results["ghi"], np.linspace(0, 1, 36).astype(np.float32) + 2)


def _ranges_worker(rank, world, port, results):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a LanceConv.ranges buffer: [-t_min[16], t_max[16], nan]; rank 1 saw a NaN
        o = Oracle()
        v = o.uniform(11 + rank, 16 * 50).reshape(16, 50) * np.float32(2.5 + rank)
        buf = torch.from_numpy(np.concatenate([-v.min(axis=1), v.max(axis=1),
                                               [1.0 if rank == 1 else 0.0]]).astype(np.float32))
        shard.allreduce_ranges(buf)
        results[rank] = buf.numpy()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_device_ranges_buffer_reduce():
    # The 2P+1-float buffer of the global-fit mode: one element-wise MAX gives
    # the global (min, max) per position (-(-x) exact) and propagates the NaN
    # flag (fmax would drop a NaN value itself, so it travels as 1.0).
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_ranges_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    o = Oracle()
    vs = [o.uniform(11 + r, 16 * 50).reshape(16, 50) * np.float32(2.5 + r) for r in range(2)]
    allv = np.concatenate(vs, axis=1)
    for r in range(2):
        got = results[r]
        assert np.array_equal(-got[:16], allv.min(axis=1))
        assert np.array_equal(got[16:32], allv.max(axis=1))
        assert got[32] == 1.0
        ps = shard.params_from_minmax(-got[:16], got[16:32], 8)
        for p, row in zip(ps, allv):
            ref = o.fit_params(row, 8)
            assert (p.t_min, p.t_max, p.scale) == (ref.t_min, ref.t_max, ref.scale)
