"""Multi-process sharding on the GPU: two ranks (gloo process group, both on
cuda:0 -- the driver's boxes have one GPU) run shard.verify_sharded: rank 0
scatters the batch, each rank runs its slice in the full-batch-parity mode
(local range pass -> MAX all-reduce of the per-position ranges -> static
forward), outputs are gathered.  The result must equal ONE full-batch
lance_gemm bitwise (and the per-shard mode must not), for F(2x2) and F(4x4)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from oracle import Oracle, Spec  # noqa: E402
from tests.golden.make_golden import make_inputs  # noqa: E402

pytestmark = pytest.mark.gpu
SPEC = Spec(5, 32, 13, 13, 24, 1)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, tile_m, results):
    import torch.distributed as dist
    import paper_2003_08646_b200 as lance
    from paper_2003_08646_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        x, w = make_inputs(o.uniform, SPEC, "relu", 77)
        cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
        spec = lance.ConvSpec(SPEC.n, SPEC.c, SPEC.h, SPEC.w, SPEC.k, SPEC.pad)
        y = shard.verify_sharded(x if rank == 0 else None, w, spec, cfg, tile_m=tile_m)
        if rank == 0:
            results["y"] = y
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tile_m", [2, 4])
def test_two_ranks_full_batch_parity(tile_m):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), tile_m, results), nprocs=2, join=True)
    o = Oracle()
    x, w = make_inputs(o.uniform, SPEC, "relu", 77)
    full = o.lance_gemm(SPEC, x, w, tile_m=tile_m)
    assert np.array_equal(results["y"].view(np.uint32), full.view(np.uint32))
