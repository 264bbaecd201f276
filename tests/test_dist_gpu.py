"""Row-shard driver on the CUDA path: world_size 2 on one B200 (gloo carries the
amax all-reduce so two ranks can share the device; the product uses NCCL).

Both ranks quantize their row shards of a list of tensors with CudaOps
(batched libss launches); the concatenated shards must be bitwise the
single-process quantization of every whole tensor (max is exact
and order-free, so every rank derives the same global scale).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ssgen

pytestmark = pytest.mark.gpu

SHAPES = [(300, 256), (7, 4096), (1, 64), (1024, 128), (129, 96)]


def _tensors():
    return [ssgen.generate("weight_outlier", r, c, seed=3, tid=700 + k) for k, (r, c) in enumerate(SHAPES)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_12464_b200.dist import CudaOps, RowShardQuantizer, ShardPlan
        plan = ShardPlan(SHAPES, rank, world)
        shards = [x[slice(*plan.rows(k))].contiguous().cuda() for k, x in enumerate(_tensors())]
        ops = CudaOps(-8, 8, want_err=True, want_sums=True)
        outs = [ops.alloc_out(x) for x in shards]
        qz = RowShardQuantizer(plan, ops, group=None, device="cuda")
        n = qz.step(shards, outs)
        torch.cuda.synchronize()
        res = [None if o.codes.numel() == 0 else
               (o.codes.cpu().numpy(), o.scales.cpu().numpy(), o.err.cpu().numpy(), float(o.G.item()))
               for o in outs]
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            q.put((n, gathered))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cuda_equals_unsharded(world):
    import paper_2605_12464_b200 as ss
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    n, gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert n >= 2  # one batched amax + one batched quantize launch at least
    for k, x in enumerate(_tensors()):
        whole = ss.quantize(x.cuda(), radius=8, gmode="tensor")
        torch.cuda.synchronize()
        parts = [g[k] for g in gathered if g[k] is not None]
        assert np.array_equal(np.concatenate([p[0] for p in parts]), whole.codes.cpu().numpy())
        assert np.array_equal(np.concatenate([p[1] for p in parts]), whole.scales.cpu().numpy())
        e = np.concatenate([p[2] for p in parts])
        assert np.array_equal(e.view(np.uint32), whole.err.cpu().numpy().view(np.uint32))
        assert all(p[3] == whole.G.item() for p in parts)
