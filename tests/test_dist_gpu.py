"""Row-shard driver on the CUDA path: world_size 2 on one B200 (gloo carries the
amax all-reduce so two ranks can share the device; the product uses NCCL).

Both ranks quantize their row shards of a list of tensors with CudaOps
(batched libss launches); the concatenated shards must be bitwise the CPU
oracle's quantization of every whole tensor (max is exact and
order-free, so every rank derives the same global scale), in both exchange
modes.  Fault injection: a NaN in one rank's shard sets the sticky
non-finite flag on EVERY rank and gives that tensor G = 1 everywhere.
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


def _worker(rank, world, port, q, exchange="grouped", nan_at=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2605_12464_b200 as ss
        from paper_2605_12464_b200.dist import CudaOps, RowShardQuantizer, ShardPlan
        plan = ShardPlan(SHAPES, rank, world)
        shards = [x[slice(*plan.rows(k))].contiguous().cuda() for k, x in enumerate(_tensors())]
        if nan_at is not None and nan_at[0] == rank:
            shards[nan_at[1]][nan_at[2], nan_at[3]] = float("nan")
        ops = CudaOps(-8, 8, want_err=True, want_sums=True)
        outs = [ops.alloc_out(x) for x in shards]
        qz = RowShardQuantizer(plan, ops, group=None, device="cuda", exchange=exchange)
        n = qz.step(shards, outs)
        torch.cuda.synchronize()
        res = [None if o.codes.numel() == 0 else
               (o.codes.cpu().numpy(), o.scales.cpu().numpy(), o.err.cpu().numpy(), float(o.G.item()))
               for o in outs]
        gathered = [None] * world
        dist.all_gather_object(gathered, (res, ss.device_status(), qz.allreduces))
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


def _run(world, exchange="grouped", nan_at=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, exchange, nan_at)) for r in range(world)]
    for p in procs:
        p.start()
    n, gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return n, gathered


@pytest.mark.parametrize("world,exchange", [(2, "grouped"), (3, "grouped"), (2, "single")])
def test_sharded_cuda_equals_oracle(oracle_lib, world, exchange):
    n, gathered = _run(world, exchange)
    assert n >= 2  # one batched amax + one batched quantize launch at least
    assert all(st == 0 for _, st, _ in gathered)
    if exchange == "single":
        assert all(ar == 1 for _, _, ar in gathered)
    for k, x in enumerate(_tensors()):
        whole = oracle_lib.quantize(x, x.shape[0], x.shape[1], -8, 8, "tensor")
        parts = [g[0][k] for g in gathered if g[0][k] is not None]
        assert np.array_equal(np.concatenate([p[0] for p in parts]), whole.codes)
        assert np.array_equal(np.concatenate([p[1] for p in parts]), whole.scales)
        e = np.concatenate([p[2] for p in parts])
        assert np.array_equal(e.view(np.uint32), whole.err.view(np.uint32))
        assert all(np.float32(p[3]) == np.float32(whole.G) for p in parts)


@pytest.mark.parametrize("exchange", ["grouped", "single"])
def test_nan_on_one_rank_flags_every_rank(oracle_lib, exchange):
    # rank 1 of 2 holds rows 150..299 of tensor 0: poison its local row 10
    n, gathered = _run(2, exchange, nan_at=(1, 0, 10, 3))
    for res, st, _ in gathered:
        assert st & 1, st                       # SS_FLAG_NONFINITE on every rank
        assert res[0][3] == 1.0                 # tensor 0: G = 1 everywhere
    for k, x in enumerate(_tensors()):
        if k == 0:
            continue
        whole = oracle_lib.quantize(x, x.shape[0], x.shape[1], -8, 8, "tensor")
        parts = [g[0][k] for g in gathered if g[0][k] is not None]
        assert np.array_equal(np.concatenate([p[0] for p in parts]), whole.codes), k
        assert all(np.float32(p[3]) == np.float32(whole.G) for p in parts), k
