"""Row-shard driver on the CUDA path: world_size 2 on one B200 (gloo carries the
amax all-reduce so two ranks can share the device; the product uses NCCL), and
the peer-memory exchange (CUDA IPC between the ranks' processes; gloo only
carries the IPC handles once).

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
        for _ in range(3 if exchange == "peer" else 1):  # peer: epochs 1..3 (both slot parities),
            n = qz.step(shards, outs)                    # enqueued back to back (ranks may run ahead)
        torch.cuda.synchronize()
        qz.close()
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


@pytest.mark.parametrize("world,exchange", [(2, "grouped"), (3, "grouped"), (2, "single"), (2, "peer"),
                                            (3, "peer")])
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


@pytest.mark.parametrize("exchange", ["grouped", "single", "peer"])
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


def test_peer_exchange_world1_equals_oracle(oracle_lib):
    """The peer-memory exchange at world size 1 (own buffer only, no process
    group): several steps (both slot parities), every output against the
    oracle; the C2 layer-0 shapes make several groups."""
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200.dist import CudaOps, RowShardQuantizer, ShardPlan
    specs = ssgen.workload("c2_qwen3_8b_weights")[:7]
    xs = [ssgen.generate(s.kind, s.rows // 8, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid) for s in specs]
    shapes = [tuple(x.shape) for x in xs] + [(0, 64), (3, 32)]
    xs += [torch.zeros(0, 64, dtype=torch.bfloat16), ssgen.generate("gaussian", 3, 32, seed=4, tid=4)]
    plan = ShardPlan(shapes, 0, 1)
    ops = CudaOps(-2, 6, want_err=True, want_sums=True)
    shards = [x.cuda() for x in xs]
    outs = [ops.alloc_out(x) for x in shards]
    qz = RowShardQuantizer(plan, ops, device="cuda", collective=True, exchange="peer")
    assert len(qz.groups) > 1
    for _ in range(3):
        qz.step(shards, outs)
    torch.cuda.synchronize()
    qz.close()
    assert ss.device_status() == 0
    for x, o in zip(xs, outs):
        if x.numel() == 0:
            continue
        r = oracle_lib.quantize(x, x.shape[0], x.shape[1], -2, 6, "tensor")
        assert np.array_equal(o.codes.cpu().numpy(), r.codes)
        assert np.array_equal(o.scales.cpu().numpy(), r.scales)
        assert np.array_equal(o.err.cpu().numpy().view(np.uint32), r.err.view(np.uint32))
        assert np.float32(o.G.item()) == np.float32(r.G)
        np.testing.assert_allclose(o.sums.cpu().numpy(), r.sums, rtol=1e-9)


def _worker_one_group(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2605_12464_b200 as ss
        from paper_2605_12464_b200.dist import CudaOps, RowShardQuantizer, ShardPlan
        x = ssgen.generate("gaussian", 2048, 4096, seed=5, tid=1)
        plan = ShardPlan([tuple(x.shape)], rank, world)
        shard = x[slice(*plan.rows(0))].contiguous().cuda()
        ops = CudaOps(-8, 8)
        outs = [ops.alloc_out(shard)]
        qz = RowShardQuantizer(plan, ops, device="cuda", exchange="peer")
        assert len(qz.groups) == 1
        for _ in range(8):   # one group: a rank can publish step e+1 before its peer consumed step e
            qz.step([shard], outs)
        torch.cuda.synchronize()
        qz.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, (outs[0].codes.cpu().numpy(), float(outs[0].G.item()),
                                          ss.device_status()))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_peer_exchange_one_group_back_to_back(oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_one_group, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = ssgen.generate("gaussian", 2048, 4096, seed=5, tid=1)
    whole = oracle_lib.quantize(x, 2048, 4096, -8, 8, "tensor")
    assert all(st == 0 for _, _, st in gathered)
    assert np.array_equal(np.concatenate([g[0] for g in gathered]), whole.codes)
    assert all(np.float32(g[1]) == np.float32(whole.G) for g in gathered)
