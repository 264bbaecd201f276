"""Row-shard driver host logic on CPU: world_size 2 over gloo.

The driver (paper_2605_12464_b200/dist.py) only sequences calls: shard amax ->
ONE max all-reduce of every tensor's amax -> quantize each shard with the
given amax.  Here the per-shard compute is the CPU oracle (test
infrastructure), so the test checks the sequencing and the exchange: the
sharded outputs, concatenated over ranks, must be bitwise the unsharded
quantization of each whole tensor, including uneven and empty shards.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ssgen

SHAPES = [(37, 64), (5, 32), (1, 16), (64, 128)]   # 1 row: one rank gets an empty shard
FMIN, FMAX = -8, 8


class OracleOps:
    """Same interface as dist.CudaOps, backed by the oracle on CPU tensors."""

    def __init__(self):
        import oracle
        self.o = oracle

    def new_amax(self, n, device):
        return torch.zeros(n, dtype=torch.int32)

    def amax_all(self, xs, buf):
        for k, x in enumerate(xs):
            buf[k] = self.o.tensor_amax(x) if x.numel() else 0
        return 1

    def alloc_out(self, x):
        return {}

    def quantize_next_amax(self, xs, buf, outs, next_xs, next_buf):
        # the grouped step's fused call: quantize this group, local amaxes of the next
        self.amax_all(next_xs, next_buf)
        return self.quantize_all(xs, buf, outs)

    def quantize_all(self, xs, buf, outs):
        for x, slot, out in zip(xs, buf, outs):
            if x.shape[0] == 0:
                continue
            r = self.o.quantize(x, x.shape[0], x.shape[1], FMIN, FMAX, "given",
                                amax_bits=int(slot.item()) & 0xFFFFFFFF)
            out.update(codes=r.codes, scales=r.scales, err=r.err, G=r.G)
        return 1


def _tensors():
    return [ssgen.generate("weight_outlier" if k % 2 else "student_t", r, c, seed=11, tid=k)
            for k, (r, c) in enumerate(SHAPES)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_12464_b200.dist import RowShardQuantizer, ShardPlan
        full = _tensors()
        plan = ShardPlan(SHAPES, rank, world)
        shards = [x[slice(*plan.rows(k))].contiguous() for k, x in enumerate(full)]
        ops = OracleOps()
        outs = [ops.alloc_out(x) for x in shards]
        qz = RowShardQuantizer(plan, ops, group=None, device="cpu")
        n = qz.step(shards, outs)
        gathered = [None] * world
        dist.all_gather_object(gathered, [{k: (v if not isinstance(v, np.ndarray) else v.copy())
                                           for k, v in o.items()} for o in outs])
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
def test_row_shards_equal_whole_tensor(oracle_lib, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    n, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert n > 0
    for k, x in enumerate(_tensors()):
        whole = oracle_lib.quantize(x, x.shape[0], x.shape[1], FMIN, FMAX, "tensor")
        parts = [g[k] for g in gathered if g[k]]
        codes = np.concatenate([p["codes"] for p in parts], 0)
        scales = np.concatenate([p["scales"] for p in parts], 0)
        err = np.concatenate([p["err"] for p in parts], 0)
        assert np.array_equal(codes, whole.codes), k
        assert np.array_equal(scales, whole.scales), k
        assert np.array_equal(err.view(np.uint32), whole.err.view(np.uint32)), k
        # every rank derived the same global scale from the all-reduced amax
        assert all(np.float32(p["G"]) == np.float32(whole.G) for p in parts)


def test_shard_plan_covers_rows():
    from paper_2605_12464_b200.dist import ShardPlan
    for rows in (1, 7, 128, 4097):
        for world in (1, 2, 3, 8):
            got = [ShardPlan([(rows, 16)], r, world).rows(0) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert all(lo <= hi for lo, hi in got)


def test_amax_groups_partition():
    """The grouped sharded step's groups cover every tensor once, in order,
    with <= 128 tensors each; the first is small (its amax is exposed)."""
    import ssgen
    from paper_2605_12464_b200.dist import amax_groups
    for numels in ([s.rows * s.cols for s in ssgen.workload("c2_qwen3_8b_weights")],
                   [s.rows * s.cols for s in ssgen.workload("c4_llama70b_kv")],
                   [7, 0, 3, 100, 5], [1, 1], [0, 0, 0]):
        g = amax_groups(numels)
        assert g[0][0] == 0 and g[-1][1] == len(numels)
        assert all(a[1] == b[0] for a, b in zip(g, g[1:]))
        assert all(0 < hi - lo <= 128 for lo, hi in g)
        if len(g) > 1 and sum(numels):
            assert sum(numels[g[0][0]:g[0][1]]) <= 0.5 * sum(numels) or g[0][1] - g[0][0] == 1
    assert amax_groups([5]) == [(0, 1)]
