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
        self.nonfinite = set()     # tensors whose all-reduced amax was NaN/Inf (the library's flag)

    def new_amax(self, n, device):
        return torch.zeros(n, dtype=torch.int32)

    def amax_all(self, xs, buf):
        for k, x in enumerate(xs):
            if not x.numel():
                buf[k] = 0
            elif not torch.isfinite(x.float()).all():
                buf[k] = 0x7FC00000           # |NaN| bits sort above every finite value (R14)
            else:
                buf[k] = self.o.tensor_amax(x)
        return 1

    def alloc_out(self, x):
        return {}

    def quantize_next_amax(self, xs, buf, outs, next_xs, next_buf):
        # the grouped step's fused call: quantize this group, local amaxes of the next
        self.amax_all(next_xs, next_buf)
        return self.quantize_all(xs, buf, outs)

    def quantize_all(self, xs, buf, outs):
        for x, slot, out in zip(xs, buf, outs):
            bits = int(slot.item()) & 0xFFFFFFFF
            out["amax_bits"] = bits
            if x.shape[0] == 0:
                continue
            if bits >= 0x7F800000:            # the library: sticky flag, G = 1 (R14)
                out["nonfinite"] = True
                out["G"] = 1.0
                continue
            r = self.o.quantize(x, x.shape[0], x.shape[1], FMIN, FMAX, "given", amax_bits=bits)
            out.update(codes=r.codes, scales=r.scales, err=r.err, G=r.G)
        return 1


def _tensors():
    return [ssgen.generate("weight_outlier" if k % 2 else "student_t", r, c, seed=11, tid=k)
            for k, (r, c) in enumerate(SHAPES)]


def _worker(rank, world, port, q, exchange="grouped", nan_at=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_12464_b200.dist import RowShardQuantizer, ShardPlan
        full = _tensors()
        plan = ShardPlan(SHAPES, rank, world)
        shards = [x[slice(*plan.rows(k))].contiguous() for k, x in enumerate(full)]
        if nan_at is not None and nan_at[0] == rank:       # fault injection on ONE rank's shard
            k, r, c = nan_at[1:]
            shards[k][r, c] = float("nan")
        ops = OracleOps()
        outs = [ops.alloc_out(x) for x in shards]
        qz = RowShardQuantizer(plan, ops, group=None, device="cpu", exchange=exchange)
        n = qz.step(shards, outs)
        assert qz.allreduces == (1 if exchange == "single" else len(qz.groups))
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


def _run(world, exchange="grouped", nan_at=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, exchange, nan_at)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    t0 = time.time()
    while True:                     # fail fast if a worker dies instead of waiting out the timeout
        try:
            n, gathered = q.get(timeout=2)
            break
        except queue.Empty:
            assert all(p.exitcode in (None, 0) for p in procs), [p.exitcode for p in procs]
            assert time.time() - t0 < 300
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return n, gathered


@pytest.mark.parametrize("world,exchange", [(2, "grouped"), (3, "grouped"), (2, "single"), (3, "single")])
def test_row_shards_equal_whole_tensor(oracle_lib, world, exchange):
    n, gathered = _run(world, exchange)
    assert n > 0
    for k, x in enumerate(_tensors()):
        whole = oracle_lib.quantize(x, x.shape[0], x.shape[1], FMIN, FMAX, "tensor")
        parts = [g[k] for g in gathered if "codes" in g[k]]
        codes = np.concatenate([p["codes"] for p in parts], 0)
        scales = np.concatenate([p["scales"] for p in parts], 0)
        err = np.concatenate([p["err"] for p in parts], 0)
        assert np.array_equal(codes, whole.codes), k
        assert np.array_equal(scales, whole.scales), k
        assert np.array_equal(err.view(np.uint32), whole.err.view(np.uint32)), k
        # every rank derived the same global scale from the all-reduced amax
        assert all(np.float32(p["G"]) == np.float32(whole.G) for p in parts)


@pytest.mark.parametrize("exchange", ["grouped", "single"])
def test_nan_on_one_rank_flags_every_rank(oracle_lib, exchange):
    """SURVEY §5 fault injection: a NaN in ONE rank's shard of tensor 3 reaches
    every rank through the max all-reduce of the amax bit patterns (NaN bits
    sort above every finite value, R14): every rank's slot for that tensor is
    non-finite, so each flags it and uses G = 1; the other tensors are
    untouched and still equal the whole-tensor quantization."""
    world = 2
    n, gathered = _run(world, exchange, nan_at=(1, 3, 8, 7))    # rank 1 holds rows 32..63 of tensor 3
    for g in gathered:
        assert g[3]["amax_bits"] >= 0x7F800000
        if "codes" in g[3] or g[3].get("nonfinite"):
            assert g[3].get("nonfinite") and g[3]["G"] == 1.0
    for k, x in enumerate(_tensors()):
        if k == 3:
            continue
        whole = oracle_lib.quantize(x, x.shape[0], x.shape[1], FMIN, FMAX, "tensor")
        parts = [g[k] for g in gathered if "codes" in g[k]]
        assert np.array_equal(np.concatenate([p["codes"] for p in parts], 0), whole.codes), k
        assert all(g[k]["amax_bits"] == whole_amax(oracle_lib, x) for g in gathered)


def whole_amax(o, x):
    return o.tensor_amax(x)


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
