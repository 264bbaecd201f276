"""Row-shard driver: one process per GPU, rows of every tensor split across ranks.

SURVEY.md §8(e): blocks never straddle rows, so contiguous row shards are
independent given the per-tensor global scale G, whose only input is the
tensor amax.  One exchange step exists: a max all-reduce of the shard amaxes
(u32 FP32 bit patterns; max is exact and order-free, so every rank derives
the same G and the sharded outputs are bitwise the unsharded ones).  All the
amaxes of a step travel in ONE all-reduce (4 B per tensor) over NCCL/NVLink.

The driver only sequences calls; the arithmetic is in libss.so.  ``ops`` is
pluggable so the host logic can be exercised on CPU with the gloo backend
(tests/test_dist_gloo.py): the product uses ``CudaOps``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch


def shard_rows(rows: int, rank: int, world: int) -> tuple:
    """Contiguous ceil-split of [0, rows); the last shards may be short or empty."""
    per = math.ceil(rows / world) if world > 0 else rows
    lo = min(rows, rank * per)
    return lo, min(rows, lo + per)


def amax_fused(shapes: Sequence[tuple], fmin: int, fmax: int) -> bool:
    """Whether libss runs the amax inside the quantize launch for a TENSOR-mode
    NVFP4 batch of these (rows, cols) shapes (asked from the library:
    ss_quantize_plan, so no rule is duplicated here)."""
    from . import _binding as B
    return bool(B.plan(list(shapes), fmin=fmin, fmax=fmax, gmode="tensor").amax_fused)


def amax_groups(numels: Sequence[int], fractions=(0.04, 0.2), max_group: int = 128) -> List[tuple]:
    """Contiguous tensor groups for the grouped sharded step: the first holds
    >= 4 % of the elements (its amax is exposed), the second reaches 20 %
    (its amax runs under the first group's search), the rest follow in
    groups of <= 128 tensors (the amax of each under the previous search;
    the search costs ~4x the amax per element at r = 8)."""
    total = sum(numels)
    if total == 0 or len(numels) < 2:
        return [(0, len(numels))]
    bounds, lo, acc = [], 0, 0
    for f in fractions:
        hi = lo
        while hi < len(numels) and (acc + numels[hi] < f * total or hi == lo) and hi - lo < max_group:
            acc += numels[hi]
            hi += 1
        if hi >= len(numels):
            break
        bounds.append((lo, hi))
        lo = hi
    while lo < len(numels):
        hi = min(len(numels), lo + max_group)
        bounds.append((lo, hi))
        lo = hi
    return bounds


class CudaOps:
    """libss.so batched calls on the current CUDA stream.  Sharded (N > 1):
    one amax launch and one quantize launch per 128 tensors of a step, the
    all-reduce between them.  Unsharded: ``quantize_local`` — one fused
    amax + quantize launch per 128 tensors (SS_GLOBAL_TENSOR)."""

    def __init__(self, fmin: int, fmax: int, want_err: bool = True, want_sums: bool = True,
                 want_offsets: bool = False):
        from . import _binding as B
        self.B = B
        self.fmin, self.fmax = fmin, fmax
        self.want_err, self.want_sums, self.want_offsets = want_err, want_sums, want_offsets

    def new_amax(self, n: int, device) -> torch.Tensor:
        return torch.zeros(n, dtype=torch.int32, device=device)

    def amax_all(self, xs, buf) -> int:
        self.B.tensor_amax_batched(xs, out=buf)
        return (len(xs) + 127) // 128

    def alloc_out(self, x: torch.Tensor):
        return self.B.alloc_out(x, self.want_err, self.want_offsets, self.want_sums, True)

    def quantize_local(self, xs, outs) -> int:
        """Whole tensors on this device: per-tensor amax inside the quantize launch."""
        live = [k for k, x in enumerate(xs) if x.shape[0] > 0]
        self.B.quantize_batched([xs[k] for k in live], [outs[k] for k in live], fmin=self.fmin,
                                fmax=self.fmax, gmode="tensor")
        p = self.B.plan([tuple(xs[k].shape) for k in live], fmin=self.fmin, fmax=self.fmax, gmode="tensor",
                        want_err=self.want_err, want_sums=self.want_sums)
        return p.launches

    def quantize_next_amax(self, xs, buf, outs, next_xs, next_buf) -> int:
        """Quantize ``xs`` (all-reduced amaxes in ``buf``) and, in the same launch,
        the local amaxes of ``next_xs`` into ``next_buf`` (ss_quantize_nvfp4_batched_next_amax)."""
        live = [k for k, x in enumerate(xs) if x.shape[0] > 0]
        self.B.quantize_batched_next_amax([xs[k] for k in live], [outs[k] for k in live],
                                          buf if len(live) == len(xs) else buf[live].contiguous(),
                                          next_xs, next_buf, fmin=self.fmin, fmax=self.fmax)
        launches = (len(live) + 127) // 128
        return launches * (2 if self.want_sums else 1) + (0 if live else 1)

    def quantize_all(self, xs, buf, outs) -> int:
        live = [k for k, x in enumerate(xs) if x.shape[0] > 0]
        self.B.quantize_batched([xs[k] for k in live], [outs[k] for k in live], fmin=self.fmin,
                                fmax=self.fmax, gmode="device_amax",
                                amax=buf if len(live) == len(xs) else buf[live].contiguous())
        launches = (len(live) + 127) // 128
        return launches * (2 if self.want_sums else 1)  # quant_kernel (+ sums_kernel)


class PeerExchange:
    """Every rank's amax exchange buffer mapped into this process (CUDA IPC
    over NVLink/NVSwitch).  The handles travel once through
    ``group`` (any backend); after that no step uses the host or a collective."""

    def __init__(self, group, rank: int, world: int, max_tensors: int, max_groups: int):
        from . import _binding as B
        self.B = B
        self.own = B.exchange_alloc(max_tensors, max_groups)
        ptrs, self.opened = [0] * world, []
        ptrs[rank] = self.own
        if world > 1:
            import torch.distributed as dist
            hs = [None] * world
            dist.all_gather_object(hs, B.ipc_handle(self.own), group=group)
            for r in range(world):
                if r != rank:
                    ptrs[r] = B.ipc_open(hs[r])
                    self.opened.append(ptrs[r])
            dist.barrier(group=group)
        self.x = B.make_exchange(world, rank, ptrs, max_tensors, max_groups)
        self.epoch = 0

    def close(self, group=None):
        for p in self.opened:
            self.B.ipc_close(p)
        if self.opened:  # no rank frees its buffer while a peer may still map it
            import torch.distributed as dist
            dist.barrier(group=group)
        self.opened = []
        if self.own:
            self.B.exchange_free(self.own)
            self.own = 0


@dataclass
class ShardPlan:
    shapes: Sequence[tuple]          # full (rows, cols) of every tensor
    rank: int
    world: int

    def rows(self, k: int) -> tuple:
        return shard_rows(self.shapes[k][0], self.rank, self.world)

    def local_numel(self) -> int:
        return sum((hi - lo) * c for (lo, hi), (_, c) in
                   ((self.rows(k), s) for k, s in enumerate(self.shapes)))


class RowShardQuantizer:
    """Quantize a list of tensors whose rows are sharded over ``world`` ranks."""

    EXCHANGES = ("grouped", "single", "peer")

    def __init__(self, plan: ShardPlan, ops, group=None, device=None, pipeline_groups: int = 1,
                 collective: bool | None = None, exchange: str = "grouped"):
        """``exchange`` (sharded steps): "single" = the north star's one max
        all-reduce of every tensor's amax per step (amax launch -> all-reduce ->
        quantize launch); "grouped" = the same exchange cut into tensor groups
        so that each group's amax runs inside the previous group's quantize
        launch (a few all-reduces per step, only the first amax exposed).
        "peer" = the grouped step with the all-reduces replaced by the
        peer-memory exchange (CUDA IPC buffers; each quantize launch reads
        its group's amaxes from every rank and publishes the next group's,
        DESIGN.md §5b): no host round trip or collective per group.
        Outputs are bit-identical either way."""
        if exchange not in self.EXCHANGES:
            raise ValueError("exchange must be one of %s" % (self.EXCHANGES,))
        self.plan, self.ops, self.group = plan, ops, group
        self.exchange = exchange
        # the amax all-reduce runs whenever ranks > 1 (or when forced, to test it with one rank)
        self.collective = plan.world > 1 if collective is None else collective
        self.allreduces = 0   # all-reduces issued by the last step
        self.amax_buf = ops.new_amax(len(plan.shapes), device)
        self.pipeline_groups = pipeline_groups
        self._side = None
        self.groups = amax_groups([r * c for r, c in plan.shapes])
        self.peer = None
        if exchange == "peer" and self.collective:
            self.peer = PeerExchange(group, plan.rank, plan.world, max(len(plan.shapes), 1),
                                     max(len(self.groups), 1))

    def close(self):
        if self.peer is not None:
            self.peer.close(self.group)
            self.peer = None

    def step(self, shards: List[torch.Tensor], outs: List, hooks=None) -> int:
        """One pass over every tensor; returns the number of kernels launched.

        N > 1: shard amaxes (one batched launch) -> the one exchange step (ONE
        max all-reduce of all the amaxes, 4 B per tensor) -> batched quantize.
        N = 1 (no collective): ``ops.quantize_local`` when the ops have it —
        the amax runs inside the quantize launch.
        N = 1 with pipeline_groups > 1: the tensors are cut into groups; the
        amax of every group is launched on a side stream up front and group k's
        quantize waits only for group k's amax, so the HBM-bound amax pass runs
        under the ALU-bound quantize (same results).  Measured on C2: 2 % less
        time per step, but the co-running amax slows the quantize kernel by
        ~10 %, so the default keeps the two passes sequential.  ``hooks`` (optional) has ``before()`` /
        ``after()`` called around each quantize call (bench.py records CUDA
        events there).
        """
        import torch.distributed as dist
        self.allreduces = 0
        if not self.collective and self.pipeline_groups <= 1 and hasattr(self.ops, "quantize_local"):
            # unsharded: the amax inside the quantize launches (one per 128 tensors,
            # or the trailing-amax chain of DESIGN.md §4.2c)
            if hooks is not None:
                hooks.before()
            n = self.ops.quantize_local(shards, outs)
            if hooks is not None:
                hooks.after()
            return n
        if not self.collective and self.pipeline_groups > 1 and torch.cuda.is_available() \
                and len(shards) > 1 and shards[0].is_cuda:
            return self._pipelined(shards, outs, hooks)
        if self.collective and self.exchange == "peer":
            return self._peer(shards, outs, hooks)
        if self.collective and self.exchange == "grouped" and len(self.groups) > 1 and \
                hasattr(self.ops, "quantize_next_amax"):
            return self._grouped(shards, outs, hooks)
        n = self.ops.amax_all(shards, self.amax_buf)
        if self.collective:   # the one exchange step: every tensor's amax in ONE all-reduce
            dist.all_reduce(self.amax_buf, op=dist.ReduceOp.MAX, group=self.group)
            self.allreduces = 1
        if hooks is not None:
            hooks.before()
        n += self.ops.quantize_all(shards, self.amax_buf, outs)
        if hooks is not None:
            hooks.after()
        return n

    def _grouped(self, shards, outs, hooks) -> int:
        """Sharded step in groups: amax(g0) -> all-reduce(g0) -> [quantize(g_k) with
        the local amax of g_{k+1} inside the same launch -> all-reduce(g_{k+1})]* ->
        quantize(g_last).  Only the first group's amax pass is exposed."""
        import torch.distributed as dist
        buf, gs = self.amax_buf, self.groups
        lo, hi = gs[0]
        n = self.ops.amax_all(shards[lo:hi], buf[lo:hi])
        dist.all_reduce(buf[lo:hi], op=dist.ReduceOp.MAX, group=self.group)
        self.allreduces = len(gs)
        for k, (lo, hi) in enumerate(gs):
            if hooks is not None:
                hooks.before()
            if k + 1 < len(gs):
                nlo, nhi = gs[k + 1]
                n += self.ops.quantize_next_amax(shards[lo:hi], buf[lo:hi], outs[lo:hi],
                                                 shards[nlo:nhi], buf[nlo:nhi])
            else:
                n += self.ops.quantize_all(shards[lo:hi], buf[lo:hi], outs[lo:hi])
            if hooks is not None:
                hooks.after()
            if k + 1 < len(gs):
                dist.all_reduce(buf[nlo:nhi], op=dist.ReduceOp.MAX, group=self.group)
        return n

    def _peer(self, shards, outs, hooks) -> int:
        """Grouped step over the peer-memory exchange: amax(g0) -> publish(g0)
        -> [quantize(g_k) reading every rank's g_k amaxes, computing and
        publishing the local g_{k+1} amaxes in the same launch]*.  The host
        only enqueues; ranks synchronise through flag words in device memory."""
        B, P, buf, gs = self.ops.B, self.peer, self.amax_buf, self.groups
        P.epoch += 1
        lo, hi = gs[0]
        n = self.ops.amax_all(shards[lo:hi], buf[lo:hi])
        B.exchange_publish(P.x, lo, 0, P.epoch, buf[lo:hi])
        n += 1
        for k, (lo, hi) in enumerate(gs):
            if hooks is not None:
                hooks.before()
            nxt = gs[k + 1] if k + 1 < len(gs) else None
            B.quantize_exchange(shards[lo:hi], outs[lo:hi], P.x, lo, k, P.epoch,
                                next_xs=shards[nxt[0]:nxt[1]] if nxt else None,
                                next_amax=buf[nxt[0]:nxt[1]] if nxt else None,
                                next_slot0=nxt[0] if nxt else 0, fmin=self.ops.fmin, fmax=self.ops.fmax)
            if hooks is not None:
                hooks.after()
            n += (1 + (1 if self.ops.want_sums else 0)) * ((hi - lo + 127) // 128)
        return n

    def _pipelined(self, shards, outs, hooks) -> int:
        main = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream(device=shards[0].device)
        side = self._side
        T = len(shards)
        per = -(-T // min(self.pipeline_groups, T))
        bounds = [(k, min(T, k + per)) for k in range(0, T, per)]
        side.wait_stream(main)          # amax slots are free once the previous step is done
        events, n = [], 0
        with torch.cuda.stream(side):
            for lo, hi in bounds:
                n += self.ops.amax_all(shards[lo:hi], self.amax_buf[lo:hi])
                events.append(side.record_event())
        for (lo, hi), ev in zip(bounds, events):
            main.wait_event(ev)
            if hooks is not None:
                hooks.before()
            n += self.ops.quantize_all(shards[lo:hi], self.amax_buf[lo:hi], outs[lo:hi])
            if hooks is not None:
                hooks.after()
        return n
