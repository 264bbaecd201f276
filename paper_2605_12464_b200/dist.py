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


class CudaOps:
    """libss.so calls on the current CUDA stream."""

    def __init__(self, fmin: int, fmax: int, want_err: bool = True, want_sums: bool = True,
                 want_offsets: bool = False):
        from . import _binding as B
        self.B = B
        self.fmin, self.fmax = fmin, fmax
        self.want_err, self.want_sums, self.want_offsets = want_err, want_sums, want_offsets

    def new_amax(self, n: int, device) -> torch.Tensor:
        return torch.zeros(n, dtype=torch.int32, device=device)

    def amax(self, x: torch.Tensor, slot: torch.Tensor):
        self.B.tensor_amax(x, out=slot)

    def alloc_out(self, x: torch.Tensor):
        rows, cols = x.shape
        nb = rows * cols // 16
        d = x.device
        return self.B.QuantOut(
            torch.empty(rows, cols // 2, dtype=torch.uint8, device=d),
            torch.empty(rows, cols // 16, dtype=torch.uint8, device=d),
            torch.empty(nb, 2, dtype=torch.float32, device=d) if self.want_err else None,
            torch.empty(nb, dtype=torch.int8, device=d) if self.want_offsets else None,
            torch.empty(2, dtype=torch.float64, device=d) if self.want_sums else None,
            torch.empty(1, dtype=torch.float32, device=d),
        )

    def quantize_given(self, x, slot, out):
        self.B.quantize(x, fmin=self.fmin, fmax=self.fmax, gmode="device_amax", amax=slot, out=out)

    def quantize_tensor(self, x, out):
        self.B.quantize(x, fmin=self.fmin, fmax=self.fmax, gmode="tensor", out=out)

    launches_amax = 1        # amax_kernel
    launches_quant = 1       # quant_kernel (sums reduced by its last CTA)
    launches_sums = 0


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

    def __init__(self, plan: ShardPlan, ops, group=None, device=None):
        self.plan, self.ops, self.group = plan, ops, group
        self.amax_buf = ops.new_amax(len(plan.shapes), device)

    def step(self, shards: List[torch.Tensor], outs: List, hooks=None) -> int:
        """One pass over every tensor; returns the number of kernels launched.

        ``hooks`` (optional) has ``before(k)`` / ``after(k)`` called around the
        quantize launch of tensor k (bench.py records CUDA events there).
        """
        import torch.distributed as dist
        n = 0
        if self.plan.world == 1:
            # single GPU: amax then quantize per tensor, so the second read of
            # each tensor (<= 100 MB) is served from the 126 MB L2
            for k, (x, o) in enumerate(zip(shards, outs)):
                if x.shape[0] == 0:
                    continue
                self.ops.amax(x, self.amax_buf[k:k + 1])
                n += self._quant(k, x, o, hooks) + self.ops.launches_amax
            return n
        for k, x in enumerate(shards):
            if x.shape[0] > 0:
                self.ops.amax(x, self.amax_buf[k:k + 1])
                n += self.ops.launches_amax
            else:
                self.amax_buf[k:k + 1].zero_()
        # the one exchange step: max of the shard amaxes of all tensors at once
        dist.all_reduce(self.amax_buf, op=dist.ReduceOp.MAX, group=self.group)
        for k, (x, o) in enumerate(zip(shards, outs)):
            if x.shape[0] > 0:
                n += self._quant(k, x, o, hooks)
        return n

    def _quant(self, k, x, o, hooks) -> int:
        if hooks is not None:
            hooks.before(k)
        self.ops.quantize_given(x, self.amax_buf[k:k + 1], o)
        if hooks is not None:
            hooks.after(k)
        return self.ops.launches_quant
