"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds none of the method's arithmetic: it only draws random bf16
tensors with the shapes and value distributions of the paper's workloads
(recipe in DESIGN.md §6) and builds adversarial test blocks
from literal values.  Both sides (oracle tests and the product/bench) receive
the *same* tensor; neither computes anything here.

Determinism: a tensor is drawn in chunks of ``CHUNK_ROWS`` rows, chunk ``k`` of
tensor ``tid`` from a torch generator seeded with ``splitmix64(seed, tid, k)``,
so any contiguous row range (a row shard on one rank) is bitwise identical to
the same rows of the full tensor.  Per-tensor outlier channels come from a
separate seed and are therefore the same on every shard.
"""
from __future__ import annotations

import math

import torch

from .workloads import WORKLOADS, TensorSpec, workload  # noqa: F401

CHUNK_ROWS = 128
_MASK = (1 << 64) - 1


def splitmix64(*words: int) -> int:
    """Counter-based seed mixer (Steele et al. SplitMix64 finaliser)."""
    z = 0x9E3779B97F4A7C15
    for w in words:
        z = (z + (w & _MASK) + 0x9E3779B97F4A7C15) & _MASK
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        z = z ^ (z >> 31)
    return z & ((1 << 63) - 1)


def _outlier_channels(seed: int, tid: int, cols: int, count: int) -> torch.Tensor:
    g = torch.Generator(device="cpu")
    g.manual_seed(splitmix64(seed, tid, 0xC4A77E1))
    return torch.randperm(cols, generator=g)[:count]


def _draw(kind: str, n_rows: int, cols: int, g: torch.Generator, device) -> torch.Tensor:
    if kind in ("gaussian", "weight_outlier", "kv_k", "kv_v"):
        return torch.randn(n_rows, cols, generator=g, device=device, dtype=torch.float32)
    if kind == "student_t":
        # Student-t, nu = 3: Z / sqrt(chi2_3 / 3), chi2_3 = sum of 3 squared normals.
        z = torch.randn(n_rows, cols, generator=g, device=device, dtype=torch.float32)
        w = torch.randn(3, n_rows, cols, generator=g, device=device, dtype=torch.float32)
        chi = (w * w).sum(0) / 3.0
        return z / torch.sqrt(chi)
    raise ValueError("unknown kind %r" % kind)


# Per-kind (std, number of outlier channels as a function of cols, outlier gain).
def _kind_params(kind: str, cols: int):
    if kind == "gaussian":
        return 1.0, 0, 1.0
    if kind == "student_t":
        return 1.0, 8, 20.0  # 8 hidden channels x20
    if kind == "weight_outlier":
        return 0.02, max(4, cols // 1000), 50.0  # 0.1% of input columns x50 (C2)
    if kind == "kv_k":
        return 1.0, 4 * max(1, cols // 128), 10.0  # 4 of 128 channels x10 (C4 K)
    if kind == "kv_v":
        return 1.0, 0, 1.0
    raise ValueError(kind)


def generate(kind: str, rows: int, cols: int, seed: int, tid: int = 0,
             row_start: int = 0, row_end: int | None = None, device="cpu",
             out: torch.Tensor | None = None) -> torch.Tensor:
    """Rows [row_start, row_end) of synthetic tensor ``tid`` as bf16 (RNE from fp32)."""
    if row_end is None:
        row_end = rows
    assert 0 <= row_start <= row_end <= rows
    n = row_end - row_start
    if out is None:
        out = torch.empty(n, cols, dtype=torch.bfloat16, device=device)
    assert out.shape == (n, cols) and out.dtype == torch.bfloat16
    if n == 0:
        return out
    std, n_out, gain = _kind_params(kind, cols)
    chans = _outlier_channels(seed, tid, cols, n_out).to(out.device) if n_out else None
    g = torch.Generator(device=out.device)
    k0, k1 = row_start // CHUNK_ROWS, (row_end - 1) // CHUNK_ROWS
    for k in range(k0, k1 + 1):
        c_lo, c_hi = k * CHUNK_ROWS, min(rows, (k + 1) * CHUNK_ROWS)
        g.manual_seed(splitmix64(seed, tid, k))
        v = _draw(kind, c_hi - c_lo, cols, g, out.device)
        if std != 1.0:
            v.mul_(std)
        if chans is not None:
            v[:, chans] *= gain
        lo, hi = max(c_lo, row_start), min(c_hi, row_end)
        out[lo - row_start:hi - row_start].copy_(v[lo - c_lo:hi - c_lo])
    return out


def shard_rows(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of ``rank`` (ceil split; the last shard may be short)."""
    per = math.ceil(rows / world) if world > 0 else rows
    lo = min(rows, rank * per)
    return lo, min(rows, lo + per)


# ---------------------------------------------------------------------------
# Adversarial blocks (literal values; used by parity tests on both sides).
# ---------------------------------------------------------------------------
def adversarial_rows(seed: int = 7) -> torch.Tensor:
    """A [rows][64] bf16 tensor of hand-built corner-case blocks.

    Every row holds four 16-element blocks of one family: exact E2M1 midpoints
    times power-of-two and 1.5x scales, heavy ties, zeros and -0, bf16
    subnormals, blocks whose max-abs scale underflows to code 0, values that
    saturate code 126, single outliers, and representable blocks s*q.
    """
    g = torch.Generator().manual_seed(seed)
    mids = [0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0]
    grid = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]
    pw = [2.0 ** e for e in range(-12, 8)]
    rows = []

    def block(vals):
        v = list(vals)[:16]
        v += [0.0] * (16 - len(v))
        return v

    # 1. midpoints (with the max 6 pinned so c0 is an exact power of two)
    for p in pw:
        for sgn in (1.0, -1.0):
            b = [6.0 * p] + [sgn * m * p for m in mids] + [-m * p for m in mids] + [0.0]
            rows.append(block(b))
    # 2. representable blocks s*q, max|q| in {4, 6}
    for _ in range(64):
        e = int(torch.randint(-9, 8, (1,), generator=g))
        m = int(torch.randint(0, 8, (1,), generator=g))
        s = (1 + m / 8) * 2.0 ** e
        qmax = 4.0 if torch.rand(1, generator=g) < 0.5 else 6.0
        idx = torch.randint(0, 8, (16,), generator=g)
        q = [grid[int(i)] * (1 if torch.rand(1, generator=g) < 0.5 else -1) for i in idx]
        q = [min(abs(x), qmax) * (1 if x >= 0 else -1) for x in q]
        q[int(torch.randint(0, 16, (1,), generator=g))] = qmax
        rows.append(block([s * x for x in q]))
    # 3. zeros and negative zeros
    rows.append(block([0.0] * 16))
    rows.append(block([-0.0] * 16))
    rows.append(block([-0.0, 0.0] * 8))
    # 4. bf16 subnormals / tiny values (c0 == 0 and scale underflow)
    for e in (-133, -130, -126, -120, -20, -16, -14, -12, -11, -10):
        rows.append(block([2.0 ** e, -(2.0 ** e), 3 * 2.0 ** e] + [0.0] * 13))
    # 5. saturation and huge values
    for v in (448 * 6, 3072.0, 1e4, 1e6, 3.0e38, -3.0e38, 2.0 ** 100):
        rows.append(block([v, -v / 3, v / 7, 1.0]))
    # 6. single outliers among small values
    for p in (1e-3, 1.0, 100.0):
        b = (torch.randn(16, generator=g) * p * 1e-2).tolist()
        b[int(torch.randint(0, 16, (1,), generator=g))] = p * 37.0
        rows.append(block(b))
    # 7. constant blocks (ties between many scales)
    for v in (1.0, 0.75, 3.0, 5.0, 1e-3):
        rows.append(block([v] * 16))
        rows.append(block([v, -v] * 8))
    t = torch.tensor(rows, dtype=torch.float32)
    n = t.shape[0]
    pad = (-n) % 4
    if pad:
        t = torch.cat([t, torch.zeros(pad, 16)], 0)
    return t.reshape(-1, 64).to(torch.bfloat16)
