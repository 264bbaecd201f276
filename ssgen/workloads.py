"""The five synthetic workloads of BASELINE.json ``configs``.

Shapes only; values come from ``ssgen.generate``.  Base seed 20261017.
"""
from __future__ import annotations

from dataclasses import dataclass

BASE_SEED = 20261017


@dataclass(frozen=True)
class TensorSpec:
    name: str
    rows: int
    cols: int
    kind: str
    tid: int

    @property
    def numel(self) -> int:
        return self.rows * self.cols


def _c1():
    # configs[0]: single 4096x4096 Gaussian bf16 matrix (P:287, P:512 setting).
    return [TensorSpec("gauss_4096x4096", 4096, 4096, "gaussian", 1)]


def _c2():
    # configs[1]: Qwen3-8B linear weights [out][in], 36 layers x 7 projections,
    # hidden 4096, 8 KV heads x 128 (k/v 1024 rows), intermediate 12288.
    shapes = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
              ("gate", 12288, 4096), ("up", 12288, 4096), ("down", 4096, 12288)]
    out = []
    for layer in range(36):
        for j, (nm, r, c) in enumerate(shapes):
            out.append(TensorSpec("L%02d.%s" % (layer, nm), r, c, "weight_outlier",
                                  1000 + layer * 16 + j))
    return out


def _c3():
    # configs[2]: dynamic activations 16384 tokens x 8192 hidden, Student-t nu=3.
    return [TensorSpec("act_16384x8192", 16384, 8192, "student_t", 3000)]


def _c4():
    # configs[3]: Llama-3.1-70B KV cache, 80 layers x 8 heads x 128 dim x 32k.
    # K as [L][H][T][D] -> per layer rows 8*32768, cols 128; V transposed
    # [L][H][D][T] -> per layer rows 8*128, cols 32768 (blocks along tokens).
    out = []
    for layer in range(80):
        out.append(TensorSpec("L%02d.K" % layer, 8 * 32768, 128, "kv_k", 4000 + 2 * layer))
        out.append(TensorSpec("L%02d.V" % layer, 8 * 128, 32768, "kv_v", 4001 + 2 * layer))
    return out


def _c5(gib: int = 1):
    # configs[4]: 1..8 GiB Gaussian; 1 GiB = 32768 x 16384 bf16.
    rows = {1: 32768, 2: 65536, 4: 65536, 8: 65536}[gib]
    cols = {1: 16384, 2: 16384, 4: 32768, 8: 65536}[gib]
    return [TensorSpec("gauss_%dGiB" % gib, rows, cols, "gaussian", 5000 + gib)]


WORKLOADS = {
    "c1_gauss4096": _c1,
    "c2_qwen3_8b_weights": _c2,
    "c3_act_student_t": _c3,
    "c4_llama70b_kv": _c4,
    "c5_gauss_1gib": lambda: _c5(1),
    "c5_gauss_2gib": lambda: _c5(2),
    "c5_gauss_4gib": lambda: _c5(4),
    "c5_gauss_8gib": lambda: _c5(8),
}


def workload(name: str):
    return WORKLOADS[name]()
