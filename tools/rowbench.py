#!/usr/bin/env python
"""Per-row global scale (SS_GLOBAL_ROW) timing on one B200: row-fused quantize
vs the two-pass path (SS_ROW_FUSION=0: rowscale kernel, then quantize), and the
per-tensor path with a precomputed amax (the quantize pass alone) as the floor.

    python tools/rowbench.py [--out gpurun_out/rowbench.jsonl]

Shapes: C3 (16384 x 8192 Student-t activations, configs[2]) and a 4096-hidden
activation batch (32768 x 4096).  Each setting runs in its own process (the
fusion switch is read once per process).  Timing: CUDA events around `reps`
back-to-back calls after 2 warm-ups; both inputs exceed L2.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess

VARIANT = "base"
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"c3_act_16384x8192": (16384, 8192), "act_32768x4096": (32768, 4096)}
RADII = [0, 1, 2, 4, 8]


def one(mode, reps):
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    dev = torch.device("cuda", 0)
    for name, (rows, cols) in SHAPES.items():
        x = ssgen.generate("student_t", rows, cols, seed=ssgen.workloads.BASE_SEED, tid=3000, device=dev)
        gm = "device_amax" if mode == "tensor" else "row"
        out = ss.alloc_out(x, want_offsets=False, gmode=gm)
        amax = torch.zeros(1, dtype=torch.int32, device=dev)
        ss.tensor_amax_batched([x], out=amax)
        for r in RADII:
            def call():
                if gm == "row":
                    ss.quantize(x, radius=r, gmode="row", out=out)
                else:
                    ss.quantize(x, radius=r, gmode="device_amax", amax=amax, out=out)
            for _ in range(2):
                call()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                call()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            print(json.dumps({"shape": name, "mode": mode, "radius": r, "ms": ms,
                              "bf16_gbs": 2 * x.numel() / ms / 1e6,
                              "variant": VARIANT}), flush=True)
        del x, out
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--one", default=None)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--variant", default="base")
    a = ap.parse_args()
    global VARIANT
    VARIANT = a.variant
    from paper_2605_12464_b200 import _binding
    _binding.use_variant(a.variant)
    if a.one:
        one(a.one, a.reps)
        return
    # A/B builds from tools/kbench.py build --variants norowfusion,rowupr1,rowupr2,rowupr4
    runs = [("row_fused", "base"), ("row_twopass", "norowfusion"), ("tensor", "base"),
            ("row_fused", "rowupr1"), ("row_fused", "rowupr2"), ("row_fused", "rowupr4")]
    lines = []
    for mode, var in runs:
        r = subprocess.run([sys.executable, __file__, "--one", mode, "--reps", str(a.reps), "--variant", var],
                           capture_output=True, text=True, timeout=900)
        sys.stderr.write(r.stderr[-2000:])
        for ln in r.stdout.splitlines():
            print(ln, flush=True)
            lines.append(ln)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
