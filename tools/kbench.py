#!/usr/bin/env python
"""Kernel tuning sweep: time the batched amax and quantize launches of libss
builds (variants compiled with different -D flags) on a fixed synthetic batch.

    python tools/kbench.py build                 # here (CPU): compile the variants
    python tools/kbench.py run [--variants a,b]  # on the GPU box: one JSON line per case

Each variant runs in its own process (_binding.use_variant loads libss_<v>.so).
Timing: CUDA events on the launching stream, 3 warm-ups, median of 10; the
batch (first LAYERS layers of the Qwen3-8B workload, > 1 GB) exceeds L2.
Not the driver's bench: that is bench.py.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {
    "base": [],
    "noprune": ["SS_NO_PRUNE=1"],
    "count": ["SS_COUNT_EVALS=1"],
    "cilp1": ["SS_CILP=1"],
    "cilp3": ["SS_CILP=3"],
    "cilp4": ["SS_CILP=4"],
    "mb3": ["SS_MIN_BLOCKS=3"],
    "prune2": ["SS_PRUNE_FROM=2"],
    "prune4": ["SS_PRUNE_FROM=4"],
    # the library's former environment switches, now compile-time (A/B builds)
    "noamaxfusion": ["SS_AMAX_FUSION=0"],
    "norowfusion": ["SS_ROW_FUSION=0"],
    "rowupr1": ["SS_ROW_UPR=1"],
    "rowupr2": ["SS_ROW_UPR=2"],
    "rowupr4": ["SS_ROW_UPR=4"],
    "nosmall": ["SS_SMALL_MAX_BLOCKS=0"],
    "unrollu": ["SS_UNROLL_U=1"],
    "prmt": ["SS_PRMT_WIDEN=1"],
    "seg512": ["SS_SEG_TASKS=512"],
    "corex2": ["SS_CORE_REPEAT=1"],
    "notrail": ["SS_TRAIL_MIN_ELEMS=0"],
    "bpl1": ["SS_BPL=1"],
    "seg256": ["SS_SEG_TASKS=256"],
    "seg128": ["SS_SEG_TASKS=128"],
    "seg64": ["SS_SEG_TASKS=64"],
    "ipu1": ["SS_IPU_MAX=1"],
    "ipu2": ["SS_IPU_MAX=2"],
    "ipu8": ["SS_IPU_MAX=8"],
}
WINDOWS = [(0, 0), (-1, 1), (-2, 2), (-4, 4), (-2, 6), (-8, 8), (-16, 16), (-126, 126)]


def build(names):
    from paper_2605_12464_b200 import build as b
    for v in names:
        if v == "base":
            b.build()
        else:
            b.build(variant=v, defines=VARIANTS[v])
        print("built", v, flush=True)


def run_one(variant, layers, windows, reps, layout="linear"):
    import torch
    import ssgen
    from paper_2605_12464_b200 import _binding
    _binding.use_variant(variant)
    import paper_2605_12464_b200 as ss
    dev = torch.device("cuda", 0)
    specs = ssgen.workload("c2_qwen3_8b_weights")[: 7 * layers]
    xs = [ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid,
                         device=dev) for s in specs]
    n = sum(x.numel() for x in xs)
    outs = [ss.alloc_out(x, want_offsets=False, scale_layout=layout) for x in xs]
    amax = torch.zeros(len(xs), dtype=torch.int32, device=dev)

    def timed(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        return ts[len(ts) // 2]

    t_amax = timed(lambda: ss.tensor_amax_batched(xs, out=amax))
    print(json.dumps({"variant": variant, "kernel": "amax", "ms": t_amax, "elements": n,
                      "hbm_gbs": 2 * n / t_amax / 1e6}), flush=True)
    counting = variant == "count"
    if counting:
        import ctypes
        L = ss.lib()
        L.ss_debug_take_evals.restype = ctypes.c_ulonglong
    for fmin, fmax in windows:
        t = timed(lambda: ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode="device_amax",
                                              amax=amax, scale_layout=layout))
        line = {"variant": variant, "kernel": "quant", "layout": layout, "window": [fmin, fmax], "ms": t,
                "elements": n, "gelem_s": n / t / 1e6, "bf16_gbs": 2 * n / t / 1e6,
                "bytes_gbs": 3.0625 * n / t / 1e6}
        if counting:   # executed block-candidate evaluations per block (one pass)
            L.ss_debug_take_evals()
            ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode="device_amax", amax=amax,
                                scale_layout=layout)
            line["evaluated_per_block"] = L.ss_debug_take_evals() / (n / 16)
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["build", "run", "one"])
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--windows", default=None, help="e.g. -8:8,0:0")
    ap.add_argument("--layout", default="linear", choices=["linear", "swizzled"])
    a = ap.parse_args()
    names = a.variants.split(",")
    wins = WINDOWS if not a.windows else [tuple(int(v) for v in w.split(":"))
                                           for w in a.windows.split(",")]
    if a.mode == "build":
        build(names)
    elif a.mode == "one":
        run_one(names[0], a.layers, wins, a.reps, a.layout)
    else:
        for v in names:
            cmd = [sys.executable, __file__, "one", "--variants", v, "--layers", str(a.layers),
                   "--reps", str(a.reps), "--windows=" + ",".join("%d:%d" % w for w in wins),
                   "--layout", a.layout]
            subprocess.run(cmd, timeout=900)


if __name__ == "__main__":
    main()
