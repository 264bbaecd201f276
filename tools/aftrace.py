#!/usr/bin/env python
"""Fused-amax timeline (tools only): one batched TENSOR-mode launch over the
first LAYERS layers of the C2 workload with a libss_<variant>.so built with
-DSS_AF_TRACE; prints when the amax warps finished relative to the launch and
the mean time a search warp spent waiting for an amax.

    python tools/aftrace.py build            # here: variants trace (1 amax warp), trace2 (2)
    python tools/aftrace.py run --variant trace
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {"trace": ["SS_AF_TRACE=1"], "trace2": ["SS_AF_TRACE=1", "SS_AMAX_WARPS=2"],
            "trace3": ["SS_AF_TRACE=1", "SS_AMAX_WARPS=3"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["build", "run"])
    ap.add_argument("--variant", default="trace")
    ap.add_argument("--layers", type=int, default=18)
    ap.add_argument("--windows", default="-8:8,-2:6,-2:2")
    ap.add_argument("--gmode", default="tensor", choices=["tensor", "device_amax"],
                    help="device_amax: the plain kernel after a separate amax launch (ncu A/B)")
    a = ap.parse_args()
    if a.mode == "build":
        from paper_2605_12464_b200 import build
        for v, d in VARIANTS.items():
            build.build(variant=v, defines=d)
        return
    from paper_2605_12464_b200 import _binding
    _binding.use_variant(a.variant)
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    L = ss.lib()
    dev = torch.device("cuda", 0)
    specs = ssgen.workload("c2_qwen3_8b_weights")[: 7 * a.layers]
    xs = [ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid, device=dev)
          for s in specs]
    outs = [ss.alloc_out(x) for x in xs]
    amax = ss.tensor_amax_batched(xs)
    trace = hasattr(L, "ss_debug_take_aftrace")
    buf = (ctypes.c_ulonglong * 4)()
    for w in a.windows.split(","):
        fmin, fmax = (int(v) for v in w.split(":"))
        for rep in range(3):
            if trace:
                L.ss_debug_take_aftrace(buf)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode=a.gmode, amax=amax)
            e1.record()
            torch.cuda.synchronize()
            if trace:
                L.ss_debug_take_aftrace(buf)
            t0, ta, wait, te = list(buf) if trace else (0, 0, 0, 0)
        grid_warps = 148 * 4 * 8
        print(json.dumps({"variant": a.variant, "window": [fmin, fmax], "tensors": len(xs),
                          "event_ms": e0.elapsed_time(e1), "kernel_ms": (te - t0) / 1e6,
                          "amax_done_ms": (ta - t0) / 1e6 if ta else None,
                          "mean_wait_ms_per_warp": wait / grid_warps / 1e6}), flush=True)


if __name__ == "__main__":
    main()
