#!/usr/bin/env python
"""One workload, one window, a few back-to-back quantize calls (for ncu captures).

    python tools/qone.py --workload c3_act_student_t --window=-1:1 [--gmode device_amax|tensor]
                         [--reps 3] [--fmt nvfp4]

The amax is computed once up front (device_amax mode), so with
`ncu -k regex:quant_kernel -s K -c 1` the capture is the search kernel alone.
Prints one JSON line per call with its CUDA-event time (not a bench number
when run under ncu).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_act_student_t")
    ap.add_argument("--window", default="-8:8")
    ap.add_argument("--gmode", default="device_amax", choices=["device_amax", "tensor", "none"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fmt", default="nvfp4")
    ap.add_argument("--tensors", type=int, default=0, help="first N tensors only (0 = all)")
    ap.add_argument("--variant", default="base", help="libss_<variant>.so (tools/kbench.py build)")
    a = ap.parse_args()
    import torch
    import ssgen
    if a.variant != "base":
        from paper_2605_12464_b200 import _binding
        _binding.use_variant(a.variant)
    import paper_2605_12464_b200 as ss
    fmin, fmax = (int(v) for v in a.window.split(":"))
    dev = torch.device("cuda", 0)
    specs = ssgen.workload(a.workload)
    if a.tensors:
        specs = specs[: a.tensors]
    xs = [ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid, device=dev)
          for s in specs]
    outs = [ss.alloc_out(x, want_offsets=False, fmt=a.fmt) for x in xs]
    amax = ss.tensor_amax_batched(xs)
    n = sum(x.numel() for x in xs)
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode=a.gmode,
                            amax=amax if a.gmode == "device_amax" else None, fmt=a.fmt)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"workload": a.workload, "window": [fmin, fmax], "gmode": a.gmode, "ms": ms,
                          "elements": n, "bf16_gbs": 2 * n / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
