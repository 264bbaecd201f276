#!/usr/bin/env python
"""Call time vs tensor size for single-tensor quantize calls (the C1 regime).

    python tools/sizescale.py [--windows -8:8,0:0] [--gmode device_amax]

For 4096-column Gaussian bf16 tensors of 2^20 .. 2^26 elements: the median
CUDA-event time of `--calls` back-to-back calls (inputs rotated over copies so
the set exceeds L2), one JSON line per size and window.  A linear fit of time
against elements separates the per-call fixed cost (launch, ramp, tail, error
sums) from the throughput slope.
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
    ap.add_argument("--windows", default="-8:8,0:0")
    ap.add_argument("--gmode", default="device_amax", choices=["device_amax", "tensor"])
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--variant", default="base")
    ap.add_argument("--logmin", type=int, default=20)
    ap.add_argument("--logmax", type=int, default=26)
    a = ap.parse_args()
    from paper_2605_12464_b200 import _binding
    _binding.use_variant(a.variant)
    import torch
    import paper_2605_12464_b200 as ss
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    wins = [tuple(int(v) for v in w.split(":")) for w in a.windows.split(",")]
    res = []
    for lg in range(a.logmin, a.logmax + 1):
        n = 1 << lg
        rows = n // 4096
        copies = max(1, min(16, (1 << 29) // (2 * n)))
        xs = [torch.randn(rows, 4096, device=dev, generator=g).to(torch.bfloat16) for _ in range(copies)]
        outs = [ss.alloc_out(x, want_offsets=False) for x in xs]
        amax = torch.zeros(1, dtype=torch.int32, device=dev)
        ss.tensor_amax(xs[0], out=amax)
        for fmin, fmax in wins:
            def call(i):
                if a.gmode == "tensor":
                    ss.quantize_batched([xs[i % copies]], [outs[i % copies]], fmin=fmin, fmax=fmax, gmode="tensor")
                else:
                    ss.quantize_batched([xs[i % copies]], [outs[i % copies]], fmin=fmin, fmax=fmax,
                                        gmode="device_amax", amax=amax)
            for i in range(3):
                call(i)
            ts = []
            for rep in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for i in range(a.calls):
                    call(i)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / a.calls)
            t = sorted(ts)[len(ts) // 2]
            line = {"variant": a.variant, "gmode": a.gmode, "window": [fmin, fmax], "elements": n,
                    "us_per_call": 1e3 * t, "bf16_gbs": 2 * n / t / 1e6, "status": ss.device_status()}
            res.append(line)
            print(json.dumps(line), flush=True)
        del xs, outs
        torch.cuda.empty_cache()
    for fmin, fmax in wins:  # least-squares fit us = a + b * Melem over the sizes
        pts = [(r["elements"] / 1e6, r["us_per_call"]) for r in res if r["window"] == [fmin, fmax]]
        k = len(pts)
        sx = sum(p[0] for p in pts)
        sy = sum(p[1] for p in pts)
        sxx = sum(p[0] ** 2 for p in pts)
        sxy = sum(p[0] * p[1] for p in pts)
        b = (k * sxy - sx * sy) / (k * sxx - sx * sx)
        print(json.dumps({"fit": [fmin, fmax], "variant": a.variant, "gmode": a.gmode,
                          "fixed_us": (sy - b * sx) / k, "us_per_melem": b}), flush=True)


if __name__ == "__main__":
    main()
