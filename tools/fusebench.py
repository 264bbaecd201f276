#!/usr/bin/env python
"""A/B of the fused amax (quant_kernel<..., AF>) against the
separate amax launch, on the bench workloads.

    python tools/fusebench.py [--configs c1_gauss4096,c2_qwen3_8b_weights] [--windows -8:8,0:0]

Per config and window, one JSON line with the median time (CUDA events, 3
warm-ups, `--reps` timed calls; inputs rotated over copies when the workload
fits in L2) of
  sep    ss_tensor_amax_batched + ss_quantize_nvfp4_batched(DEVICE_AMAX)
  search ss_quantize_nvfp4_batched(DEVICE_AMAX) alone (workloads over L2 only)
  fused  ss_quantize_nvfp4_batched(TENSOR)   (amax units inside the launch)
and whether the fused outputs (codes, scales, errors, sums, G) equal the
separate path's bit for bit.  --variant noamaxfusion (a build with
-DSS_AMAX_FUSION=0, tools/kbench.py build) times the TENSOR call without fusion.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def trail_ends(ns, max_tensors=64):
    """The library's trailing-amax batches (ss_api.cu trail_batches)."""
    n_all = sum(ns)
    lim = max(n_all // 64, 1)
    ends, i = [], 0
    while i < len(ns):
        el = nt = 0
        while i < len(ns) and nt < max_tensors:
            if nt > 0 and (el + ns[i] > lim or el + ns[i] > (1 << 36)):
                break
            el += ns[i]
            nt += ns[i] > 0
            i += 1
        ends.append(i)
        lim = 2 * max(el, 1)
    return ends


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1_gauss4096,c2_qwen3_8b_weights,c4_llama70b_kv")
    ap.add_argument("--windows", default="-8:8,0:0")
    ap.add_argument("--variant", default="base")
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    from paper_2605_12464_b200 import _binding
    _binding.use_variant(a.variant)
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    dev = torch.device("cuda", 0)
    wins = [tuple(int(v) for v in w.split(":")) for w in a.windows.split(",")]
    for cfg in a.configs.split(","):
        specs = ssgen.workload(cfg)
        xs = [ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid,
                             device=dev) for s in specs]
        n = sum(x.numel() for x in xs)
        copies = max(1, min(40, (1 << 30) // (2 * n)))
        sets = [xs] + [[x.clone() for x in xs] for _ in range(copies - 1)]
        outs_a = [ss.alloc_out(x, want_offsets=True) for x in xs]
        outs_b = [ss.alloc_out(x, want_offsets=True) for x in xs]
        amax = torch.zeros(len(xs), dtype=torch.int32, device=dev)

        def timed(fn):
            for i in range(3):
                fn(sets[i % copies])
            ts = []
            for i in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(sets[i % copies])
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return sorted(ts)[len(ts) // 2]

        for fmin, fmax in wins:
            def sep(s):
                ss.tensor_amax_batched(s, out=amax)
                ss.quantize_batched(s, outs_a, fmin=fmin, fmax=fmax, gmode="device_amax", amax=amax)

            def fused(s):
                ss.quantize_batched(s, outs_b, fmin=fmin, fmax=fmax, gmode="tensor")

            def search(s):  # the quantize launches alone (amax precomputed by sep)
                ss.quantize_batched(s, outs_a, fmin=fmin, fmax=fmax, gmode="device_amax", amax=amax)

            t_sep = timed(sep)
            t_fused = timed(fused)
            t_search = timed(search) if copies == 1 else None
            # the search alone in the launch structure of the trailing-amax chain
            pl = ss.plan([tuple(x.shape) for x in xs], fmin=fmin, fmax=fmax, gmode="tensor")
            t_search_chain = None
            if copies == 1 and pl.trail_batches > 1:
                ends = trail_ends([x.numel() for x in xs])

                def search_chain(s):
                    i0 = 0
                    for e in ends:
                        ss.quantize_batched(s[i0:e], outs_a[i0:e], fmin=fmin, fmax=fmax, gmode="device_amax",
                                            amax=amax[i0:e])
                        i0 = e
                t_search_chain = timed(search_chain)
            sep(xs)
            fused(xs)
            torch.cuda.synchronize()
            same = all(torch.equal(getattr(oa, f), getattr(ob, f))
                       for oa, ob in zip(outs_a, outs_b)
                       for f in ("codes", "scales", "err", "offsets", "sums", "G")
                       if getattr(oa, f) is not None)
            print(json.dumps({"config": cfg, "window": [fmin, fmax], "tensors": len(xs), "elements": n,
                              "variant": a.variant,
                              "sep_ms": t_sep, "fused_ms": t_fused, "search_only_ms": t_search, "search_chain_ms": t_search_chain, "speedup": t_sep / t_fused,
                              "sep_gbs": 2 * n / t_sep / 1e6, "fused_gbs": 2 * n / t_fused / 1e6,
                              "bit_identical": bool(same),
                              "status": ss.device_status()}), flush=True)
        del xs, sets, outs_a, outs_b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
