#!/usr/bin/env python
"""One C2 step as the trailing-amax chain (gmode tensor) and the same batches
searched with precomputed amaxes (gmode device_amax), for an ncu launch list:

    ncu --metrics gpu__time_duration.sum -k regex:quant_kernel --csv python tools/chainprof.py [--chain-only]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    from fusebench import trail_ends
    dev = torch.device("cuda", 0)
    specs = ssgen.workload("c2_qwen3_8b_weights")
    xs = [ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid, device=dev)
          for s in specs]
    outs = [ss.alloc_out(x) for x in xs]
    amax = ss.tensor_amax_batched(xs)
    ss.quantize_batched(xs, outs, fmin=-8, fmax=8, gmode="tensor")      # the chain
    ends = trail_ends([x.numel() for x in xs])
    print("elements", sum(x.numel() for x in xs))
    if "--chain-only" in sys.argv:
        torch.cuda.synchronize()
        print("ends", ends)
        return
    i0 = 0
    for e in ends:                                                        # the same batches, amax given
        ss.quantize_batched(xs[i0:e], outs[i0:e], fmin=-8, fmax=8, gmode="device_amax", amax=amax[i0:e])
        i0 = e
    torch.cuda.synchronize()
    print("ends", ends)


if __name__ == "__main__":
    main()
