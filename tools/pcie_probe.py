#!/usr/bin/env python
"""PCIe probe (tools only): pinned host <-> device copy bandwidth alone and
with both directions at once, to bound bench.py's e2e leg."""
import json
import torch

dev = torch.device("cuda", 0)
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n // 2, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device=dev)
d_out = torch.empty(n // 2, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_gbs": n / t1 / 1e6, "d2h_gbs": (n // 2) / t2 / 1e6,
                  "both_ms": t3, "both_h2d_gbs_if_h2d_bound": n / t3 / 1e6,
                  "bytes_h2d": n, "bytes_d2h": n // 2}))
