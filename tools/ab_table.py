#!/usr/bin/env python
"""Summarise tools/ab.sh output: median ms per (workload, window, variant)."""
import json
import sys
from collections import defaultdict


def main(tag):
    d = defaultdict(list)
    for fn, kind in (("gpurun_out/kbench_%s.jsonl" % tag, "c2x4"), ("gpurun_out/qone_%s.jsonl" % tag, "c5_1g")):
        try:
            for ln in open(fn):
                if not ln.strip():
                    continue
                r = json.loads(ln)
                if r.get("kernel", "quant") != "quant":
                    continue
                d[(r.get("workload", kind) if kind != "c2x4" else kind, tuple(r["window"]), r["variant"])].append(
                    r["ms"])
        except FileNotFoundError:
            pass
    variants = sorted({k[2] for k in d}, key=lambda v: (v != "prev", v != "base", v))
    keys = sorted({(k[0], k[1]) for k in d})
    print("| case | " + " | ".join(variants) + " |")
    print("|---|" + "---|" * len(variants))
    for k in keys:
        row = []
        for v in variants:
            xs = sorted(d.get((k[0], k[1], v), []))
            row.append("%.3f" % xs[len(xs) // 2] if xs else "")
        print("| %s %s | %s |" % (k[0], list(k[1]), " | ".join(row)))


if __name__ == "__main__":
    main(sys.argv[1])
