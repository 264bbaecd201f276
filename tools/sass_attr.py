#!/usr/bin/env python
"""Attribute a kernel's executed instructions to CUDA source lines (CPU host).

    python tools/sass_attr.py gpurun_out/X.sass.csv [--lib paper_2605_12464_b200/libss.so] [--top 40]

Input: `ncu -i rep --page source --csv --print-source sass` of one kernel
(per-SASS-line "Instructions Executed" and stall samples).  The line table
comes from `nvdisasm -g` of the same kernel in the locally built libss.so
(same sources and compiler as the box build).  Output: per source line, warp
instructions executed (total and per 16-element half-block when
--halfblocks is given), stall samples, and the source text.
"""
from __future__ import annotations

import argparse
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def mangled(name: str) -> str:
    # void ss::quant_kernel<(int)0, (int)0, (int)0, (int)0, (bool)0>(ss::QuantBatch)
    kn = re.search(r"ss::(quant_\w+)<", name).group(1)
    m = re.search(r"%s<(.*)>\(" % kn, name)
    args = [a.strip() for a in m.group(1).split(",")]
    enc = ""
    for a in args:
        v = a.split(")")[-1]
        if a.startswith("(bool)"):
            enc += "Lb%sE" % v
        else:
            iv = int(v)
            enc += "Li%sE" % (str(iv) if iv >= 0 else "n%d" % -iv)
    return "_ZN2ss%d%sI%sEEvNS_10QuantBatchE" % (len(kn), kn, enc)


def line_table(lib: str, fn: str):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout
    start = out.index(".text.%s:" % fn)
    end = out.find("\n.text.", start + 10)
    body = out[start:end if end > 0 else None]
    cur = None
    table = {}
    for ln in body.splitlines():
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2))
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2605_12464_b200", "libss.so"))
    ap.add_argument("--top", type=int, default=45)
    ap.add_argument("--halfblocks", type=float, default=0.0, help="half-blocks per launch (per-hb counts)")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    kname = rows[0][1]
    head = rows[1]
    ia, ie, iss = head.index("Address"), head.index("Instructions Executed"), head.index("# Samples")
    stall_cols = [(k, c) for k, c in enumerate(head) if c.startswith("stall_") and "(Not Issued)" not in c]
    data = [r for r in rows[2:] if len(r) > ie and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    table = line_table(a.lib, mangled(kname))
    agg = defaultdict(lambda: [0, 0, set(), defaultdict(int)])
    total = 0
    for r in data:
        off = int(r[ia], 16) - base
        loc, ins = table.get(off, (None, "?"))
        n = int(r[ie] or 0)
        total += n
        e = agg[loc]
        e[0] += n
        e[1] += int(r[iss] or 0)
        e[2].add(ins.split()[0] if not ins.startswith("@") else ins.split()[1])
        for k, c in stall_cols:
            if k < len(r) and r[k] not in ("", "0"):
                e[3][c[6:]] += int(float(r[k]))
    srcs = {}
    for d in ("paper_2605_12464_b200/csrc",):
        for f in os.listdir(os.path.join(ROOT, d)):
            srcs[f] = open(os.path.join(ROOT, d, f)).read().splitlines()
    print("kernel:", kname)
    print("warp instructions executed: %d%s" % (total, "  (%.1f per half-block per lane)" % (
        total * 32 / a.halfblocks) if a.halfblocks else ""))
    tot_smp = sum(v[1] for v in agg.values()) or 1
    print("\n| file:line | warp inst | share | per hb | stall samples (share) | top stall reasons | opcodes | source |")
    print("|---|---|---|---|---|---|---|---|")
    for loc, (n, smp, ops, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
        txt = srcs.get(loc[0], [""] * (loc[1] + 1))[loc[1] - 1].strip() if loc else ""
        top = ", ".join("%s %d" % kv for kv in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print("| %s | %d | %.1f%% | %s | %d (%.1f%%) | %s | %s | `%s` |" % (
            "%s:%d" % loc if loc else "?", n, 100.0 * n / total,
            "%.1f" % (n * 32 / a.halfblocks) if a.halfblocks else "-", smp, 100.0 * smp / tot_smp, top,
            " ".join(sorted(ops))[:50], txt[:60].replace("|", "\\|")))


if __name__ == "__main__":
    main()
