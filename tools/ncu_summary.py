#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (runs here, on the CPU host).

    python tools/ncu_summary.py full  gpurun_out/quant_full_TAG.ncu-rep  > profiles/rNN/quant_TAG.md
    python tools/ncu_summary.py launches gpurun_out/launches_TAG.csv    > profiles/rNN/launches_TAG.md

`full` prints the metrics the roofline and the optimisation notes cite
(duration, DRAM bytes, pipe utilisations, issue activity, stall reasons,
occupancy) plus the per-opcode dynamic instruction mix from the source page.
`launches` prints per-kernel totals and shares of a --metrics
gpu__time_duration.sum launch list.
"""
from __future__ import annotations

import csv
import io
import re
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum",
]


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def full(rep: str):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    head, units = raw[0], raw[1]
    for row in raw[2:]:
        vals = dict(zip(head, row))
        un = dict(zip(head, units))
        print("## %s  (grid %s x %s)\n" % (vals.get("Kernel Name", "?"), vals.get("launch__grid_size"),
                                          vals.get("launch__block_size")))
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in vals:
                print("| %s | %s | %s |" % (k, vals[k], un.get(k, "")))
        stalls = [(k, float(v)) for k, v in vals.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "n/a")]
        stalls.sort(key=lambda kv: -kv[1])
        print("\nstall reasons (warps per issue):\n")
        for k, v in stalls[:8]:
            print("- %s: %.3f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""), v))
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        ie, sc = h.index("Instructions Executed"), h.index("Source")
        cnt, tot = Counter(), 0
        for r in src[2:]:
            try:
                n = int(r[ie])
            except (ValueError, IndexError):
                continue
            op = re.sub(r"^@!?U?P\w+\s+", "", r[sc].strip()).split()
            cnt[op[0] if op else "?"] += n
            tot += n
        print("\ndynamic instruction mix (warp-level, top 20 of %d):\n" % tot)
        print("| opcode | executed | share |\n|---|---|---|")
        for op, n in cnt.most_common(20):
            print("| %s | %d | %.1f%% |" % (op, n, 100.0 * n / tot))


def hot(rep: str, top: int = 60):
    """SASS-line stall attribution from the source page: warp-stall samples per
    stall reason, totals by opcode, and the hottest lines with their top reasons."""
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) < 3:
        print("no source page")
        return
    h = src[1]
    sc, ss_, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    reasons = [c for c in h if c.startswith("stall_") and not c.endswith("(Not Issued)")]
    ri = [h.index(c) for c in reasons]
    rows, tot_r, by_op, tot = [], Counter(), Counter(), 0
    for k, r in enumerate(src[2:]):
        try:
            smp = int(r[ss_] or 0)
        except (ValueError, IndexError):
            continue
        op = re.sub(r"^@!?U?P\w+\s+", "", r[sc].strip()).split()
        opn = op[0] if op else "?"
        rv = {}
        for c, i in zip(reasons, ri):
            try:
                v = int(r[i] or 0)
            except ValueError:
                v = 0
            if v:
                rv[c[6:]] = v
                tot_r[c[6:]] += v
        by_op[opn] += smp
        tot += smp
        rows.append((smp, k, r[sc].strip(), int(r[ie] or 0) if r[ie].isdigit() else 0, rv))
    print("warp-stall samples: %d\n" % tot)
    print("| reason | samples | share |\n|---|---|---|")
    for c, v in tot_r.most_common():
        print("| %s | %d | %.1f%% |" % (c, v, 100.0 * v / max(tot, 1)))
    print("\n| opcode | samples | share |\n|---|---|---|")
    for c, v in by_op.most_common(25):
        print("| %s | %d | %.1f%% |" % (c, v, 100.0 * v / max(tot, 1)))
    print("\nhottest SASS lines (index in the listing, samples, executed, top reasons):\n")
    print("| # | samples | share | executed | instruction | reasons |\n|---|---|---|---|---|---|")
    for smp, k, txt, n, rv in sorted(rows, key=lambda t: -t[0])[:top]:
        rs = ", ".join("%s %d" % kv for kv in sorted(rv.items(), key=lambda kv: -kv[1])[:3])
        print("| %d | %d | %.2f%% | %d | `%s` | %s |" % (k, smp, 100.0 * smp / max(tot, 1), n, txt[:70], rs))


def launches(path: str):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        k = r[ki].split("(")[0]
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print("| %s | %d | %.1f | %.1f | %.1f%% |" % (k, cnt[k], tot[k] / 1e3, tot[k] / 1e3 / cnt[k],
                                                     100 * tot[k] / s))


if __name__ == "__main__":
    {"full": full, "launches": launches, "hot": hot}[sys.argv[1]](sys.argv[2])
