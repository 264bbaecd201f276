#!/usr/bin/env python
"""Format sweeps of the paper's §4.1 "Other formats" on the GPU
generic-format kernel (ss_quantize_gen, reading R21):

  scale -- fig:nvfp-scale: value format fixed at E2M1, scale UExMy swept,
           16-element blocks, per-tensor global scale
  value -- fig:nvfp-val: scale format fixed at UE4M3, value ExMy swept,
           16-element blocks, per-tensor global scale
  mx    -- fig:mxfp: scale format fixed at UE8M0, value ExMy swept,
           32-element blocks, no global scale (the MX convention, R19)

Each point is the MSE cut of the exhaustive search (every valid scale code,
f in [-maxc, maxc]) against the max-abs scale (f = 0) on a unit-Gaussian bf16
tensor (P:287's synthetic setting), plus the offsets the search used.

    python tools/format_sweep.py [--rows 1024 --cols 4096] [--out profiles/r02/format_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STANDARD = {(2, 1, 4, 3, 16): "NVFP4 (paper 27 %)", (2, 1, 8, 0, 32): "MXFP4 (paper 8 %)",
            (2, 3, 8, 0, 32): "MXFP6 E2M3 (paper 11 %)", (3, 2, 8, 0, 32): "MXFP6 E3M2",
            (2, 3, 4, 3, 16): "NVFP6 E2M3"}


def sweeps():
    scale = [(2, 1, se, sm, 16) for se in range(2, 8) for sm in range(0, 6) if se + sm <= 8]
    scale.append((2, 1, 8, 0, 16))
    value = [(ve, vm, 4, 3, 16) for ve in range(1, 6) for vm in range(0, 6) if ve + vm <= 7]
    mx = [(ve, vm, 8, 0, 32) for ve in range(1, 6) for vm in range(0, 6) if ve + vm <= 7]
    return {"scale": scale, "value": value, "mx": mx}


def oracle_numer(fmt):
    """vmax * smax of a format (host arithmetic, the R21 definitions)."""
    ve, vm, se, sm, _ = fmt
    vb = (1 << (ve - 1)) - 1
    vmax = ((2 << vm) - 1) * 2.0 ** ((1 << ve) - 1 - vb - vm)
    sb = (1 << (se - 1)) - 1
    mc = (1 << (se + sm)) - 2
    smax = 2.0 ** (mc - sb) if sm == 0 else ((1 << sm) + (mc & ((1 << sm) - 1))) * 2.0 ** ((mc >> sm) - sb - sm)
    return vmax * smax


def point(torch, ss, x, fmt):
    lim = (1 << (fmt[2] + fmt[3])) - 2
    # per-tensor G = RN(vmax * smax / A) (R21) unless the scale range is so
    # wide that G would push the y-domain squared errors past binary32 (the
    # UE8M0 MX convention, and UE7M1): then no global scale, which such a
    # range does not need
    numer = float(oracle_numer(fmt))
    gm = "tensor" if numer <= 2.0 ** 40 else "none"
    o = ss.quantize_gen(x, fmt, fmin=-lim, fmax=lim, gmode=gm)
    s = o.sums.cpu().tolist()
    h = torch.bincount(o.offsets.to(torch.int64) + 128, minlength=256).cpu()
    top = torch.argsort(h, descending=True)[:4].tolist()
    n = x.numel()
    G2 = 1.0 if gm == "none" else float(o.G.item()) ** 2
    return {"format": "E%dM%d/UE%dM%d/%d" % fmt, "fmt": list(fmt), "gmode": gm,
            "mse_base": s[1] / G2 / n, "mse_best": s[0] / G2 / n,
            "cut_pct": 100.0 * (1 - s[0] / s[1]) if s[1] > 0 else 0.0,
            "top_offsets": {str(k - 128): int(h[k]) for k in top if h[k] > 0},
            "offsets_used": int((h > 0).sum())}


def table(rows, key_e, key_m, title):
    es = sorted({r["fmt"][key_e] for r in rows})
    ms = sorted({r["fmt"][key_m] for r in rows})
    by = {(r["fmt"][key_e], r["fmt"][key_m]): r for r in rows}
    lines = ["### %s (MSE cut %%, exhaustive search vs max-abs scale)\n" % title,
             "| E \\ M | " + " | ".join("M%d" % m for m in ms) + " |",
             "|---|" + "---|" * len(ms)]
    for e in es:
        cells = []
        for m in ms:
            r = by.get((e, m))
            if r is None:
                cells.append("")
                continue
            mark = " **" + STANDARD[tuple(r["fmt"])] + "**" if tuple(r["fmt"]) in STANDARD else ""
            cells.append("%.1f%s%s" % (r["cut_pct"], "" if r["gmode"] == "tensor" else " (no G)", mark))
        lines.append("| E%d | %s |" % (e, " | ".join(cells)))
    return "\n".join(lines) + "\n"


def main():
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    x = ssgen.generate("gaussian", a.rows, a.cols, seed=ssgen.workloads.BASE_SEED, tid=1, device=dev)
    res = {"elements": a.rows * a.cols, "data": "unit Gaussian bf16 (ssgen gaussian, tid 1)"}
    md = []
    for name, fmts in sweeps().items():
        rows = [point(torch, ss, x, f) for f in fmts]
        res[name] = rows
        if name == "scale":
            md.append(table(rows, 2, 3, "fig:nvfp-scale: E2M1 values, UExMy scales, 16-blocks"))
        elif name == "value":
            md.append(table(rows, 0, 1, "fig:nvfp-val: ExMy values, UE4M3 scales, 16-blocks"))
        else:
            md.append(table(rows, 0, 1, "fig:mxfp: ExMy values, UE8M0 scales, 32-blocks"))
    allc = [r for k in ("scale", "value", "mx") for r in res[k]]
    best = max(allc, key=lambda r: r["cut_pct"])
    md.append("Largest cut: %.1f %% at %s (paper: 'up to about 80 %%', P:302)\n" % (best["cut_pct"], best["format"]))
    print("\n".join(md))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
