#!/usr/bin/env python
"""ScaleSearch study tooling, driven by the libss kernels.

Reproduces, on synthetic data and this build's kernels, the analyses of the
paper's §4.1:
  mse     -- MSE vs number of scales searched, f_min = 1 - f_max (fig:mse)
  hist    -- offset histogram of the exhaustive search (fig:histogram, P:289-298;
             fig:histogrammxf4)
  formats -- MSE cut per block format at the full search
  blocks  -- MSE cut vs block size 16..256 (fig:block_size)

    python tools/study.py [--out profiles/r01/study.json]   (one GPU)

Data: unit Gaussian (the paper's synthetic setting) and the Student-t
activations of C3.  Each figure's numbers go to one JSON document and a
markdown summary on stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cut_and_hist(torch, ss, x, fmin, fmax, fmt="nvfp4"):
    gm = "none" if fmt.startswith("mx") else "tensor"
    o = ss.quantize(x, fmin=fmin, fmax=fmax, gmode=gm, fmt=fmt)
    s = o.sums.cpu().tolist()
    h = torch.bincount(o.offsets.to(torch.int64) + 254, minlength=509).cpu().tolist()
    hist = {str(k - 254): v for k, v in enumerate(h) if v}
    n = x.numel()
    G2 = 1.0 if gm == "none" else float(o.G.item()) ** 2
    return {"mse_base": s[1] / G2 / n, "mse_best": s[0] / G2 / n,
            "cut_pct": 100.0 * (1 - s[0] / s[1]) if s[1] > 0 else 0.0, "hist": hist}


def main():
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=4096)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    data = {
        "gaussian": ssgen.generate("gaussian", a.rows, a.cols, seed=ssgen.workloads.BASE_SEED, tid=1,
                                   device=dev),
        "student_t": ssgen.generate("student_t", a.rows, a.cols, seed=ssgen.workloads.BASE_SEED,
                                    tid=3000, device=dev),
    }
    out = {"elements": a.rows * a.cols, "mse": {}, "hist": {}, "formats": {}, "blocks": {}}
    # fig:mse -- number of scales searched = f_max - f_min + 1 with f_min = 1 - f_max
    for name, x in data.items():
        rows = []
        for fmax in range(1, 17):
            r = cut_and_hist(torch, ss, x, 1 - fmax, fmax)
            rows.append({"scales": 2 * fmax, "window": [1 - fmax, fmax], "mse": r["mse_best"],
                         "mse_base": r["mse_base"], "cut_pct": r["cut_pct"]})
        full = cut_and_hist(torch, ss, x, -126, 126)
        rows.append({"scales": 253, "window": [-126, 126], "mse": full["mse_best"],
                     "mse_base": full["mse_base"], "cut_pct": full["cut_pct"]})
        out["mse"][name] = rows
    # fig:histogram -- exhaustive search offsets (NVFP4) and MXFP4
    out["hist"]["nvfp4_gaussian"] = cut_and_hist(torch, ss, data["gaussian"], -126, 126)["hist"]
    out["hist"]["nvfp4_student_t"] = cut_and_hist(torch, ss, data["student_t"], -126, 126)["hist"]
    out["hist"]["mxfp4_gaussian"] = cut_and_hist(torch, ss, data["gaussian"], -254, 254, "mxfp4")["hist"]
    # formats at the full search
    for fmt, lim in (("nvfp4", 126), ("nvfp6_e2m3", 126), ("mxfp4", 254), ("mxfp6_e2m3", 254)):
        r = cut_and_hist(torch, ss, data["gaussian"], -lim, lim, fmt)
        out["formats"][fmt] = {k: r[k] for k in ("mse_base", "mse_best", "cut_pct")}
        out["formats"][fmt]["offsets_used"] = len(r["hist"])
    # block sizes (fig:block_size): NVFP4 values and scales on 16..256-element blocks
    for name, x in data.items():
        out["blocks"][name] = {}
        for fmt, bs in (("nvfp4", 16), ("nvfp4_b32", 32), ("nvfp4_b64", 64), ("nvfp4_b128", 128),
                        ("nvfp4_b256", 256)):
            r = cut_and_hist(torch, ss, x, -126, 126, fmt)
            out["blocks"][name][bs] = {k: r[k] for k in ("mse_base", "mse_best", "cut_pct")}

    print("## MSE vs scales searched (f_min = 1 - f_max), unit Gaussian\n")
    print("| scales | window | MSE | cut |\n|---|---|---|---|")
    for r in out["mse"]["gaussian"]:
        print("| %d | [%d, %d] | %.5f | %.2f%% |" % (r["scales"], r["window"][0], r["window"][1],
                                                   r["mse"], r["cut_pct"]))
    print("\n## Formats at the full search (unit Gaussian)\n")
    print("| format | MSE base | MSE best | cut | offsets used |\n|---|---|---|---|---|")
    for k, v in out["formats"].items():
        print("| %s | %.5f | %.5f | %.2f%% | %d |" % (k, v["mse_base"], v["mse_best"], v["cut_pct"],
                                                    v["offsets_used"]))
    print("\n## Block size (NVFP4 values and scales, full search)\n")
    print("| data | block | MSE base | MSE best | cut |\n|---|---|---|---|---|")
    for name, d in out["blocks"].items():
        for bs, v in d.items():
            print("| %s | %d | %.5f | %.5f | %.2f%% |" % (name, bs, v["mse_base"], v["mse_best"], v["cut_pct"]))
    print("\n## Offset histogram, NVFP4 exhaustive search, unit Gaussian\n")
    h = out["hist"]["nvfp4_gaussian"]
    print(" ".join("%s:%d" % (k, h[k]) for k in sorted(h, key=int)))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
