#!/usr/bin/env python
"""Markdown tables for DESIGN.md §11 from a tools/sweep.py JSON-lines file.

    python tools/sweep_table.py profiles/r01/sweep_v9.jsonl
"""
import json
import sys


def main(path):
    L = [json.loads(l) for l in open(path) if l.strip()]
    print("| config | format | window | C_eff | quant ms | GB/s bf16 (quant) | GB/s (TENSOR call) "
          "| GB/s (amax + quant launches) | bound | frac (algorithmic) | MSE cut |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for d in L:
        if "quant_ms" not in d:
            continue
        print("| %s | %s | [%d, %d] | %.2f | %.3f | %.0f | %.0f | %.0f | %s | %.3f | %.2f%% |" % (
            d["config"], d["format"], d["window"][0], d["window"][1], d["c_eff"], d["quant_ms"],
            d["quant_bf16_gbs"], d["e2e_bf16_gbs"], d.get("e2e_sep_bf16_gbs") or 0, d["bound"],
            d["roofline_frac"], d["mse_cut_pct"]))
    f32 = [d for d in L if d["config"].startswith("f32")]
    if f32:
        print("\n| window | FP32 routine ms | G elem/s | bf16 kernel ms | G elem/s | FP32 in GB/s |")
        print("|---|---|---|---|---|---|")
        for d in f32:
            print("| [%d, %d] | %.3f | %.0f | %.3f | %.0f | %.0f |" % (
                d["window"][0], d["window"][1], d["f32_ms"], d["f32_gelem_s"], d["bf16_kernel_ms"],
                d["bf16_gelem_s"], d["f32_in_gbs"]))


if __name__ == "__main__":
    main(sys.argv[1])
