#!/usr/bin/env python
"""Markdown tables for DESIGN.md §11 from a tools/sweep.py JSON-lines file.

    python tools/sweep_table.py SWEEP.jsonl [COUNT_SWEEP.jsonl]

The optional second file is the same sweep run with --variant count; its
executed candidate counts give the executed 3-op fraction, which is the
headline wherever the algorithmic 4-op fraction exceeds 1.
"""
import json
import sys


def main(path):
    L = [json.loads(l) for l in open(path) if l.strip()]
    # executed counts from a --variant count run of the same sweep, if given
    ex = {}
    if len(sys.argv) > 2:
        for ln in open(sys.argv[2]):
            if ln.strip():
                d = json.loads(ln)
                if "evaluated_per_block" in d or "executed_c_per_block" in d:
                    ex[(d["config"], d["format"], tuple(d["window"]))] = d.get(
                        "executed_c_per_block", d.get("evaluated_per_block"))
    print("| config | format | window | C_eff | executed C | quant ms | GB/s bf16 (quant) | GB/s (TENSOR call) "
          "| bound | frac (algorithmic, 4-op) | frac (executed, 3-op) | headline (SURVEY §8(d)) | MSE cut |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for d in L:
        if "quant_ms" not in d:
            continue
        ev = d.get("executed_c_per_block", ex.get((d["config"], d["format"], tuple(d["window"]))))
        f3 = (3.0 * ev + 2.0) / (4.0 * d["c_eff"] + 2.0) * d["alu_frac"] if ev is not None else None
        head = d["roofline_frac"] if d["roofline_frac"] <= 1.0 or f3 is None else f3
        print("| %s | %s | [%d, %d] | %.2f | %s | %.3f | %.0f | %.0f | %s | %.3f | %s | %.3f%s | %.2f%% |" % (
            d["config"], d["format"], d["window"][0], d["window"][1], d["c_eff"],
            "%.2f" % ev if ev is not None else "-", d["quant_ms"], d["quant_bf16_gbs"], d["e2e_bf16_gbs"],
            d["bound"], d["roofline_frac"], "%.3f" % f3 if f3 is not None else "-", head,
            "" if head is d["roofline_frac"] else " (executed)", d["mse_cut_pct"]))
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
