#!/usr/bin/env python
"""Per-config measurements on one B200 for BASELINE.json's five configs
(SURVEY §8(d)): quantize-only and end-to-end (amax + quantize) throughput,
ALU / HBM roofline fractions, valid-candidate count, and the MSE cut.

    python tools/sweep.py [--configs c1,c2,c3,c4,c5] [--out gpurun_out/sweep.jsonl]

Timing: CUDA events on the launching stream around `reps` back-to-back calls
(2 warm-ups first).  With --variant count (libss_count.so) each line also
carries the candidate evaluations the kernel executed per block (exact pruning
skips the rest) and the ALU fraction of that executed work.
C1 (33.5 MB) is rotated over 40 copies (> L2) between runs; the others
exceed L2.  The driver's bench line is bench.py; this is the table behind
DESIGN.md §11.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RADII_C3 = list(range(0, 17))
RADII_C5 = [0, 1, 2, 3, 4, 6, 8, 12, 16, 32, 64, 126]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), float(m["sm_max_mhz"])
    except Exception:
        return 6650.0, 1965.0


VARIANT = "base"


def med(ts):
    ts = sorted(ts)
    return ts[len(ts) // 2]


def measure(torch, ss, groups, fmin, fmax, reps=5, fmt="nvfp4"):
    """groups: list of tensor lists (rotated between runs).  Returns timings and stats."""
    outs = [[ss.alloc_out(x, fmt=fmt) for x in g] for g in groups]
    amax = [torch.zeros(len(g), dtype=torch.int32, device=g[0].device) for g in groups]
    mx = fmt.startswith("mx")              # UE8M0 scales: no global scale (R19)

    def q_only(i):
        if mx:
            ss.quantize_batched(groups[i], outs[i], fmin=fmin, fmax=fmax, gmode="none", fmt=fmt)
        else:
            ss.quantize_batched(groups[i], outs[i], fmin=fmin, fmax=fmax, gmode="device_amax",
                                amax=amax[i], fmt=fmt)

    def e2e_sep(i):
        ss.tensor_amax_batched(groups[i], out=amax[i])
        q_only(i)

    def e2e(i):   # the library's per-tensor-G call (amax fused into the launch where it pays)
        if mx:
            q_only(i)
        else:
            ss.quantize_batched(groups[i], outs[i], fmin=fmin, fmax=fmax, gmode="tensor", fmt=fmt)

    for i in range(len(groups)):
        ss.tensor_amax_batched(groups[i], out=amax[i])
    res = {}
    if VARIANT == "count":   # executed evaluations, one pass
        import ctypes
        L = ss.lib()
        L.ss_debug_take_evals.restype = ctypes.c_ulonglong
        L.ss_debug_take_evals()
        q_only(0)
        nb = sum(x.numel() for x in groups[0]) // 16
        res["evaluated_per_block"] = L.ss_debug_take_evals() / nb * (2 if mx else 1)
    for name, fn in (("quant", q_only), ("amax_quant_sep", e2e_sep), ("amax_quant", e2e)):
        for w in range(2):
            fn(w % len(groups))
        torch.cuda.synchronize()
        # `reps` calls back to back between one event pair (rotating the input
        # groups): the host enqueues ahead of the device, so host overhead per
        # call is hidden whenever a call's device time exceeds it
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(reps):
            fn(r % len(groups))
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) / reps
    # statistics from group 0: valid candidates, x-domain SSE, f* histogram
    g, o = groups[0], outs[0]
    tot_valid, tot_blocks, s_best, s_base = 0, 0, 0.0, 0.0
    hist = torch.zeros(253, dtype=torch.int64, device=g[0].device)
    for x, oo in zip(g, o):
        c0 = oo.scales.reshape(-1).to(torch.int32) - oo.offsets.to(torch.int32)
        # valid candidates of a block: f in [fmin, fmax] with 1 <= c0 + f <= 126,
        # plus the zero-scale candidate when c0 == 0 (R2, R3)
        if mx:     # every UE8M0 code 0..254 is a scale
            hi = torch.clamp(254 - c0, max=fmax)
            lo = torch.clamp(-c0, min=fmin)
            valid = torch.clamp(hi - lo + 1, min=0)
        else:
            hi = torch.clamp(126 - c0, max=fmax)
            lo = torch.clamp(1 - c0, min=fmin)
            valid = torch.clamp(hi - lo + 1, min=0) + (c0 == 0).to(torch.int32)
        tot_valid += int(valid.sum())
        tot_blocks += c0.numel()
        G2 = 1.0 if mx else float(oo.G.item()) ** 2
        s = oo.sums.cpu().tolist()
        s_best += s[0] / G2
        s_base += s[1] / G2
        hist += torch.bincount(oo.offsets.to(torch.int64) + 126, minlength=253)
        del valid, c0
    n = sum(x.numel() for x in g)
    h = hist.cpu().tolist()
    return res, n, tot_valid / max(tot_blocks, 1), s_best, s_base, {str(k - 126): v for k, v in enumerate(h) if v}


# bytes per element written+read by the quantize kernel: bf16 in + codes +
# scales + float2 errors per scale block
FMT_BYTES = {"nvfp4": 2 + 0.5 + 1 / 16 + 8 / 16, "mxfp4": 2 + 0.5 + 1 / 32 + 8 / 32,
             "mxfp6_e2m3": 2 + 1 + 1 / 32 + 8 / 32, "nvfp6_e2m3": 2 + 1 + 1 / 16 + 8 / 16}


def report(cfg, fmin, fmax, res, n, ceff, s_best, s_base, hist, hbm, mhz, extra=None, fmt="nvfp4"):
    alu_peak = 148 * 128 * mhz * 1e6
    tq = res["quant"] * 1e-3
    te = res["amax_quant"] * 1e-3
    ops = (4.0 * ceff + 2.0) * n
    bytes_q = FMT_BYTES[fmt] * n
    t_roof = max(bytes_q / (hbm * 1e9), ops / alu_peak)
    line = {"config": cfg, "format": fmt, "window": [fmin, fmax], "elements": n, "c_eff": ceff,
            "quant_ms": res["quant"], "amax_quant_ms": res["amax_quant"],
            "amax_quant_sep_ms": res.get("amax_quant_sep"),
            "quant_bf16_gbs": 2 * n / tq / 1e9, "e2e_bf16_gbs": 2 * n / te / 1e9,
            "e2e_sep_bf16_gbs": 2 * n / (res["amax_quant_sep"] * 1e-3) / 1e9 if res.get("amax_quant_sep") else None,
            "bound": "alu" if ops / alu_peak > bytes_q / (hbm * 1e9) else "hbm",
            "roofline_frac": t_roof / tq, "alu_frac": ops / alu_peak / tq,
            "hbm_frac": bytes_q / (hbm * 1e9) / tq,
            "mse_cut_pct": 100.0 * (1 - s_best / s_base) if s_base > 0 else 0.0,
            "mse_base": s_base / n, "mse_best": s_best / n}
    if hist is not None and len(hist) <= 40:
        line["fstar_hist"] = hist
    if "evaluated_per_block" in res:
        ev = res["evaluated_per_block"]
        line["executed_c_per_block"] = ev
        line["executed_alu_frac"] = (4.0 * ev + 2.0) * n / alu_peak / tq
        line["executed_frac_3op"] = (3.0 * ev + 2.0) * n / alu_peak / tq
    # the algorithmic (4-op, every valid candidate) fraction is
    # the headline while it is <= 1; past 1 (pruning skips work) the executed
    # 3-op fraction is, when a counting run measured it
    if line["roofline_frac"] <= 1.0 or "executed_frac_3op" not in line:
        line["headline_frac"], line["headline_basis"] = line["roofline_frac"], "algorithmic"
    else:
        line["headline_frac"], line["headline_basis"] = line["executed_frac_3op"], "executed 3-op"
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)
    return line


def main():
    import torch
    import ssgen
    import paper_2605_12464_b200 as ss
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,oracle,oracle_samples,c2,c3,c4,f32,paper_tab,c5,formats")
    ap.add_argument("--c5-gib", default="1,8")
    ap.add_argument("--out", default=None)
    ap.add_argument("--variant", default="base", help="tools build libss_<variant>.so (e.g. count)")
    a = ap.parse_args()
    global VARIANT
    VARIANT = a.variant
    from paper_2605_12464_b200 import _binding
    _binding.use_variant(a.variant)
    hbm, mhz = peaks()
    dev = torch.device("cuda", 0)
    lines = []
    seed = ssgen.workloads.BASE_SEED

    def gen(specs):
        return [ssgen.generate(s.kind, s.rows, s.cols, seed=seed, tid=s.tid, device=dev) for s in specs]

    cfgs = a.configs.split(",")
    if "c1" in cfgs:
        x = gen(ssgen.workload("c1_gauss4096"))
        groups = [[x[0].clone()] for _ in range(40)]   # 1.34 GB rotated > L2
        del x
        for w in [(-8, 8), (0, 0), (-1, 1), (-2, 6), (-126, 126)]:
            lines.append(report("c1_gauss4096", *w, *measure(torch, ss, groups, *w, reps=80), hbm, mhz))
        del groups
        torch.cuda.empty_cache()
    if "oracle" in cfgs:   # the oracle on the full C1 tensor, 1 thread and all cores,
        import time       # plus a full-tensor bit-exact check of the GPU output against it
        import numpy as np
        import oracle
        oracle.build()
        x = gen(ssgen.workload("c1_gauss4096"))[0]
        xc = x.cpu()
        o = ss.quantize(x, radius=8, gmode="tensor")
        torch.cuda.synchronize()
        for th in (1, os.cpu_count()):
            t0 = time.perf_counter()
            r = oracle.quantize(xc, 4096, 4096, -8, 8, "tensor", threads=th)
            dt = time.perf_counter() - t0
            same = (np.array_equal(o.codes.cpu().numpy(), r.codes) and
                    np.array_equal(o.scales.cpu().numpy(), r.scales) and
                    np.array_equal(o.err.cpu().numpy().view(np.uint32), r.err.view(np.uint32)))
            line = {"config": "oracle_c1_gauss4096", "window": [-8, 8], "threads": th,
                    "cpu": os.cpu_count(), "oracle_s": dt, "oracle_gbs_bf16": 2 * x.numel() / dt / 1e9,
                    "gpu_equals_oracle_full_tensor": bool(same)}
            print(json.dumps(line), flush=True)
            lines.append(line)
        del x, xc, o
        torch.cuda.empty_cache()
    if "oracle_samples" in cfgs:   # a fixed 2^24-element sample per config and radius,
        import time               # all host cores, with the extrapolated full-workload oracle time
        import oracle
        oracle.build()
        for name, windows in (("c2_qwen3_8b_weights", [(0, 0), (-2, 6), (-8, 8)]),
                              ("c3_act_student_t", [(0, 0), (-1, 1), (-2, 2), (-8, 8), (-16, 16)]),
                              ("c4_llama70b_kv", [(-8, 8)]),
                              ("c5_gauss_1gib", [(0, 0), (-1, 1), (-8, 8), (-126, 126)])):
            specs = ssgen.workload(name)
            full = sum(sp.numel for sp in specs)
            sample, need = [], 1 << 24   # leading rows of the leading tensors, 2^24 elements
            for sp in specs:
                rows = min(sp.rows, -(-need // sp.cols))
                sample.append(ssgen.generate(sp.kind, sp.rows, sp.cols, seed=seed, tid=sp.tid, row_start=0,
                                             row_end=rows))
                need -= rows * sp.cols
                if need <= 0:
                    break
            n = sum(x.numel() for x in sample)
            for w in windows:
                t0 = time.perf_counter()
                for x in sample:
                    oracle.quantize(x, x.shape[0], x.shape[1], w[0], w[1], "tensor", threads=0)
                dt = time.perf_counter() - t0
                line = {"config": "oracle_sample_" + name, "window": list(w), "elements": n,
                        "cpu": os.cpu_count(), "threads": os.cpu_count(), "oracle_s": dt,
                        "oracle_gelem_s": n / dt / 1e9, "oracle_gbs_bf16": 2 * n / dt / 1e9,
                        "extrapolated_full_s": dt * full / n,
                        "note": "G from each sample tensor's own amax (timing only)"}
                print(json.dumps(line), flush=True)
                lines.append(line)
    if "c2" in cfgs:
        xs = gen(ssgen.workload("c2_qwen3_8b_weights"))
        for w in [(-8, 8), (-2, 6), (0, 0)]:
            lines.append(report("c2_qwen3_8b_weights", *w, *measure(torch, ss, [xs], *w, reps=3), hbm, mhz))
        del xs
        torch.cuda.empty_cache()
    if "c3" in cfgs:
        xs = gen(ssgen.workload("c3_act_student_t"))
        for r in RADII_C3:
            lines.append(report("c3_act_student_t", -r, r, *measure(torch, ss, [xs], -r, r), hbm, mhz))
        del xs
        torch.cuda.empty_cache()
    if "c4" in cfgs:
        xs = gen(ssgen.workload("c4_llama70b_kv"))
        lines.append(report("c4_llama70b_kv", -8, 8, *measure(torch, ss, [xs], -8, 8, reps=3), hbm, mhz))
        del xs
        torch.cuda.empty_cache()
    if "f32" in cfgs:   # the one-thread block routine through ss_quantize_nvfp4_f32
        x = gen(ssgen.workload("c3_act_student_t"))[0]
        xf = x.float()
        amax = ss.tensor_amax(x)
        out = ss.quantize(x, radius=8, gmode="tensor")
        G = out.G
        for w in [(-8, 8), (-2, 6), (0, 0)]:
            def run_f32():
                ss.quantize_f32(xf, fmin=w[0], fmax=w[1], G=G)

            def run_bf16():
                ss.quantize(x, fmin=w[0], fmax=w[1], gmode="device_amax", amax=amax, out=out)
            t = {}
            for name, fn in (("f32", run_f32), ("bf16", run_bf16)):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                t[name] = e0.elapsed_time(e1) / 10
            n = x.numel()
            line = {"config": "f32_routine_c3_shape", "window": list(w), "elements": n,
                    "f32_ms": t["f32"], "bf16_kernel_ms": t["bf16"],
                    "f32_gelem_s": n / t["f32"] / 1e6, "bf16_gelem_s": n / t["bf16"] / 1e6,
                    "f32_in_gbs": 4 * n / t["f32"] / 1e6}
            print(json.dumps(line), flush=True)
            lines.append(line)
        del x, xf, out
        torch.cuda.empty_cache()
    if "paper_tab" in cfgs:   # tab:quant_overhead: FP32 2048x2048 Gaussian, G given
        gen_ = torch.Generator(device="cpu").manual_seed(seed)
        x32 = torch.randn(2048, 2048, generator=gen_).to(dev)
        xb = x32.to(torch.bfloat16)
        amax = ss.tensor_amax(xb)
        G = ss.quantize(xb, radius=0, gmode="tensor").G
        copies = 64                                   # 64 x 16.8 MB > L2 for the cold runs
        x32s = [x32] + [x32.clone() for _ in range(copies - 1)]
        xbs = [xb] + [xb.clone() for _ in range(copies - 1)]
        out_b = ss.alloc_out(xb, want_err=False, want_offsets=False, want_sums=False, want_g=False)
        for w in [(0, 0), (-1, 1), (-2, 6)]:
            t = {}
            fns = (("f32", lambda i: ss.quantize_f32(x32s[i], fmin=w[0], fmax=w[1], G=G, want_err=False,
                                                     want_offsets=False)),
                   ("bf16", lambda i: ss.quantize(xbs[i], fmin=w[0], fmax=w[1], gmode="device_amax",
                                                  amax=amax, out=out_b)))
            for name, fn in fns:
                for mode, rot in (("hot", 1), ("cold", copies)):
                    # 64 calls captured in a CUDA graph: device time without host launch overhead
                    st = torch.cuda.Stream()
                    st.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(st):
                        for i in range(3):
                            fn(i % rot)
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=st):
                        for i in range(64):
                            fn(i % rot)
                    g.replay()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5):
                        g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    t["%s_%s_ms" % (name, mode)] = e0.elapsed_time(e1) / (5 * 64)
                    del g
            paper = {(0, 0): 0.0258, (-1, 1): 0.0328, (-2, 6): 0.0449}[w]
            line = {"config": "paper_tab_quant_overhead_2048sq_fp32", "window": list(w),
                    "elements": x32.numel(), "paper_ms_unstated_hw": paper, **t}
            print(json.dumps(line), flush=True)
            lines.append(line)
        del x32s, xbs
        torch.cuda.empty_cache()
    if "c5" in cfgs:
        for gib in [int(v) for v in a.c5_gib.split(",")]:
            xs = gen(ssgen.workload("c5_gauss_%dgib" % gib))
            for r in RADII_C5:
                lines.append(report("c5_gauss_%dgib" % gib, -r, r,
                                    *measure(torch, ss, [xs], -r, r, reps=3), hbm, mhz))
            del xs
            torch.cuda.empty_cache()
    if "formats" in cfgs:   # other block formats on C5 (1 GiB Gaussian)
        xs = gen(ssgen.workload("c5_gauss_1gib"))
        for fmt, radii in (("mxfp4", [0, 1, 2]), ("mxfp6_e2m3", [0, 1, 2]),
                           ("nvfp6_e2m3", [0, 1, 2, 8]), ("nvfp4", [0, 8])):
            for r in radii:
                lines.append(report("c5_gauss_1gib", -r, r, *measure(torch, ss, [xs], -r, r, reps=3, fmt=fmt),
                                    hbm, mhz, fmt=fmt))
        del xs
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
