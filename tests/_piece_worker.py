"""Worker of tests/test_pieces_gpu.py (run in its own process): loads the test
build libss_piece.so (SS_MAX_PIECE_BLOCKS=4096 half-blocks, so tensors of a
few thousand blocks already run as row pieces) and checks every output
against the oracle.  Prints one line per case; exits non-zero on a mismatch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import ssgen
    import oracle
    from paper_2605_12464_b200 import _binding
    _binding.use_variant("piece")
    import paper_2605_12464_b200 as ss
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_scale_layout import blocked  # linear -> swizzled (its own pinned helper)

    def cmp(g, r, what, swz=False, rows=None, cols=None, bs=16):
        sc = g.scales.cpu().numpy()
        ref_sc = r.scales if not swz else blocked(r.scales.reshape(rows, cols // bs))
        assert np.array_equal(g.codes.cpu().numpy(), r.codes), what + " codes"
        assert np.array_equal(sc.reshape(-1)[: ref_sc.size], np.asarray(ref_sc).reshape(-1)), what + " scales"
        if g.err is not None:
            assert np.array_equal(g.err.cpu().numpy().view(np.uint32), r.err.view(np.uint32)), what + " err"
        if g.offsets is not None:
            assert np.array_equal(g.offsets.cpu().numpy(), r.offsets), what + " offsets"
        s = g.sums.cpu().numpy()
        assert np.allclose(s, r.sums, rtol=1e-9, atol=0), what + " sums %r %r" % (s, r.sums)

    cases = 0
    for kind, rows, cols, lo, hi, gm in [("student_t", 1000, 256, -8, 8, "tensor"),
                                         ("weight_outlier", 300, 1024, -2, 6, "tensor"),
                                         ("gaussian", 129, 4096, -1, 1, "none"),
                                         ("kv_k", 777, 128, 0, 0, "tensor")]:
        x = ssgen.generate(kind, rows, cols, seed=91, tid=rows)
        g = ss.quantize(x.cuda(), fmin=lo, fmax=hi, gmode=gm)
        torch.cuda.synchronize()
        r = oracle.quantize(x, rows, cols, lo, hi, gm)
        cmp(g, r, "%s %dx%d" % (kind, rows, cols))
        assert np.float32(g.G.cpu().numpy()[0]) == np.float32(r.G)
        d = ss.dequantize(g.codes, g.scales, rows, cols, g.G)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16),
                              oracle.dequantize(r.codes, r.scales, rows, cols, r.G)), "dequant"
        cases += 1
    # a batch: a split tensor between whole ones (pieces stay in one launch), device amax
    xs = [ssgen.generate("student_t", r_, c_, seed=92, tid=r_) for r_, c_ in ((3, 64), (2000, 256), (40, 512))]
    amax = ss.tensor_amax_batched([x.cuda() for x in xs])
    outs = [ss.alloc_out(x.cuda()) for x in xs]
    ss.quantize_batched([x.cuda() for x in xs], outs, fmin=-3, fmax=5, gmode="device_amax", amax=amax)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        r = oracle.quantize(x, x.shape[0], x.shape[1], -3, 5, "given", amax_bits=oracle.tensor_amax(x))
        cmp(o, r, "batch %dx%d" % tuple(x.shape))
        cases += 1
    # per-row G (two-pass and row-fused) and the swizzled layout (128-row pieces)
    for rows, cols, layout in ((600, 512, "swizzled"), (1000, 1024, "linear"), (300, 2048, "linear")):
        x = ssgen.generate("student_t", rows, cols, seed=93, tid=rows)
        for lo, hi in ((-1, 1), (-8, 8)):
            g = ss.quantize(x.cuda(), fmin=lo, fmax=hi, gmode="row", scale_layout=layout)
            torch.cuda.synchronize()
            r = oracle.quantize(x, rows, cols, lo, hi, "row")
            cmp(g, r, "row %dx%d %s" % (rows, cols, layout), swz=layout == "swizzled", rows=rows, cols=cols)
            assert np.array_equal(g.G.cpu().numpy().view(np.uint32), r.G.view(np.uint32)), "G_r"
            d = ss.dequantize(g.codes, g.scales, rows, cols, g.G, scale_layout=layout)
            torch.cuda.synchronize()
            assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16),
                                  oracle.dequantize(r.codes, r.scales, rows, cols, r.G)), "dequant row"
            cases += 1
    # 32-element blocks (half-block pieces) and E2M3 codes
    for fmt, gm in (("mxfp4", "none"), ("nvfp6_e2m3", "tensor")):
        x = ssgen.generate("gaussian", 700, 512, seed=94, tid=7)
        g = ss.quantize(x.cuda(), fmin=-2, fmax=2, gmode=gm, fmt=fmt)
        torch.cuda.synchronize()
        r = oracle.quantize_fmt(x, 700, 512, -2, 2, fmt, gm)
        cmp(g, r, fmt, bs=32 if fmt.startswith("mx") else 16)
        cases += 1
    print("piece cases ok:", cases)


if __name__ == "__main__":
    main()
