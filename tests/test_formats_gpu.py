"""Other block formats on the GPU: MXFP4 (E2M1 / UE8M0 / 32),
MXFP6 E2M3 (E2M3 / UE8M0 / 32) and NVFP6 E2M3 (E2M3 / UE4M3 / 16) against the
oracle's general-format path, element by element: codes, scales, offsets,
per-block errors and G bit-exact (hardware cvt.rn.satfinite.e2m3x2 /
cvt.rp.satfinite.ue8m0x2 semantics included), sums within 1e-9; both scale
layouts; dequantization.
"""
import os
import sys

import numpy as np
import pytest
import torch

import ssgen

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_scale_layout import blocked  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = [(37, 32), (129, 256), (300, 96), (64, 4096), (5, 12288)]
FMTS = {"mxfp4": ["none"], "mxfp6_e2m3": ["none"], "nvfp6_e2m3": ["none", "tensor", "row"]}


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def _cmp(g, ref, G=True):
    assert np.array_equal(g.codes.cpu().numpy(), ref.codes)
    assert np.array_equal(g.scales.cpu().numpy(), ref.scales)
    assert np.array_equal(g.offsets.cpu().numpy(), ref.offsets)
    assert np.array_equal(g.err.cpu().numpy().view(np.uint32), ref.err.view(np.uint32))
    s = g.sums.cpu().numpy()
    for k in range(2):
        if np.isfinite(ref.sums[k]):
            assert abs(s[k] - ref.sums[k]) <= 1e-9 * abs(ref.sums[k]) + 1e-300
        else:
            assert s[k] == ref.sums[k]
    if G:
        assert np.array_equal(np.atleast_1d(g.G.cpu().numpy()).view(np.uint32),
                              np.atleast_1d(np.float32(ref.G)).view(np.uint32))


@pytest.mark.parametrize("fmt", list(FMTS))
@pytest.mark.parametrize("shape", SHAPES)
def test_format_parity(ss, oracle_lib, fmt, shape):
    x = ssgen.generate("student_t", *shape, seed=31, tid=shape[0] + 3 * shape[1])
    lim = 254 if fmt.startswith("mx") else 126
    for gmode in FMTS[fmt]:
        for w in [(0, 0), (-1, 1), (-2, 2), (-lim, lim)]:
            g = ss.quantize(x.cuda(), fmin=w[0], fmax=w[1], gmode=gmode, fmt=fmt)
            torch.cuda.synchronize()
            ref = oracle_lib.quantize_fmt(x, *shape, w[0], w[1], fmt, gmode)
            _cmp(g, ref, G=gmode != "none")


@pytest.mark.parametrize("fmt", list(FMTS))
def test_format_adversarial(ss, oracle_lib, fmt):
    x = ssgen.adversarial_rows()                      # [rows][64]: 32-blocks fit
    rows, cols = x.shape
    lim = 254 if fmt.startswith("mx") else 126
    for w in [(0, 0), (-1, 1), (-lim, lim)]:
        g = ss.quantize(x.cuda(), fmin=w[0], fmax=w[1], gmode="none", fmt=fmt)
        torch.cuda.synchronize()
        _cmp(g, oracle_lib.quantize_fmt(x, rows, cols, w[0], w[1], fmt, "none"), G=False)


@pytest.mark.parametrize("fmt", list(FMTS))
def test_format_swizzled_and_dequant(ss, oracle_lib, fmt):
    rows, cols = 300, 256
    x = ssgen.generate("weight_outlier", rows, cols, seed=32, tid=9)
    g = ss.quantize(x.cuda(), radius=2, gmode="none", fmt=fmt, scale_layout="swizzled")
    torch.cuda.synchronize()
    ref = oracle_lib.quantize_fmt(x, rows, cols, -2, 2, fmt, "none")
    assert np.array_equal(g.scales.cpu().numpy(), blocked(ref.scales))
    assert g.scales.numel() == ss.scale_bytes(rows, cols, "swizzled", fmt)
    for layout, out in (("swizzled", g), ("linear", ss.quantize(x.cuda(), radius=2, gmode="none", fmt=fmt))):
        d = ss.dequantize(out.codes, out.scales, rows, cols, None, scale_layout=layout, fmt=fmt)
        torch.cuda.synchronize()
        rd = oracle_lib.dequantize_fmt(ref.codes, ref.scales, rows, cols, fmt, 1.0)
        assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16), rd)


def test_mx_batched_many(ss, oracle_lib):
    xs = [ssgen.generate("gaussian", 1 + k % 9, 32 * (1 + k % 5), seed=33, tid=k) for k in range(150)]
    xd = [x.cuda() for x in xs]
    outs = [ss.alloc_out(x, fmt="mxfp4") for x in xd]
    ss.quantize_batched(xd, outs, radius=2, gmode="none", fmt="mxfp4")
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        _cmp(o, oracle_lib.quantize_fmt(x, *x.shape, -2, 2, "mxfp4", "none"), G=False)


def test_mx_rejects_global_scale(ss):
    x = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ss.SSError):
        ss.quantize(x, radius=1, gmode="tensor", fmt="mxfp4")
    with pytest.raises(ss.SSError):
        ss.quantize(torch.zeros(4, 48, dtype=torch.bfloat16, device="cuda"), radius=1, gmode="none",
                    fmt="mxfp4")                     # cols % 32 != 0


BLOCK_FMTS = ["nvfp4_b32", "nvfp4_b64", "nvfp4_b128", "nvfp4_b256"]


@pytest.mark.parametrize("fmt", BLOCK_FMTS)
@pytest.mark.parametrize("shape", [(37, 256), (65, 512), (9, 4096)])
def test_block_size_parity(ss, oracle_lib, fmt, shape):
    x = ssgen.generate("gaussian", *shape, seed=34, tid=shape[0] + shape[1])
    for gmode in ("none", "tensor", "row"):
        for w in [(0, 0), (-2, 2), (-126, 126)]:
            g = ss.quantize(x.cuda(), fmin=w[0], fmax=w[1], gmode=gmode, fmt=fmt)
            torch.cuda.synchronize()
            _cmp(g, oracle_lib.quantize_fmt(x, *shape, w[0], w[1], fmt, gmode), G=gmode != "none")


def test_block_size_swizzled(ss, oracle_lib):
    rows, cols = 300, 512
    x = ssgen.generate("student_t", rows, cols, seed=35, tid=1)
    g = ss.quantize(x.cuda(), radius=8, gmode="tensor", fmt="nvfp4_b64", scale_layout="swizzled")
    torch.cuda.synchronize()
    ref = oracle_lib.quantize_fmt(x, rows, cols, -8, 8, "nvfp4_b64", "tensor")
    assert np.array_equal(g.scales.cpu().numpy(), blocked(ref.scales))
    d = ss.dequantize(g.codes, g.scales, rows, cols, g.G, scale_layout="swizzled", fmt="nvfp4_b64")
    torch.cuda.synchronize()
    rd = oracle_lib.dequantize_fmt(ref.codes, ref.scales, rows, cols, "nvfp4_b64", ref.G)
    assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16), rd)
