"""SURVEY NEXT(1) on the GPU: per-row global scale and the tensor-core scale layout.

- SS_GLOBAL_ROW: codes, scales, per-block errors and the per-row G array are
  bit-exact against the oracle's mode "row" (each row its own tensor, R9).
- SS_SCALE_SWIZZLED: the scale bytes equal the oracle's linear scales placed
  by the block-scaled MMA layout (R15b).  The index function is
  tests/test_scale_layout.py's, pinned there against two other statements of
  the layout; padding bytes must be zero.
- Dequantization reads both layouts and per-row G.
- The outputs are directly consumable: cuBLASLt's NVFP4 GEMM
  (torch.nn.functional.scaled_mm, BlockWise1x16 + SWIZZLE_32_4_4) on our
  codes and swizzled scales reproduces the FP32 product of the dequantized
  operands.
"""
import os
import sys

import numpy as np
import pytest
import torch

import ssgen

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_scale_layout import blocked  # noqa: E402  (the layout statement, pinned on CPU)

pytestmark = pytest.mark.gpu

SHAPES = [(37, 16), (129, 128), (300, 96), (257, 4096), (5, 12288), (128, 64)]


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("win", [(-8, 8), (-2, 6), (0, 0)])
def test_row_mode_parity(ss, oracle_lib, shape, win):
    x = ssgen.generate("weight_outlier", *shape, seed=17, tid=shape[0] * 7 + shape[1])
    g = ss.quantize(x.cuda(), fmin=win[0], fmax=win[1], gmode="row")
    torch.cuda.synchronize()
    ref = oracle_lib.quantize(x, *shape, win[0], win[1], "row")
    assert np.array_equal(g.codes.cpu().numpy(), ref.codes)
    assert np.array_equal(g.scales.cpu().numpy(), ref.scales)
    assert np.array_equal(g.offsets.cpu().numpy(), ref.offsets)
    assert np.array_equal(g.err.cpu().numpy().view(np.uint32), ref.err.view(np.uint32))
    assert np.array_equal(g.G.cpu().numpy().view(np.uint32), ref.G.view(np.uint32))
    s = g.sums.cpu().numpy()
    assert abs(s[0] - ref.sums[0]) <= 1e-9 * abs(ref.sums[0]) + 1e-300


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("gmode", ["tensor", "row"])
def test_swizzled_scales(ss, oracle_lib, shape, gmode):
    x = ssgen.generate("student_t", *shape, seed=18, tid=shape[0] + shape[1])
    g = ss.quantize(x.cuda(), radius=8, gmode=gmode, scale_layout="swizzled")
    torch.cuda.synchronize()
    ref = oracle_lib.quantize(x, *shape, -8, 8, gmode)
    assert g.scales.numel() == ss.scale_bytes(*shape, "swizzled")
    assert np.array_equal(g.scales.cpu().numpy(), blocked(ref.scales))   # includes zero padding
    assert np.array_equal(g.codes.cpu().numpy(), ref.codes)
    assert np.array_equal(g.err.cpu().numpy().view(np.uint32), ref.err.view(np.uint32))


def test_batched_mixed_layouts_row_mode(ss, oracle_lib):
    xs = [ssgen.generate("gaussian", r, c, seed=19, tid=k) for k, (r, c) in enumerate(SHAPES)]
    xd = [x.cuda() for x in xs]
    outs = [ss.alloc_out(x, scale_layout="swizzled", gmode="row") for x in xd]
    ss.quantize_batched(xd, outs, radius=8, gmode="row", scale_layout="swizzled")
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        ref = oracle_lib.quantize(x, *x.shape, -8, 8, "row")
        assert np.array_equal(o.codes.cpu().numpy(), ref.codes)
        assert np.array_equal(o.scales.cpu().numpy(), blocked(ref.scales))
        assert np.array_equal(o.G.cpu().numpy().view(np.uint32), ref.G.view(np.uint32))


@pytest.mark.parametrize("layout", ["linear", "swizzled"])
def test_dequantize_row_mode(ss, oracle_lib, layout):
    rows, cols = 300, 96
    x = ssgen.generate("weight_outlier", rows, cols, seed=20, tid=5)
    g = ss.quantize(x.cuda(), radius=8, gmode="row", scale_layout=layout)
    d = ss.dequantize(g.codes, g.scales, rows, cols, g.G, scale_layout=layout)
    torch.cuda.synchronize()
    ref = oracle_lib.quantize(x, rows, cols, -8, 8, "row")
    rd = oracle_lib.dequantize(ref.codes, ref.scales, rows, cols, ref.G)
    assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16), rd)


@pytest.mark.parametrize("gmode", ["none", "tensor"])
def test_nvfp4_gemm_consumes_codes_and_swizzled_scales(ss, gmode):
    import torch.nn.functional as F
    if not hasattr(torch, "float4_e2m1fn_x2") or not hasattr(F, "scaled_mm"):
        pytest.skip("torch without NVFP4 scaled_mm")
    M, N, K = 256, 384, 1024
    a = ssgen.generate("gaussian", M, K, seed=21, tid=1).cuda()
    b = ssgen.generate("weight_outlier", N, K, seed=21, tid=2).cuda()
    qa = ss.quantize(a, radius=8, gmode=gmode, scale_layout="swizzled")
    qb = ss.quantize(b, radius=8, gmode=gmode, scale_layout="swizzled")
    # reference: FP32 product of the dequantized operands q*s (G = 1 dequantization is exact in bf16)
    da = ss.dequantize(qa.codes, qa.scales, M, K, None, scale_layout="swizzled").float()
    db = ss.dequantize(qb.codes, qb.scales, N, K, None, scale_layout="swizzled").float()
    torch.backends.cuda.matmul.allow_tf32 = False
    ref = da @ db.t()
    def gemm(dt):
        return F.scaled_mm(qa.codes.view(torch.float4_e2m1fn_x2), qb.codes.view(torch.float4_e2m1fn_x2).t(),
                           qa.scales.view(torch.float8_e4m3fn), F.ScalingType.BlockWise1x16,
                           qb.scales.view(torch.float8_e4m3fn), F.ScalingType.BlockWise1x16,
                           swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                           output_dtype=dt)
    try:
        out, tol = gemm(torch.float32), 1e-3
    except (NotImplementedError, RuntimeError):
        out, tol = gemm(torch.bfloat16), 1e-2      # bf16 output rounding (2^-8 relative)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    assert err <= tol * ref.abs().max().item(), err
    if gmode == "tensor":  # x-domain product = (A G_a)(B G_b)^T / (G_a G_b)
        xr = (a.float() @ b.float().t())
        y = out.float() / (qa.G.item() * qb.G.item())
        rel = ((y - xr).norm() / xr.norm()).item()
        assert rel < 0.15, rel                                  # NVFP4 quantisation error only
