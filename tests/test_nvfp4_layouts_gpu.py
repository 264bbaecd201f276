"""SURVEY NEXT(1) on the GPU: per-row global scale and the tensor-core scale layout.

- SS_GLOBAL_ROW: codes, scales, per-block errors and the per-row G array are
  bit-exact against the oracle's mode "row" (each row its own tensor, R9).
- SS_SCALE_SWIZZLED: the scale bytes equal the oracle's linear scales placed
  by the block-scaled MMA layout (R15b).  The index function below is this
  test's own; it is checked against torch's reference `to_blocked`
  (torch.testing._internal.common_quantized), padding bytes must be zero.
- Dequantization reads both layouts and per-row G.
- The outputs are directly consumable: cuBLASLt's NVFP4 GEMM
  (torch.nn.functional.scaled_mm, BlockWise1x16 + SWIZZLE_32_4_4) on our
  codes and swizzled scales reproduces the FP32 product of the dequantized
  operands.
"""
import numpy as np
import pytest
import torch

import ssgen

pytestmark = pytest.mark.gpu

SHAPES = [(37, 16), (129, 128), (300, 96), (257, 4096), (5, 12288), (128, 64)]


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def blocked(lin: np.ndarray) -> np.ndarray:
    """Our statement of the layout: 512-B tiles of 128 rows x 4 scale columns,
    tile (rb, cb) at (rb * ceil(ncol/4) + cb) * 512, byte (r%32)*16 + (r//32%4)*4 + c%4."""
    rows, ncol = lin.shape
    nrb, ncb = -(-rows // 128), -(-ncol // 4)
    out = np.zeros(nrb * ncb * 512, np.uint8)
    r, c = np.meshgrid(np.arange(rows), np.arange(ncol), indexing="ij")
    off = ((r // 128) * ncb + c // 4) * 512 + (r % 32) * 16 + ((r // 32) % 4) * 4 + c % 4
    out[off.ravel()] = lin.ravel()
    return out


def test_layout_statement_matches_torch_reference():
    from torch.testing._internal.common_quantized import to_blocked
    rng = np.random.default_rng(0)
    for rows, ncol in [(1, 1), (37, 6), (128, 4), (257, 256), (300, 13)]:
        lin = rng.integers(0, 127, (rows, ncol), dtype=np.uint8)
        ref = to_blocked(torch.from_numpy(lin)).numpy()
        assert np.array_equal(blocked(lin), ref)


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
    try:
        out = F.scaled_mm(qa.codes.view(torch.float4_e2m1fn_x2), qb.codes.view(torch.float4_e2m1fn_x2).t(),
                          qa.scales.view(torch.float8_e4m3fn), F.ScalingType.BlockWise1x16,
                          qb.scales.view(torch.float8_e4m3fn), F.ScalingType.BlockWise1x16,
                          swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                          output_dtype=torch.float32)
    except (NotImplementedError, RuntimeError) as e:
        pytest.skip("cuBLASLt NVFP4 GEMM unavailable: %s" % str(e)[:200])
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err
    if gmode == "tensor":  # x-domain product = (A G_a)(B G_b)^T / (G_a G_b)
        xr = (a.float() @ b.float().t())
        y = out.float() / (qa.G.item() * qb.G.item())
        rel = ((y - xr).norm() / xr.norm()).item()
        assert rel < 0.15, rel                                  # NVFP4 quantisation error only
