"""Generic ExMy block formats on the GPU (fig:nvfp-scale,
fig:nvfp-val, fig:mxfp P:237-260; reading R21) against the oracle's
generic search (tests/test_oracle_gen.py pins it), element by element: value
codes, scale codes, offsets, per-block errors and G bit-exact, sums within
1e-9; dequantization bit-exact; the NVFP4 point equals the NVFP4 kernel.
"""
import numpy as np
import pytest
import torch

import ssgen

pytestmark = pytest.mark.gpu

# (value_e, value_m, scale_e, scale_m, block): the sweeps' corners and
# standard points (NVFP4, NVFP6, MXFP4, MXFP6, FP6 E3M2), subnormal-heavy
# and pure-power-of-two scales, 16- and 32-blocks
FORMATS = [(2, 1, 4, 3, 16), (2, 3, 4, 3, 16), (3, 2, 4, 3, 16), (1, 2, 4, 3, 16), (3, 0, 4, 3, 16),
           (4, 3, 4, 3, 16), (2, 1, 2, 3, 16), (2, 1, 3, 4, 16), (2, 1, 5, 2, 16), (2, 1, 6, 1, 16),
           (2, 1, 4, 0, 16), (2, 1, 7, 1, 16), (2, 1, 8, 0, 32), (2, 3, 8, 0, 32), (3, 2, 8, 0, 32),
           (1, 4, 8, 0, 32), (2, 1, 5, 0, 32), (2, 2, 3, 3, 32)]
SHAPES = [(37, 32), (129, 256), (64, 1024)]


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def _data(shape, seed):
    x = ssgen.generate("student_t", *shape, seed=seed, tid=shape[0] * 7 + shape[1])
    x[0, :32] = 0.0                                   # all-zero blocks (R3 / smallest scale)
    x[1, :32] = x[1, :32] * 1e-30                     # tiny blocks (subnormal scales, flushed values)
    return x


def _cmp(g, ref, G=True):
    assert np.array_equal(g.codes.cpu().numpy(), ref.codes)
    assert np.array_equal(g.scales.cpu().numpy(), ref.scales)
    assert np.array_equal(g.offsets.cpu().numpy(), ref.offsets)
    assert np.array_equal(g.err.cpu().numpy().view(np.uint32), ref.err.view(np.uint32))
    s = g.sums.cpu().numpy()
    for k in range(2):
        assert abs(s[k] - ref.sums[k]) <= 1e-9 * abs(ref.sums[k]) + 1e-300
    if G:
        assert np.float32(g.G.cpu().numpy()[0]).view(np.uint32) == np.float32(ref.G).view(np.uint32)


@pytest.mark.parametrize("fmt", FORMATS, ids=lambda f: "e%dm%d_ue%dm%d_b%d" % f)
def test_gen_parity(ss, oracle_lib, fmt):
    lim = (1 << (fmt[2] + fmt[3])) - 2
    for shape in SHAPES:
        if shape[1] % fmt[4]:
            continue
        x = _data(shape, 41)
        xc = x.cuda()
        gmodes = ("none",) if not np.isfinite(oracle_lib.gen_numer(*fmt[:4])) else ("tensor", "none")
        for gmode in gmodes:
            for w in [(0, 0), (-1, 1), (-3, 5), (-8, 8), (-lim, lim)]:
                g = ss.quantize_gen(xc, fmt, fmin=w[0], fmax=w[1], gmode=gmode)
                torch.cuda.synchronize()
                ref = oracle_lib.quantize_gen(x, *shape, w[0], w[1], fmt, gmode)
                _cmp(g, ref, G=gmode != "none")
                if w == (-8, 8):
                    G = g.G if gmode == "tensor" else None
                    d = ss.dequantize_gen(g.codes, g.scales, *shape, fmt, G)
                    torch.cuda.synchronize()
                    rd = oracle_lib.dequantize_gen(ref.codes, ref.scales, *shape, fmt,
                                                   ref.G if gmode == "tensor" else 1.0)
                    assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16), rd)


def test_gen_device_amax(ss, oracle_lib):
    x = _data((96, 512), 43)
    fmt = (3, 2, 5, 2, 16)
    amax = ss.tensor_amax(x.cuda())
    ab = int(amax.cpu().numpy().view(np.uint32)[0])
    g = ss.quantize_gen(x.cuda(), fmt, fmin=-4, fmax=6, gmode="device_amax", amax=amax)
    torch.cuda.synchronize()
    ref = oracle_lib.quantize_gen(x, 96, 512, -4, 6, fmt, "given", amax_bits=ab)
    _cmp(g, ref)


def test_gen_nvfp4_point_equals_nvfp4_kernel(ss):
    """The UE4M3 / E2M1 / 16 point of the sweep is the north-star path, bit for bit."""
    x = ssgen.generate("weight_outlier", 256, 2048, seed=5, tid=9).cuda()
    for w in ((-8, 8), (-2, 6), (0, 0)):
        a = ss.quantize_gen(x, (2, 1, 4, 3, 16), fmin=w[0], fmax=w[1], gmode="tensor")
        b = ss.quantize(x, fmin=w[0], fmax=w[1], gmode="tensor")
        torch.cuda.synchronize()
        pk = b.codes.cpu().numpy()
        nib = np.empty((256, 2048), np.uint8)
        nib[:, 0::2] = pk & 15
        nib[:, 1::2] = pk >> 4
        assert np.array_equal(a.codes.cpu().numpy(), nib)
        assert np.array_equal(a.scales.cpu().numpy(), b.scales.cpu().numpy())
        assert np.array_equal(a.err.cpu().numpy().view(np.uint32), b.err.cpu().numpy().view(np.uint32))
        assert np.array_equal(a.offsets.cpu().numpy(), b.offsets.cpu().numpy())


def test_gen_sampled_large(ss, oracle_lib):
    """A C3-row-shaped tensor (8 rows x 8192, 4096 blocks) at the sweep's widest scale format."""
    x = ssgen.generate("gaussian", 64, 8192, seed=7, tid=3)
    fmt = (2, 1, 5, 3, 16)
    g = ss.quantize_gen(x.cuda(), fmt, fmin=-16, fmax=16, gmode="tensor")
    torch.cuda.synchronize()
    ref = oracle_lib.quantize_gen(x, 64, 8192, -16, 16, fmt, "tensor")
    _cmp(g, ref)


def test_gen_argument_errors(ss):
    """Synchronous argument checks (no launch): bad formats, a global scale for UE8M0."""
    x = torch.zeros(16, 64, dtype=torch.bfloat16, device="cuda")
    for fmt in ((0, 3, 4, 3, 16), (2, 6, 4, 3, 16), (2, 1, 8, 1, 16), (2, 1, 4, 3, 48), (2, 1, 9, 0, 16)):
        with pytest.raises(ss.SSError):
            ss.quantize_gen(x, fmt, radius=2, gmode="none")
    with pytest.raises(ss.SSError):
        ss.quantize_gen(x, (2, 1, 8, 0, 32), radius=2, gmode="tensor")
