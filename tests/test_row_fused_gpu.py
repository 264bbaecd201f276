"""Row-fused per-row global scale on the GPU (SS_GLOBAL_ROW, R9b).

For rows of 64..512 half-blocks (1024..8192 elements) the quantize kernel
computes each row's amax itself (one warp pass over the row, then the row's
chunks) instead of a separate rowscale pass.  Everything stays bit-exact
against the oracle's mode "row": codes, scales, offsets, per-block errors and
the G_r array, across
- exact and ragged last chunks (cols % 1024 != 0),
- rows cut into units of one chunk (few rows) and of several chunks (many rows),
- the size limits on both sides (hpr 63 / 64, 512 / 513: the two-pass path),
- fixed and runtime windows, both scale layouts, E2M3 values and 64/256 blocks,
- batches mixing fused, two-pass and per-tensor tensors, with error sums.
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

# (rows, cols): fused unless hpr = cols / 16 is outside [64, 512]
SHAPES = [(64, 1024), (33, 1040), (5, 8192), (300, 8192), (41, 3008), (2, 2048), (1, 1024),
          (130, 4096), (3, 8208), (9, 1008)]
WINDOWS = [(-8, 8), (0, 0), (-2, 6), (-1, 1), (-126, 126)]


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def _cmp(g, ref, swz=False):
    assert np.array_equal(g.codes.cpu().numpy(), ref.codes)
    sc = blocked(ref.scales) if swz else ref.scales
    assert np.array_equal(g.scales.cpu().numpy(), sc)
    assert np.array_equal(g.offsets.cpu().numpy(), ref.offsets)
    assert np.array_equal(g.err.cpu().numpy().view(np.uint32), ref.err.view(np.uint32))
    assert np.array_equal(g.G.cpu().numpy().view(np.uint32), ref.G.view(np.uint32))
    s = g.sums.cpu().numpy()
    for k in range(2):
        assert abs(s[k] - ref.sums[k]) <= 1e-9 * abs(ref.sums[k]) + 1e-300


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("win", WINDOWS)
def test_row_fused_parity(ss, oracle_lib, shape, win):
    x = ssgen.generate("student_t", *shape, seed=41, tid=shape[0] * 5 + shape[1])
    g = ss.quantize(x.cuda(), fmin=win[0], fmax=win[1], gmode="row")
    torch.cuda.synchronize()
    _cmp(g, oracle_lib.quantize(x, *shape, win[0], win[1], "row"))


@pytest.mark.parametrize("shape", [(130, 4096), (41, 3008), (5, 8192)])
def test_row_fused_swizzled(ss, oracle_lib, shape):
    x = ssgen.generate("weight_outlier", *shape, seed=42, tid=shape[1])
    g = ss.quantize(x.cuda(), radius=8, gmode="row", scale_layout="swizzled")
    torch.cuda.synchronize()
    _cmp(g, oracle_lib.quantize(x, *shape, -8, 8, "row"), swz=True)


@pytest.mark.parametrize("shape", [(4096, 8192), (12000, 8192), (16384, 4096)])
def test_row_fused_unit_split(ss, oracle_lib, shape):
    """Large row counts: the library gives a scheduling unit several chunks of
    a row (cpu > 1, about 6 units per warp of the grid), while the shapes
    above give one chunk per unit (each unit recomputes G_r)."""
    assert ss.plan([shape], radius=8, gmode="row").row_fused == 1
    x = ssgen.generate("gaussian", *shape, seed=43, tid=shape[0])
    g = ss.quantize(x.cuda(), radius=8, gmode="row")
    torch.cuda.synchronize()
    _cmp(g, oracle_lib.quantize(x, *shape, -8, 8, "row"))


@pytest.mark.parametrize("fmt", ["nvfp6_e2m3", "nvfp4_b64", "nvfp4_b256"])
def test_row_fused_formats(ss, oracle_lib, fmt):
    shape = (37, 2048)
    x = ssgen.generate("student_t", *shape, seed=44, tid=len(fmt))
    for w in [(0, 0), (-2, 2), (-126, 126)]:
        g = ss.quantize(x.cuda(), fmin=w[0], fmax=w[1], gmode="row", fmt=fmt)
        torch.cuda.synchronize()
        _cmp(g, oracle_lib.quantize_fmt(x, *shape, w[0], w[1], fmt, "row"))


def test_row_fused_batched_mixed(ss, oracle_lib):
    shapes = [(64, 1024), (9, 1008), (33, 1040), (3, 8208), (300, 8192), (2, 16)]
    xs = [ssgen.generate("student_t", r, c, seed=45, tid=k) for k, (r, c) in enumerate(shapes)]
    xd = [x.cuda() for x in xs]
    outs = [ss.alloc_out(x, gmode="row") for x in xd]
    ss.quantize_batched(xd, outs, radius=8, gmode="row")
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        _cmp(o, oracle_lib.quantize(x, *x.shape, -8, 8, "row"))


def test_row_fused_special_rows(ss, oracle_lib):
    """All-zero rows (G_r = 1), a row with one huge value, tiny subnormal-range rows."""
    rows, cols = 6, 2048
    x = ssgen.generate("gaussian", rows, cols, seed=46, tid=1).float()
    x[1] = 0.0
    x[2, 1000] = 3.0e38
    x[3] *= 1e-30
    x = x.to(torch.bfloat16)
    g = ss.quantize(x.cuda(), radius=8, gmode="row")
    torch.cuda.synchronize()
    _cmp(g, oracle_lib.quantize(x, rows, cols, -8, 8, "row"))
