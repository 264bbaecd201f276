"""Seeded randomized parity: many small random configurations through the C ABI
against the oracle -- format x window x global-scale mode x scale layout x
batch composition x data family, with ragged shapes.  Complements the
structured tests by covering their interactions."""
import os
import sys

import numpy as np
import pytest
import torch

import ssgen

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_scale_layout import blocked  # noqa: E402

pytestmark = pytest.mark.gpu

FMT_BS = {"nvfp4": 16, "mxfp4": 32, "mxfp6_e2m3": 32, "nvfp6_e2m3": 16, "nvfp4_b64": 64,
          "nvfp4_b256": 256}
KINDS = ["gaussian", "student_t", "weight_outlier", "kv_k"]


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def _case(rng):
    fmt = rng.choice(list(FMT_BS))
    bs = FMT_BS[fmt]
    mx = fmt.startswith("mx")
    lim = 254 if mx else 126
    fmin = -int(rng.choice([0, 1, 2, 3, 8, 17, lim]))
    fmax = int(rng.choice([0, 1, 2, 5, 8, 16, lim]))
    gmode = "none" if mx else str(rng.choice(["none", "tensor", "row", "device_amax"]))
    layout = str(rng.choice(["linear", "swizzled"]))
    n = int(rng.integers(1, 5))
    shapes = [(int(rng.integers(1, 300)), bs * int(rng.integers(1, 9))) for _ in range(n)]
    kinds = [str(rng.choice(KINDS)) for _ in range(n)]
    return fmt, fmin, fmax, gmode, layout, shapes, kinds


@pytest.mark.parametrize("seed", range(40))
def test_random_configuration(ss, oracle_lib, seed):
    rng = np.random.default_rng(1000 + seed)
    fmt, fmin, fmax, gmode, layout, shapes, kinds = _case(rng)
    xs = [ssgen.generate(k, r, c, seed=seed, tid=i) for i, (k, (r, c)) in enumerate(zip(kinds, shapes))]
    if seed % 5 == 0:                                  # sprinkle exact zeros and tiny values
        xs[0][0, :] = 0
        xs[-1][-1, :16] = 1e-30
    xd = [x.cuda() for x in xs]
    outs = [ss.alloc_out(x, scale_layout=layout, gmode=gmode, fmt=fmt) for x in xd]
    amax = ss.tensor_amax_batched(xd) if gmode == "device_amax" else None
    ss.quantize_batched(xd, outs, fmin=fmin, fmax=fmax, gmode=gmode, amax=amax,
                        scale_layout=layout, fmt=fmt)
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        r, c = x.shape
        ref = oracle_lib.quantize_fmt(x, r, c, fmin, fmax, fmt,
                                      "tensor" if gmode == "device_amax" else gmode)
        assert np.array_equal(o.codes.cpu().numpy(), ref.codes)
        scales = ref.scales if layout == "linear" else blocked(ref.scales)
        assert np.array_equal(o.scales.cpu().numpy().reshape(-1), scales.reshape(-1))
        assert np.array_equal(o.offsets.cpu().numpy(), ref.offsets)
        assert np.array_equal(o.err.cpu().numpy().view(np.uint32), ref.err.view(np.uint32))
        s = o.sums.cpu().numpy()
        if np.isfinite(ref.sums[0]):
            assert abs(s[0] - ref.sums[0]) <= 1e-9 * abs(ref.sums[0]) + 1e-300
        if gmode in ("tensor", "device_amax"):
            assert o.G.item() == np.float32(ref.G)
        elif gmode == "row":
            assert np.array_equal(o.G.cpu().numpy().view(np.uint32), ref.G.view(np.uint32))

