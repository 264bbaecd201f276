"""Per-row global scale (mode "row"; "after per-row scaling"; SURVEY
NEXT(1)): each row is quantized as its own tensor with G_r = RN(2688 / max|x_r|).

Pins: (1) the definition, row by row, against mode "tensor" on 1-row
tensors; (2) an exact invariance: multiplying a row by 2^k changes G_r by
2^-k exactly and leaves y = RN(x G_r) -- hence every code, scale and error --
unchanged; (3) a zero row gets G_r = 1 and all-zero codes; (4) rows with equal
amax reproduce mode "tensor".
"""
import numpy as np
import torch

import ssgen


def _q(o, x, mode, w=(-8, 8)):
    return o.quantize(x, x.shape[0], x.shape[1], w[0], w[1], mode)


def test_row_mode_is_tensor_mode_per_row(oracle_lib):
    x = ssgen.generate("weight_outlier", 23, 96, seed=4, tid=41)
    full = _q(oracle_lib, x, "row")
    assert full.G.shape == (23,)
    for r in range(23):
        one = _q(oracle_lib, x[r:r + 1].contiguous(), "tensor")
        assert np.array_equal(full.codes[r], one.codes[0])
        assert np.array_equal(full.scales[r], one.scales[0])
        assert np.float32(full.G[r]) == np.float32(one.G)
        nbr = 96 // 16
        assert np.array_equal(full.err[r * nbr:(r + 1) * nbr].view(np.uint32), one.err.view(np.uint32))


def test_power_of_two_row_scaling_invariance(oracle_lib):
    x = ssgen.generate("gaussian", 8, 64, seed=5, tid=42).to(torch.float32)
    k = torch.tensor([0, 3, -5, 7, -2, 1, 10, -9], dtype=torch.float32)[:, None]
    xs = (x * torch.pow(2.0, k)).to(torch.bfloat16)        # exact: power-of-two scaling
    a, b = _q(oracle_lib, x.to(torch.bfloat16), "row"), _q(oracle_lib, xs, "row")
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.scales, b.scales)
    assert np.array_equal(a.err.view(np.uint32), b.err.view(np.uint32))
    assert np.array_equal(b.G, (a.G * np.power(2.0, -k.numpy()[:, 0])).astype(np.float32))


def test_zero_row(oracle_lib):
    x = ssgen.generate("gaussian", 3, 32, seed=6, tid=43)
    x[1] = 0
    r = _q(oracle_lib, x, "row")
    assert r.G[1] == 1.0 and not r.codes[1].any() and not r.scales[1].any()


def test_equal_row_amax_matches_tensor_mode(oracle_lib):
    x = ssgen.generate("gaussian", 6, 48, seed=7, tid=44).to(torch.float32)
    x[:, 5] = 3.0                                            # every row's amax is 3.0
    x = x.clamp(-2.9, 2.9)
    x[:, 5] = 3.0
    x = x.to(torch.bfloat16)
    a, b = _q(oracle_lib, x, "row"), _q(oracle_lib, x, "tensor")
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.scales, b.scales)
    assert np.all(a.G == np.float32(b.G))
