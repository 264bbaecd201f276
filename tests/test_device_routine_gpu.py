"""The one-thread block-search routine (include/ss_device.cuh) through its
FP32-input consumer ss_quantize_nvfp4_f32 (the search a
fused kernel such as FP4 attention reuses).

* bf16-representable inputs with the same G: bit-identical to the bf16 path
  (ss_quantize_nvfp4_ex) for every output.
* general FP32 inputs (not bf16-representable: full 24-bit mantissas, softmax
  probabilities as attention's P, exact E2M1 midpoints at FP32 precision):
  per block against the oracle's Algorithm 1 (oracle.search_block).
"""
import numpy as np
import pytest
import torch

import ssgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def _nibbles(codes_row):
    b = codes_row.astype(np.uint8)
    return np.stack([b & 0xF, b >> 4], axis=-1).reshape(-1)


@pytest.mark.parametrize("window", [(-8, 8), (-2, 6), (-1, 1), (0, 0), (-3, 5), (-126, 126)])
@pytest.mark.parametrize("kind", ["gaussian", "student_t", "weight_outlier"])
def test_f32_equals_bf16_path(ss, window, kind):
    x = ssgen.generate(kind, 257, 384, seed=21, tid=3, device="cuda")
    ref = ss.quantize(x, fmin=window[0], fmax=window[1], gmode="tensor")
    got = ss.quantize_f32(x.float().contiguous(), fmin=window[0], fmax=window[1], G=ref.G)
    torch.cuda.synchronize()
    assert torch.equal(got.codes, ref.codes)
    assert torch.equal(got.scales, ref.scales)
    assert torch.equal(got.err.view(torch.int32), ref.err.view(torch.int32))
    assert torch.equal(got.offsets, ref.offsets)
    assert ss.device_status() == 0


def _f32_cases(rng):
    n = 4096
    fam = [
        rng.standard_normal((n, 16)),                                          # full FP32 mantissas
        rng.standard_t(3, (n, 16)) * np.exp(rng.uniform(-20, 8, (n, 1))),      # wide dynamic range
        np.exp(rng.standard_normal((n, 16)) * 2 - 3).clip(0, 1),               # softmax-like P in [0, 1]
        (rng.integers(-12, 13, (n, 16)) / 2.0) * 2.0 ** rng.integers(-8, 8, (n, 1)),  # midpoints / ties
    ]
    x = np.concatenate(fam).astype(np.float32)
    x[:, 0] += np.float32(2.0 ** -20) * (x[:, 0] != 0)                         # off the bf16 grid
    return x


@pytest.mark.parametrize("window", [(-8, 8), (-2, 6), (-5, 3)])
def test_f32_against_oracle(ss, oracle_lib, window):
    rng = np.random.default_rng(33)
    x = _f32_cases(rng)                                  # [blocks][16]
    G = np.float32(448.0 * 6.0)                          # a fixed global scale, as for attention's P
    xd = torch.from_numpy(x.reshape(-1, 64)).cuda()
    g = torch.tensor([G], dtype=torch.float32, device="cuda")
    got = ss.quantize_f32(xd, fmin=window[0], fmax=window[1], G=g)
    torch.cuda.synchronize()
    codes = got.codes.cpu().numpy().reshape(-1, 8)
    scales = got.scales.cpu().numpy().reshape(-1)
    err = got.err.cpu().numpy()
    offs = got.offsets.cpu().numpy()
    y = (x * G).astype(np.float32)                       # y = RN(x * G) (R9), elementwise fp32
    for b in range(0, len(x), 7):                        # every 7th block, all four families
        r = oracle_lib.search_block(y[b], *window)
        assert scales[b] == r.cstar and offs[b] == r.fstar, b
        assert np.array_equal(_nibbles(codes[b]), r.nib), b
        assert err[b, 0] == np.float32(r.err_best) and err[b, 1] == np.float32(r.err_base), b


def test_f32_nonfinite_flag_and_edges(ss):
    x = torch.zeros(3, 32, dtype=torch.float32, device="cuda")
    got = ss.quantize_f32(x, radius=8)                   # all zero: zero scale, zero nibbles (R3)
    torch.cuda.synchronize()
    assert int(got.scales.max()) == 0 and int(got.codes.max()) == 0
    assert ss.device_status() == 0
    x[1, 5] = float("nan")
    ss.quantize_f32(x, radius=8)
    assert ss.device_status() & 1
    empty = torch.zeros(0, 16, dtype=torch.float32, device="cuda")
    ss.quantize_f32(empty, radius=8)
    assert ss.device_status() == 0
