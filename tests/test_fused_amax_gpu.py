"""Fused amax (quant_kernel<..., AF>): SS_GLOBAL_TENSOR calls
whose window has >= 4 offsets run the tensor amax (a2) inside the
quantize launch.  Their outputs must equal, bit for bit, the separate path
(ss_tensor_amax_batched + SS_GLOBAL_DEVICE_AMAX) on batches that cross the
128-tensor launch split, ragged / one-block / all-zero / subnormal-only
tensors, and the non-finite flag (R14).  Oracle parity of the fused path is
covered by every TENSOR-mode test in test_parity_gpu.py / test_random_gpu.py."""
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


def _batch(n, seed):
    rng = np.random.default_rng(seed)
    kinds = ["gaussian", "student_t", "weight_outlier", "kv_k"]
    xs = []
    for i in range(n):
        rows = int(rng.choice([1, 3, 17, 64, 129, 300]))
        cols = 16 * int(rng.choice([1, 2, 5, 64, 130]))
        xs.append(ssgen.generate(kinds[i % 4], rows, cols, seed=seed, tid=i, device="cuda"))
    return xs


def _run(ss, xs, fmin, fmax, fused):
    outs = [ss.alloc_out(x) for x in xs]
    if fused:
        ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode="tensor")
    else:
        amax = ss.tensor_amax_batched(xs)
        ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode="device_amax", amax=amax)
    flags = ss.device_status()
    return outs, flags


def _same(a, b):
    for oa, ob in zip(a, b):
        for f in ("codes", "scales", "err", "offsets", "sums", "G"):
            x, y = getattr(oa, f), getattr(ob, f)
            assert torch.equal(x.view(torch.uint8) if x.dtype != torch.uint8 else x,
                               y.view(torch.uint8) if y.dtype != torch.uint8 else y), f


@pytest.mark.parametrize("window", [(-8, 8), (-2, 6), (-2, 2), (-16, 16), (-126, 126), (-1, 1)])
def test_fused_equals_separate(ss, window):
    xs = _batch(150, seed=5)             # two launches (128 + 22 tensors)
    a, fa = _run(ss, xs, *window, fused=True)
    b, fb = _run(ss, xs, *window, fused=False)
    assert fa == fb == 0
    _same(a, b)


def test_fused_corner_tensors(ss):
    z = torch.zeros(5, 48, dtype=torch.bfloat16, device="cuda")                 # all zero: G = 1
    sub = torch.full((2, 32), 2.0 ** -130, dtype=torch.bfloat16, device="cuda")  # bf16 subnormals only
    sub[1, 3] = -(2.0 ** -133)
    one = torch.tensor([[0.0] * 15 + [-3.0]], dtype=torch.bfloat16, device="cuda")  # one block, amax < 0 value
    adv = ssgen.adversarial_rows().to("cuda")
    big = ssgen.generate("gaussian", 1024, 4096, seed=3, tid=9, device="cuda")     # many amax units
    xs = [z, sub, one, adv, big, z.clone()]
    a, fa = _run(ss, xs, -8, 8, fused=True)
    b, fb = _run(ss, xs, -8, 8, fused=False)
    assert fa == fb
    _same(a, b)
    assert a[0].G.item() == 1.0 and a[2].G.item() == np.float32(2688.0) / np.float32(3.0)


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_fused_nonfinite_flag(ss, bad):
    xs = [torch.ones(1, 16, dtype=torch.bfloat16, device="cuda")] + _batch(6, seed=8)   # small first: fused
    xs[3] = xs[3].clone()
    xs[3].view(-1)[xs[3].numel() // 2] = bad
    a, fa = _run(ss, xs, -8, 8, fused=True)
    b, fb = _run(ss, xs, -8, 8, fused=False)
    assert fa == fb and (fa & 1) == 1      # SS_FLAG_NONFINITE, G falls back to 1 (R14)
    assert a[3].G.item() == 1.0
    _same(a[:3] + a[4:], b[:3] + b[4:])


def test_fused_repeated_calls_rearm(ss):
    """The in-kernel counters re-arm themselves: back-to-back calls on one
    stream and calls with a different batch size give the same outputs."""
    xs = _batch(20, seed=12)
    ref, _ = _run(ss, xs, -4, 4, fused=False)
    for k in (20, 3, 20, 130):
        ys = xs[:k] if k <= 20 else (xs * 7)[:k]
        out, f = _run(ss, ys, -4, 4, fused=True)
        assert f == 0
        _same(out[:min(k, 20)], ref[:min(k, 20)])


@pytest.mark.parametrize("window", [(-8, 8), (0, 0)])
def test_next_amax_call(ss, window):
    """ss_quantize_nvfp4_batched_next_amax: this group's outputs equal the
    two-launch path, and the next group's local amaxes equal
    ss_tensor_amax_batched (empty next tensors give 0; NaN propagates)."""
    xs = _batch(40, seed=31)
    nxt = _batch(12, seed=32) + [torch.zeros(0, 16, dtype=torch.bfloat16, device="cuda")]
    nxt[5] = nxt[5].clone()
    nxt[5].view(-1)[7] = float("nan")
    amax = ss.tensor_amax_batched(xs)
    ref, _ = _run(ss, xs, *window, fused=False)
    outs = [ss.alloc_out(x) for x in xs]
    next_amax = torch.full((len(nxt),), 12345, dtype=torch.int32, device="cuda")
    ss.quantize_batched_next_amax(xs, outs, amax, nxt, next_amax, fmin=window[0], fmax=window[1])
    torch.cuda.synchronize()
    _same(outs, ref)
    want = ss.tensor_amax_batched(nxt)
    got = next_amax.cpu().numpy().view(np.uint32)
    exp = want.cpu().numpy().view(np.uint32)
    for j in range(len(nxt)):
        if j == 5:
            assert got[j] >= 0x7F800000 and exp[j] >= 0x7F800000   # NaN sorts above every finite value
        else:
            assert got[j] == exp[j], j
    # no tensors to quantize: only the next amaxes (separate launch)
    next_amax.fill_(7)
    ss.quantize_batched_next_amax([], [], amax, nxt[:3], next_amax[:3], radius=8)
    torch.cuda.synchronize()
    assert np.array_equal(next_amax[:3].cpu().numpy(), want[:3].cpu().numpy())
