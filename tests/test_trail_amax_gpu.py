"""Trailing amax: a per-tensor-G call over >= 2^26 elements
runs as a chain of quantize launches; launch 0 computes its own small batch's
amax (the fused amax warps of §4.2a) and every launch's search warps fold the
NEXT batch's amax (a2) after each scheduling unit.  The outputs must
equal, bit for bit, the separate path (ss_tensor_amax_batched +
SS_GLOBAL_DEVICE_AMAX); every tensor's G must equal the oracle's
RN(2688 / amax) from the oracle's own amax, and sampled rows of every tensor
the oracle's quantization under that amax."""
import numpy as np
import pytest
import torch

import oracle
import ssgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200 import build
    build.build()
    return ss


def _batch(seed):
    """~100 M elements over 60 tensors of mixed shape and kind, with an empty
    tensor, an all-zero tensor and one-row tensors in the later batches."""
    rng = np.random.default_rng(seed)
    kinds = ["gaussian", "student_t", "weight_outlier", "kv_k"]
    xs = []
    for i in range(60):
        rows = int(rng.choice([1, 96, 512, 1024, 2304, 4096]))
        cols = 16 * int(rng.choice([64, 256, 257]))
        xs.append(ssgen.generate(kinds[i % 4], rows, cols, seed=seed, tid=i, device="cuda"))
    xs[41] = torch.zeros(0, 4096, dtype=torch.bfloat16, device="cuda")
    xs[47] = torch.zeros(300, 1024, dtype=torch.bfloat16, device="cuda")
    return xs


def _run(ss, xs, fmin, fmax, fused):
    outs = [ss.alloc_out(x) for x in xs]
    if fused:
        ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode="tensor")
    else:
        amax = ss.tensor_amax_batched(xs)
        ss.quantize_batched(xs, outs, fmin=fmin, fmax=fmax, gmode="device_amax", amax=amax)
    return outs, ss.device_status()


def _same(a, b):
    for k, (oa, ob) in enumerate(zip(a, b)):
        if oa.codes.numel() == 0:  # an empty tensor's G is not written
            continue
        for f in ("codes", "scales", "err", "offsets", "sums", "G"):
            x, y = getattr(oa, f), getattr(ob, f)
            if x is None:
                continue
            assert torch.equal(x.view(torch.uint8) if x.dtype != torch.uint8 else x,
                               y.view(torch.uint8) if y.dtype != torch.uint8 else y), (k, f)


@pytest.mark.parametrize("window", [(-8, 8), (-2, 6), (-16, 16)])
def test_trail_equals_separate_and_oracle(ss, window):
    xs = _batch(seed=11)
    n = sum(x.numel() for x in xs)
    assert n >= 1 << 26
    pl = ss.plan([tuple(x.shape) for x in xs], fmin=window[0], fmax=window[1], gmode="tensor")
    assert pl.amax_fused == 1 and pl.trail_batches > 2, "the call must take the trailing-amax path"
    a, fa = _run(ss, xs, *window, fused=True)
    b, fb = _run(ss, xs, *window, fused=False)
    torch.cuda.synchronize()
    assert fa == fb == 0
    _same(a, b)
    rng = np.random.default_rng(3)
    for k, x in enumerate(xs):
        if x.numel() == 0:
            continue
        xc = x.cpu()
        ab = oracle.tensor_amax(xc)
        g = oracle.global_scale(1, ab)
        assert np.float32(a[k].G.item()) == np.float32(g), k
        r0 = int(rng.integers(0, x.shape[0]))
        r1 = min(x.shape[0], r0 + 2)
        ref = oracle.quantize(xc[r0:r1], r1 - r0, x.shape[1], window[0], window[1], "given", amax_bits=ab)
        assert np.array_equal(a[k].codes[r0:r1].cpu().numpy(), ref.codes), k
        assert np.array_equal(a[k].scales[r0:r1].cpu().numpy(), ref.scales), k


@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_trail_nonfinite_in_later_batch(ss, bad):
    """A non-finite value in a tensor whose amax a previous launch folded
    raises the flag and gives that tensor G = 1 (R14), as the separate path."""
    xs = _batch(seed=12)
    xs[55] = xs[55].clone()
    xs[55][xs[55].shape[0] // 2, 17] = bad
    a, fa = _run(ss, xs, -8, 8, fused=True)
    b, fb = _run(ss, xs, -8, 8, fused=False)
    torch.cuda.synchronize()
    assert fa == fb and fa & 1
    assert a[55].G.item() == 1.0
    _same(a, b)


def test_trail_repeated_calls(ss):
    """Back-to-back calls re-arm every counter (the amax slots are re-zeroed per call)."""
    xs = _batch(seed=13)
    ref, _ = _run(ss, xs, -8, 8, fused=False)
    for _ in range(3):
        a, fa = _run(ss, xs, -8, 8, fused=True)
        assert fa == 0
        _same(a, ref)


def test_trail_skewed_sizes_self_amax(ss):
    """Small tensors followed by one that alone exceeds twice the batch before
    it: that batch computes its own amax (too few warps would fold it) in a
    2-launch chain; the call equals the separate path and the oracle's G."""
    xs = [ssgen.generate("gaussian", 1, 64, seed=14, tid=i, device="cuda") for i in range(30)]
    xs.append(ssgen.generate("student_t", 16384, 4096, seed=14, tid=99, device="cuda"))
    pl = ss.plan([tuple(x.shape) for x in xs], fmin=-8, fmax=8, gmode="tensor")
    assert pl.amax_fused == 1 and pl.trail_batches == 2
    a, fa = _run(ss, xs, -8, 8, fused=True)
    b, fb = _run(ss, xs, -8, 8, fused=False)
    torch.cuda.synchronize()
    assert fa == fb == 0
    _same(a, b)
    assert np.float32(a[30].G.item()) == np.float32(oracle.global_scale(1, oracle.tensor_amax(xs[30].cpu())))


def test_trail_self_batch_mid_chain(ss):
    """A chain whose middle batch starts with a tensor over twice its
    predecessor: batches before and after it fold, it computes its own amax."""
    xs = [ssgen.generate("gaussian", 2048, 4096, seed=15, tid=i, device="cuda") for i in range(4)]
    xs.append(ssgen.generate("student_t", 16384, 4096, seed=15, tid=50, device="cuda"))
    xs += [ssgen.generate("kv_k", 4096, 4096, seed=15, tid=60 + i, device="cuda") for i in range(6)]
    pl = ss.plan([tuple(x.shape) for x in xs], fmin=-8, fmax=8, gmode="tensor")
    assert pl.amax_fused == 1 and pl.trail_batches > 2
    a, fa = _run(ss, xs, -8, 8, fused=True)
    b, fb = _run(ss, xs, -8, 8, fused=False)
    torch.cuda.synchronize()
    assert fa == fb == 0
    _same(a, b)
