"""Small single tensors (<= 2^19 NVFP4 blocks) run through quant_small_kernel:
one thread per block over the block-search device routine.
Its outputs must equal the persistent kernel's bit for bit.  The persistent
path is forced by quantizing the same tensor in a batch with a second, tiny
tensor (the small path takes single tensors only; ss_quantize_plan confirms
which path each call takes), including the FP64 error sums' determinism
across repeated calls.  Oracle parity of the small path is covered by the
single-tensor tests of test_parity_gpu.py, which take it."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [("gaussian", 37, 48, -8, 8, "tensor"), ("student_t", 513, 1024, -2, 6, "tensor"),
         ("weight_outlier", 256, 4096, -3, 5, "tensor"), ("kv_k", 100, 128, 0, 0, "none"),
         ("gaussian", 1024, 1024, -126, 126, "tensor"), ("gaussian", 4096, 4096, -8, 8, "tensor"),
         ("student_t", 3, 16, -1, 1, "device_amax")]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "%s-%dx%d-%d:%d-%s" % c)
def test_small_path_equals_persistent(case):
    import ssgen
    import paper_2605_12464_b200 as ss
    kind, rows, cols, lo, hi, gm = case
    x = ssgen.generate(kind, rows, cols, seed=77, tid=rows, device="cuda")
    tiny = ssgen.generate("gaussian", 1, 16, seed=78, tid=1, device="cuda")
    assert ss.plan([(rows, cols)], fmin=lo, fmax=hi, gmode=gm).small_path == (rows * cols // 16 <= 1 << 19)
    assert ss.plan([(rows, cols), (1, 16)], fmin=lo, fmax=hi, gmode=gm).small_path == 0
    amax = ss.tensor_amax_batched([x, tiny]) if gm == "device_amax" else None
    a = ss.quantize(x, fmin=lo, fmax=hi, gmode=gm, amax=amax)                 # small path
    outs = [ss.alloc_out(x), ss.alloc_out(tiny)]
    ss.quantize_batched([x, tiny], outs, fmin=lo, fmax=hi, gmode=gm, amax=amax)  # persistent kernel
    torch.cuda.synchronize()
    b = outs[0]
    for f in ("codes", "scales", "err", "offsets", "G"):
        assert torch.equal(getattr(a, f).view(torch.uint8), getattr(b, f).view(torch.uint8)), f
    # different fixed summation trees: equal to ~1e-15 relative
    np.testing.assert_allclose(a.sums.cpu().numpy(), b.sums.cpu().numpy(), rtol=1e-12, atol=0)


def test_small_path_sums_deterministic():
    import ssgen
    import paper_2605_12464_b200 as ss
    x = ssgen.generate("student_t", 2048, 2048, seed=5, tid=1, device="cuda")
    s0 = ss.quantize(x, radius=8).sums.clone()
    for _ in range(3):
        assert torch.equal(ss.quantize(x, radius=8).sums, s0)
