"""Small single tensors (<= SS_SMALL_MAX_BLOCKS NVFP4 blocks) run through
quant_small_kernel: one thread per block over the block-search device
routine.  Its outputs must equal the persistent kernel's bit
for bit (a subprocess with SS_SMALL_MAX_BLOCKS=0 forces the persistent path),
including the FP64 error sums' determinism across repeated calls.  Oracle
parity of the small path is covered by the single-tensor tests of
test_parity_gpu.py, which now take it."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [("gaussian", 37, 48, -8, 8, "tensor"), ("student_t", 513, 1024, -2, 6, "tensor"),
         ("weight_outlier", 256, 4096, -3, 5, "tensor"), ("kv_k", 100, 128, 0, 0, "none"),
         ("gaussian", 1024, 1024, -126, 126, "tensor"), ("gaussian", 4096, 4096, -8, 8, "tensor"),
         ("student_t", 3, 16, -1, 1, "device_amax")]

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import ssgen, paper_2605_12464_b200 as ss
out = {}
for k, (kind, rows, cols, lo, hi, gm) in enumerate(%r):
    x = ssgen.generate(kind, rows, cols, seed=77, tid=k, device="cuda")
    amax = ss.tensor_amax(x) if gm == "device_amax" else None
    o = ss.quantize(x, fmin=lo, fmax=hi, gmode=gm, amax=amax)
    for f in ("codes", "scales", "err", "offsets", "sums", "G"):
        out["%%d_%%s" %% (k, f)] = getattr(o, f).cpu().numpy()
np.savez(sys.argv[1], **out)
"""


def _run(env_small, path):
    env = dict(os.environ)
    env["SS_SMALL_MAX_BLOCKS"] = str(env_small)
    subprocess.run([sys.executable, "-c", SCRIPT % (ROOT, CASES), path], check=True, env=env, timeout=600)
    return np.load(path)


def test_small_path_equals_persistent(tmp_path):
    a = _run(1 << 30, str(tmp_path / "small.npz"))
    b = _run(0, str(tmp_path / "persistent.npz"))
    assert set(a.files) == set(b.files)
    for f in a.files:
        if f.endswith("_sums"):      # different fixed summation trees: equal to ~1e-15 relative
            np.testing.assert_allclose(a[f], b[f], rtol=1e-12, atol=0)
        else:
            assert np.array_equal(a[f].view(np.uint8), b[f].view(np.uint8)), f


def test_small_path_sums_deterministic():
    import ssgen
    import paper_2605_12464_b200 as ss
    x = ssgen.generate("student_t", 2048, 2048, seed=5, tid=1, device="cuda")
    s0 = ss.quantize(x, radius=8).sums.clone()
    for _ in range(3):
        assert torch.equal(ss.quantize(x, radius=8).sums, s0)
