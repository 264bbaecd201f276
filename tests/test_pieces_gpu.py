"""Tensors over the kernels' 32-bit half-block index run as row pieces
(ss_api.cu quantize_core).  Two checks:

  - the piece logic at small sizes: a test build with a 4096-half-block piece
    limit (libss_piece.so, -DSS_MAX_PIECE_BLOCKS=4096) quantizes multi-piece
    tensors, batches, per-row G, both scale layouts and 32-element formats,
    every output against the oracle (tests/_piece_worker.py, own process);
  - one real tensor of 2^31 + 2^20 half-blocks (34 G elements, 68.7 GB bf16)
    through libss.so, sampled rows at and around the piece boundary against
    the oracle (skipped when the GPU has < 110 GB free).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_piece_path_small_limit():
    from paper_2605_12464_b200 import build
    build.build(variant="piece", defines=["SS_MAX_PIECE_BLOCKS=4096"])
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_piece_worker.py")],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "piece cases ok" in r.stdout


def test_tensor_over_2e31_half_blocks(oracle_lib):
    import paper_2605_12464_b200 as ss
    free, _ = torch.cuda.mem_get_info()
    if free < 110e9:
        pytest.skip("needs ~90 GB of free device memory")
    rows, cols = (1 << 20) + 1024, 32768          # 2^31 + 2^21 half-blocks
    x = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(20261017)
    for r0 in range(0, rows, 1 << 16):               # unit Gaussian, in chunks
        x[r0:r0 + (1 << 16)].normal_(generator=g)
    out = ss.alloc_out(x, want_err=False, want_offsets=False, want_sums=True, want_g=True)
    ss.quantize(x, fmin=-2, fmax=2, gmode="none", out=out)
    torch.cuda.synchronize()
    per_piece = ((1 << 31) - (1 << 16)) // (cols // 16)
    for r in (0, 1, per_piece - 1, per_piece, per_piece + 1, rows - 1):
        xr = x[r:r + 1].cpu()
        ref = oracle_lib.quantize(xr, 1, cols, -2, 2, "none")
        assert np.array_equal(out.codes[r].cpu().numpy(), ref.codes[0]), r
        assert np.array_equal(out.scales[r].cpu().numpy(), ref.scales[0]), r
    assert np.isfinite(out.sums.cpu().numpy()).all()
    del x, out
    torch.cuda.empty_cache()
