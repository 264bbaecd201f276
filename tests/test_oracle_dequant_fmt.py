"""Pin of the oracle's general dequantizer so_dequantize_fmt (P:154-162,
xhat = RNE_bf16(RN((q * s) / G))) against library decodes: ml_dtypes
float4_e2m1fn / float6_e2m3fn for the value codes, float8_e4m3fn for UE4M3
scales, the closed form 2^(c-127) for UE8M0 (R19), numpy binary32 division
and ml_dtypes' round-to-nearest-even bfloat16 cast.  Every format, a per-tensor
and a per-row global scale, every code (both signs, -0) and every scale code.
"""
import ml_dtypes
import numpy as np
import pytest

FMTS = ["nvfp4", "mxfp4", "mxfp6_e2m3", "nvfp6_e2m3", "nvfp4_b32", "nvfp4_b64", "nvfp4_b128", "nvfp4_b256"]


def _expected(codes_vals, scales, rows, cols, vf, sf, bs, G):
    q = codes_vals.astype(np.float32)                                  # [rows][cols] decoded values
    if sf == 0:
        s = scales.view(ml_dtypes.float8_e4m3fn).astype(np.float32)   # UE4M3 (R1, R2: codes 0..126)
    else:
        s = np.ldexp(np.float64(1.0), scales.astype(np.int32) - 127).astype(np.float32)  # UE8M0
    s_full = np.repeat(s, bs, axis=1)
    xs = (q * s_full).astype(np.float32)                                # exact: few significant bits
    g = np.asarray(G, np.float32).reshape(-1, 1) if np.ndim(G) else np.float32(G)
    y = (xs / g).astype(np.float32)                                    # binary32 RN division
    return y.astype(ml_dtypes.bfloat16).view(np.uint16)               # RNE to bf16


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("per_row", [False, True])
def test_dequantize_fmt_matches_library_decodes(oracle_lib, fmt, per_row):
    vf, sf, bs = oracle_lib.FORMATS[fmt]
    rng = np.random.default_rng(hash((fmt, per_row)) & 0xFFFF)
    rows, cols = 37, 4 * 256
    if vf == 0:
        nib = rng.integers(0, 16, (rows, cols), dtype=np.uint8)       # all 16 nibbles incl. -0 (0x8)
        vals = nib.view(ml_dtypes.float4_e2m1fn)
        codes = (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)  # low nibble = even element (R15)
    else:
        c6 = rng.integers(0, 64, (rows, cols), dtype=np.uint8)        # sign bit 5
        vals = c6.view(ml_dtypes.float6_e2m3fn)
        codes = c6
    hi = 126 if sf == 0 else 254
    scales = rng.integers(0, hi + 1, (rows, cols // bs), dtype=np.uint8)
    scales.flat[: hi + 1] = np.arange(hi + 1, dtype=np.uint8)          # every scale code appears
    if per_row:
        G = (2.0 ** rng.uniform(-12, 12, rows)).astype(np.float32)
        G[0], G[1] = 1.0, np.float32(2688.0 / 3.0)
    else:
        G = np.float32(2688.0 / 1.7)
    got = oracle_lib.dequantize_fmt(codes, scales, rows, cols, fmt, G)
    want = _expected(vals, scales, rows, cols, vf, sf, bs, G)
    assert got.shape == want.shape
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (fmt, per_row, bad[:5], got.flat[bad[:5]], want.flat[bad[:5]])


def test_dequantize_nvfp4_equals_general_form(oracle_lib):
    """so_dequantize (the NVFP4 entry point) is the general dequantizer's NVFP4 case."""
    rng = np.random.default_rng(9)
    rows, cols = 16, 256
    codes = rng.integers(0, 256, (rows, cols // 2), dtype=np.uint8)
    scales = rng.integers(0, 127, (rows, cols // 16), dtype=np.uint8)
    a = oracle_lib.dequantize(codes, scales, rows, cols, 3.25)
    b = oracle_lib.dequantize_fmt(codes, scales, rows, cols, "nvfp4", np.float32(3.25))
    assert np.array_equal(a, b)
