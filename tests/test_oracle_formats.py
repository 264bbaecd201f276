"""Pins for the oracle's number formats against the paper and independent libraries.

E2M1 value set: PAPER.md P:104 (§3).  E4M3 scale: OCP E4M3 (reading R1 in
DESIGN.md §3; the ratio of the worked example P:296).  Independent
implementations: ml_dtypes float4_e2m1fn / float8_e4m3fn and torch's
float8_e4m3fn cast.
"""
import ml_dtypes
import numpy as np
import pytest
import torch

F4 = ml_dtypes.float4_e2m1fn
F8 = ml_dtypes.float8_e4m3fn


def test_e2m1_value_set_matches_paper(oracle_lib):
    # R_E2M1 = {0, ±0.5, ±1, ±1.5, ±2, ±3, ±4, ±6}
    vals = sorted({oracle_lib.e2m1_value(n) for n in range(16)})
    assert vals == [-6, -4, -3, -2, -1.5, -1, -0.5, 0, 0.5, 1, 1.5, 2, 3, 4, 6]
    for n in range(16):
        lib = float(np.array([n], np.uint8).view(F4)[0])
        assert oracle_lib.e2m1_value(n) == lib


def _structured_floats():
    """All float32 sign/exponent/top-mantissa patterns x a few low-bit endings,
    plus every exact E2M1 midpoint and its neighbours, plus random values."""
    hi = np.arange(1 << 19, dtype=np.uint32) << 13          # sign+exp+10 mantissa bits
    lows = np.array([0, 1, 0xFFF, 0x1000, 0x1001, 0x1FFF], np.uint32)
    pats = (hi[:, None] | lows[None, :]).ravel()
    f = pats.view(np.float32)
    f = f[np.isfinite(f)]
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0, 7.0], np.float32)
    near = np.concatenate([mids, np.nextafter(mids, 0), np.nextafter(mids, 10)])
    rnd = np.random.default_rng(1).standard_normal(1 << 20).astype(np.float32) * 3
    allv = np.concatenate([f, near, -near, rnd, np.array([0.0, -0.0], np.float32)])
    return allv


def test_e2m1_encode_matches_ml_dtypes(oracle_lib):
    t = _structured_floats()
    got = oracle_lib.e2m1_encode(t)
    ref = t.astype(F4).view(np.uint8)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (t[bad[:8]], got[bad[:8]], ref[bad[:8]])


def test_e2m1_ties_to_even_and_saturation(oracle_lib):
    # P:148 nearest rounding; ties to the even code (R10); SPEC example E2M1(2.5) = 2
    t = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.5, 1e30, -0.1, -0.0], np.float32)
    mags = [oracle_lib.e2m1_value(n) for n in oracle_lib.e2m1_encode(t)]
    assert mags == [0.0, 1.0, 1.0, 2.0, 2.0, 4.0, 4.0, 6.0, 6.0, -0.0, -0.0]
    # -0 nibble (R11): negative values that round to zero keep the sign bit
    assert list(oracle_lib.e2m1_encode(np.array([-0.1, -0.0], np.float32))) == [8, 8]


def test_e4m3_decode_all_codes(oracle_lib):
    for c in range(127):
        lib = float(np.array([c], np.uint8).view(F8)[0])
        assert oracle_lib.e4m3_value(c) == lib, c
    assert np.isnan(oracle_lib.e4m3_value(127))


def test_e4m3_worked_example_ratio(oracle_lib):
    # "+4 codes from a zero-mantissa code is x1.5".  The paper's absolute
    # codes (64 = 1.0, 68 = 1.5) are off by one binade for OCP E4M3 (R1).
    assert oracle_lib.e4m3_value(0x38) == 1.0
    assert oracle_lib.e4m3_value(0x3C) == 1.5
    assert oracle_lib.e4m3_value(0x3C) / oracle_lib.e4m3_value(0x38) == 1.5
    assert oracle_lib.e4m3_value(64) == 2.0 and oracle_lib.e4m3_value(68) == 3.0
    assert oracle_lib.e4m3_value(0x7E) == 448.0
    assert oracle_lib.e4m3_value(1) == 2.0 ** -9
    assert oracle_lib.e4m3_value(8) == 2.0 ** -6
    # scales strictly increase with the code
    v = [oracle_lib.e4m3_value(c) for c in range(127)]
    assert all(a < b for a, b in zip(v, v[1:]))


def test_e4m3_encode_matches_libraries(oracle_lib):
    t = np.abs(_structured_floats())
    t = t[t < 1e6]
    got = oracle_lib.e4m3_encode(t)
    clamped = np.minimum(t, np.float32(448.0))   # satfinite (ml_dtypes overflows to NaN past 464)
    ref = clamped.astype(F8).view(np.uint8)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (t[bad[:8]], got[bad[:8]], ref[bad[:8]])
    ref_t = torch.from_numpy(clamped).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(got, ref_t)
    # underflow tie at 2^-10 goes to the even code 0; satfinite above 448
    e = oracle_lib.e4m3_encode(np.array([2.0 ** -10, np.nextafter(np.float32(2.0 ** -10), np.float32(1)), 449, 1e30], np.float32))
    assert list(e) == [0, 1, 126, 126]
