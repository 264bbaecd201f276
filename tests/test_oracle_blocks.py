"""Oracle pins at block level: hand-worked blocks, exhaustive brute force,
invariants of Algorithm 1, representable blocks, and r = 0 as the textbook
max-abs quantizer built from library casts."""
import json
import os

import ml_dtypes
import numpy as np
import pytest

F4 = ml_dtypes.float4_e2m1fn
F8 = ml_dtypes.float8_e4m3fn
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_blocks.json")
GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
CODES = np.arange(1, 127, dtype=np.uint8)
SCALES = CODES.view(F8).astype(np.float64)                        # library decode


def _blocks(n, seed):
    rng = np.random.default_rng(seed)
    fam = [
        rng.standard_normal((n, 16)),
        rng.standard_t(3, (n, 16)),
        rng.standard_normal((n, 16)) * np.exp(rng.uniform(-12, 6, (n, 1))),
        rng.integers(-12, 13, (n, 16)) / 2.0,                      # many exact ties
    ]
    x = np.concatenate(fam).astype(np.float32)
    # round through bf16 like real inputs (RNE) -- values only, no arithmetic of the method
    import torch
    return torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()


@pytest.mark.parametrize("case", json.load(open(GOLDEN))["blocks"], ids=lambda c: c["id"])
def test_hand_worked_blocks(oracle_lib, case):
    y = np.zeros(16, np.float32)
    y[: len(case["values"])] = case["values"]
    r = oracle_lib.search_block(y, case["fmin"], case["fmax"])
    assert (r.c0, r.cstar, r.fstar) == (case["c0"], case["cstar"], case["fstar"])
    assert r.err_base == case["err_base"] and r.err_best == case["err_best"]
    assert (int(r.nib[0]), int(r.nib[1])) == (case["nib0"], case["nib1"])


def _exact_errors(y):
    """Brute force, independent of the oracle: for every finite positive UE4M3
    scale (library decode), each element's nearest grid value in float64 and
    the exact squared error.  Returns [nblocks][126]."""
    a = np.abs(y.astype(np.float64))[:, None, :, None]            # [n,1,16,1]
    cand = SCALES[None, :, None, None] * GRID[None, None, None, :]  # [1,126,1,8]
    d = np.min((a - cand) ** 2, axis=3)                          # nearest per element
    return d.sum(axis=2)


def test_full_range_equals_brute_force(oracle_lib):
    # f in [-127, 127] finds the closest vector of V_NVFP4.
    y = _blocks(600, 11)
    ex = _exact_errors(y)
    exmin = np.minimum(ex.min(axis=1), (y.astype(np.float64) ** 2).sum(1))
    for i in range(y.shape[0]):
        r = oracle_lib.search_block(y[i], -126, 126)
        tol = 2e-6 * exmin[i] + 1e-30
        assert abs(r.err_best - exmin[i]) <= tol + 1e-6 * abs(r.err_best), i
        if r.cstar > 0:
            assert ex[i, r.cstar - 1] <= exmin[i] * (1 + 4e-6) + 1e-30, i


def test_winner_reconstruction_error(oracle_lib):
    # the reported error is the squared distance of the emitted block, recomputed
    # in float64 from library decodes of the emitted nibbles and scale
    y = _blocks(300, 12)
    for i in range(y.shape[0]):
        r = oracle_lib.search_block(y[i], -8, 8)
        q = r.nib.astype(np.uint8).view(F4).astype(np.float64)
        s = 0.0 if r.cstar == 0 else float(np.array([r.cstar], np.uint8).view(F8)[0])
        e = ((y[i].astype(np.float64) - q * s) ** 2).sum()
        assert abs(e - r.err_best) <= 1e-5 * e + 1e-30, i


def test_invariants(oracle_lib):
    y = _blocks(400, 13)
    for i in range(y.shape[0]):
        prev = None
        for (lo, hi) in [(0, 0), (-1, 1), (-2, 6), (-8, 8), (-126, 126)]:
            r = oracle_lib.search_block(y[i], lo, hi)
            assert r.err_best <= r.err_base                       # dominance
            assert lo <= r.fstar <= hi                            # f* in range
            assert (1 <= r.cstar <= 126) or (r.cstar == 0 and r.c0 == 0)
            if prev is not None:
                assert r.err_best <= prev                         # wider range never worse
            prev = r.err_best
            if (lo, hi) == (0, 0):
                assert r.cstar == r.c0 and r.err_best == r.err_base


def test_representable_blocks_recovered(oracle_lib):
    # blocks in V_NVFP4 with max|q| in {4, 6} are found exactly at r >= 5
    rng = np.random.default_rng(5)
    for c in range(1, 127):
        s = float(np.array([c], np.uint8).view(F8)[0])
        for qmax in (4.0, 6.0):
            q = rng.choice(GRID[GRID <= qmax], 16) * rng.choice([-1, 1], 16)
            q[rng.integers(16)] = qmax * rng.choice([-1, 1])
            y = (q * s).astype(np.float32)
            r = oracle_lib.search_block(y, -8, 8)
            assert r.err_best == 0.0, (c, qmax)
            r5 = oracle_lib.search_block(y, -5, 5)
            assert r5.err_best == 0.0, (c, qmax)
            if qmax == 6.0:
                assert r.cstar == c and r.fstar == 0


def test_radius_zero_is_textbook_maxabs(oracle_lib):
    # P:142-147 / figVLLMnvf4: s = round_UE4M3(max|x| * (1/6)), q = round_E2M1(x * (1/s));
    # written with numpy float32 arithmetic and ml_dtypes casts (RNE, saturated).
    y = _blocks(500, 14)
    m = np.abs(y).max(1)
    v = m * (np.float32(1.0) / np.float32(6.0))
    sc = np.minimum(v, np.float32(448)).astype(F8)
    codes = sc.view(np.uint8)
    s = sc.astype(np.float32)
    with np.errstate(divide="ignore"):
        rho = np.where(s > 0, np.float32(1.0) / s, np.float32(0.0)).astype(np.float32)
    t = (y * rho[:, None]).astype(np.float32)
    nib = t.astype(F4).view(np.uint8)
    xh = nib.view(F4).astype(np.float64) * s[:, None]
    for i in range(y.shape[0]):
        r = oracle_lib.search_block(y[i], 0, 0)
        assert r.cstar == codes[i]
        assert np.array_equal(r.nib, nib[i]), i
        e = ((y[i].astype(np.float64) - xh[i]) ** 2).sum()
        assert abs(r.err_base - e) <= 1e-5 * e + 1e-30


def test_maxabs_scale_for_every_bf16_block_max(oracle_lib):
    # P:144 / Alg. 1 line 2 for every positive finite bf16 value as the block
    # max: c0 = round_UE4M3(m * RN(1/6)) (R8), via numpy float32 and ml_dtypes.
    pats = np.arange(1, 0x7F80, dtype=np.uint32) << 16
    m = pats.view(np.float32)
    v = m * (np.float32(1.0) / np.float32(6.0))
    ref = np.minimum(v, np.float32(448)).astype(F8).view(np.uint8)
    y = np.zeros(16, np.float32)
    for k in range(m.size):
        y[5] = -m[k] if k % 2 else m[k]
        r = oracle_lib.search_block(y, 0, 0)
        assert r.c0 == ref[k], (m[k], r.c0, ref[k])


def test_r7_reciprocal_vs_division(oracle_lib):
    import oracle
    """R7 (DESIGN.md §3): t = RN(y * RN(1/s)) (vLLM, P:132-135) is not always the
    E2M1 value nearest y/s (Alg. 1 writes x_i / s, P:190).  Pins the documented
    example and bounds how often the two readings pick different values."""
    s = np.float32(oracle.e4m3_value(38))
    assert s == np.float32(0.21875)
    y = np.nextafter(np.float32(1.75) * s, np.float32(0))  # 1 ulp below the 1.75 midpoint
    t_rcp = np.float32(y * np.float32(np.float32(1) / s))
    q_rcp = oracle.e2m1_value(int(oracle.e2m1_encode(np.array([t_rcp], np.float32))[0]))
    q_div = oracle.e2m1_value(int(oracle.e2m1_encode(np.array([np.float32(y / s)], np.float32))[0]))
    assert (q_rcp, q_div) == (2.0, 1.5)
    # the nearer value is the division's: |y - 1.5 s| < |y - 2 s|
    assert abs(float(y) - 1.5 * float(s)) < abs(float(y) - 2.0 * float(s))
    # random bf16-representable y over every normal scale: differences are rare
    rng = np.random.default_rng(7)
    yy = (rng.standard_normal(1 << 16) * 3).astype(np.float32)
    yy = (yy.view(np.uint32) & 0xFFFF0000).view(np.float32)
    diff = 0
    for c in range(8, 127, 3):
        sc = np.float32(oracle.e4m3_value(c))
        a = oracle.e2m1_encode((yy * sc * np.float32(np.float32(1) / sc)).astype(np.float32))
        b = oracle.e2m1_encode(((yy * sc).astype(np.float32) / sc).astype(np.float32))
        diff += int((a != b).sum())
    assert diff < 1e-3 * len(yy) * len(range(8, 127, 3))
