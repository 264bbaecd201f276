"""Pins of the oracle's generic ExMy block formats (fig:nvfp-scale,
fig:nvfp-val, fig:mxfp P:237-260; reading R21 in DESIGN.md §3).

What fixes them from outside the oracle:
  - value and scale decodes against ml_dtypes' own format definitions, where
    ml_dtypes has the format (E2M1, E2M3, E3M2; UE4M3, UE5M2, UE3M4, UE8M0);
  - value / scale encodes against ml_dtypes' RNE casts in the finite range;
  - the generic search reduces exactly to the separately pinned NVFP4, NVFP6,
    MXFP4 and MXFP6 oracles at those four formats (every output bit);
  - an independently written exact-rational brute force (Python Fractions,
    binary32 rounding by exact bracketing) over every valid scale of small
    blocks in formats no hardware has.
"""
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest

import oracle

# ---------------------------------------------------------------------------
# decodes / encodes against ml_dtypes
# ---------------------------------------------------------------------------
VALUE_DT = {(2, 1): ml_dtypes.float4_e2m1fn, (2, 3): ml_dtypes.float6_e2m3fn,
            (3, 2): ml_dtypes.float6_e3m2fn}


@pytest.mark.parametrize("fmt", list(VALUE_DT))
def test_gen_value_matches_ml_dtypes(oracle_lib, fmt):
    e, m = fmt
    n = 1 << (e + m + 1)
    ref = np.arange(n, dtype=np.uint8).view(VALUE_DT[fmt]).astype(np.float64)
    got = np.array([oracle.gen_value(e, m, c) for c in range(n)])
    assert np.array_equal(got, ref)
    assert np.array_equal(np.signbit(got), np.signbit(ref))


@pytest.mark.parametrize("fmt", list(VALUE_DT))
def test_gen_encode_matches_ml_dtypes_rne(oracle_lib, fmt):
    e, m = fmt
    vmax = oracle.gen_value(e, m, (1 << (e + m)) - 1)
    rng = np.random.default_rng(11)
    t = np.concatenate([rng.uniform(-vmax, vmax, 4000),
                        rng.standard_normal(2000) * vmax / 8]).astype(np.float32)
    # exact midpoints of the grid (ties to even)
    grid = np.array([oracle.gen_value(e, m, c) for c in range(1 << (e + m))])
    mids = ((grid[1:] + grid[:-1]) / 2).astype(np.float32)
    t = np.concatenate([t, mids, -mids])
    ref = t.astype(VALUE_DT[fmt]).view(np.uint8)
    got = np.array([oracle.gen_encode(e, m, float(v)) for v in t], np.uint8)
    assert np.array_equal(got, ref)
    # saturation beyond vmax (satfinite, R10)
    for v in (vmax * 1.01, vmax * 7, 1e30, float("inf")):
        assert oracle.gen_encode(e, m, v) == (1 << (e + m)) - 1
        assert oracle.gen_encode(e, m, -v) == (1 << (e + m + 1)) - 1


def test_gen_value_formats_without_library(oracle_lib):
    """E1M2, E3M0, E3M1, E4M2: closed-form spot values, grid size, monotonicity."""
    assert [oracle.gen_value(1, 2, c) for c in range(8)] == [0, .5, 1, 1.5, 2, 2.5, 3, 3.5]
    assert [oracle.gen_value(3, 0, c) for c in range(8)] == [0, .25, .5, 1, 2, 4, 8, 16]
    assert oracle.gen_value(3, 1, 15) == 24.0 and oracle.gen_value(3, 1, 1) == 0.125
    assert oracle.gen_value(4, 2, 63) == 1.75 * 2 ** 8 and oracle.gen_value(4, 2, 1) == 2.0 ** -8
    for e, m in ((1, 2), (3, 0), (3, 1), (4, 2), (1, 4)):
        v = [oracle.gen_value(e, m, c) for c in range(1 << (e + m))]
        assert all(a < b for a, b in zip(v, v[1:]))


SCALE_DT = {(4, 3): (ml_dtypes.float8_e4m3fn, 126), (5, 2): (ml_dtypes.float8_e5m2, 123),
            (3, 4): (ml_dtypes.float8_e3m4, 111), (8, 0): (ml_dtypes.float8_e8m0fnu, 254)}


@pytest.mark.parametrize("fmt", list(SCALE_DT))
def test_gen_scale_value_matches_ml_dtypes(oracle_lib, fmt):
    """UExMy decodes: the library format's positive half (codes below its
    special values; R21 reserves only the all-ones code)."""
    e, m = fmt
    dt, top = SCALE_DT[fmt]
    ref = np.arange(top + 1, dtype=np.uint8).view(dt).astype(np.float64)
    got = np.array([oracle.gen_scale_value(e, m, c) for c in range(top + 1)])
    assert np.array_equal(got, ref)
    assert np.isnan(oracle.gen_scale_value(e, m, (1 << (e + m)) - 1))


@pytest.mark.parametrize("fmt", [(4, 3), (5, 2), (3, 4)])
def test_gen_scale_encode_matches_ml_dtypes_rne(oracle_lib, fmt):
    e, m = fmt
    dt, top = SCALE_DT[fmt]
    smax = oracle.gen_scale_value(e, m, top)
    rng = np.random.default_rng(5)
    v = np.exp(rng.uniform(np.log(oracle.gen_scale_value(e, m, 1)) - 1, np.log(smax), 4000)).astype(np.float32)
    ref = v.astype(dt).view(np.uint8)
    got = np.array([oracle.gen_scale_encode(e, m, float(a)) for a in v], np.uint8)
    assert np.array_equal(got, ref)


def test_gen_scale_encode_pow2_rounds_up(oracle_lib):
    """m = 0 (R19): the smallest power of two >= v, saturating; = the pinned UE8M0 rule."""
    rng = np.random.default_rng(9)
    v = np.exp(rng.uniform(-95, 95, 3000)).astype(np.float32)
    for a in v:
        assert oracle.gen_scale_encode(8, 0, float(a)) == oracle.ue8m0_encode(float(a))
    for e in (3, 5, 6):
        bias = (1 << (e - 1)) - 1
        for a in (0.3, 1.0, 1.0001, 3.0, 2.0 ** 40):
            c = oracle.gen_scale_encode(e, 0, a)
            maxc = (1 << e) - 2
            want = min(max(int(np.ceil(np.log2(a))) + bias, 0), maxc)
            assert c == want


# ---------------------------------------------------------------------------
# the generic search reduces to the separately pinned format oracles
# ---------------------------------------------------------------------------
def _bf16(rows, cols, seed, kind="student"):
    import torch
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(rows, cols, generator=g)
    if kind == "student":
        x = x / torch.sqrt(torch.distributions.Chi2(3.0).sample((rows, cols)) / 3.0)
    x[0, :16] = 0.0  # an all-zero block (c0 = 0, the zero-scale candidate)
    return x.to(torch.bfloat16)


def _nib_unpack(packed, rows, cols):
    p = np.asarray(packed).reshape(rows, cols // 2)
    out = np.empty((rows, cols), np.uint8)
    out[:, 0::2] = p & 15
    out[:, 1::2] = p >> 4
    return out


@pytest.mark.parametrize("window", [(-8, 8), (-2, 6), (0, 0), (-126, 126)])
def test_gen_equals_nvfp4_oracle(oracle_lib, window):
    x = _bf16(32, 256, 1)
    a = oracle.quantize_gen(x, 32, 256, *window, (2, 1, 4, 3, 16), "tensor")
    b = oracle.quantize(x, 32, 256, *window, "tensor")
    assert np.array_equal(a.codes, _nib_unpack(b.codes, 32, 256))
    assert np.array_equal(a.scales, b.scales)
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.err.view(np.uint32), b.err.view(np.uint32))
    assert np.array_equal(a.sums, b.sums) and a.G == b.G and a.n_eval == b.n_eval


@pytest.mark.parametrize("name,fmt,gmode", [("nvfp6_e2m3", (2, 3, 4, 3, 16), "tensor"),
                                             ("mxfp4", (2, 1, 8, 0, 32), "none"),
                                             ("mxfp6_e2m3", (2, 3, 8, 0, 32), "none")])
def test_gen_equals_format_oracles(oracle_lib, name, fmt, gmode):
    x = _bf16(16, 512, 2)
    for window in ((-3, 3), (-1, 1), (0, 2)):
        a = oracle.quantize_gen(x, 16, 512, *window, fmt, gmode)
        b = oracle.quantize_fmt(x, 16, 512, *window, name, gmode)
        codes_b = _nib_unpack(b.codes, 16, 512) if fmt[1] == 1 else b.codes
        assert np.array_equal(a.codes, codes_b)
        assert np.array_equal(a.scales, b.scales)
        assert np.array_equal(a.err.view(np.uint32), b.err.view(np.uint32))
        assert np.array_equal(a.sums, b.sums)


def test_gen_dequantize_equals_format_dequantizers(oracle_lib):
    x = _bf16(8, 256, 3)
    a = oracle.quantize_gen(x, 8, 256, -4, 4, (2, 1, 4, 3, 16), "tensor")
    b = oracle.quantize(x, 8, 256, -4, 4, "tensor")
    da = oracle.dequantize_gen(a.codes, a.scales, 8, 256, (2, 1, 4, 3, 16), a.G)
    db = oracle.dequantize(b.codes, b.scales, 8, 256, b.G)
    assert np.array_equal(da, db)


# ---------------------------------------------------------------------------
# exact-rational brute force (independent of the C oracle)
# ---------------------------------------------------------------------------
def _rn32(q: Fraction) -> np.float32:
    """Round a rational to the nearest binary32, ties to even (exact bracketing)."""
    f = np.float32(float(q))
    best = None
    for c in (np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))):
        d = abs(Fraction(float(c)) - q)
        if best is None or d < best[0] or (d == best[0] and (c.view(np.uint32) & 1) == 0):
            best = (d, c)
    return np.float32(best[1])


def _grid(e, m, pow2=False):
    bias = (1 << (e - 1)) - 1
    out = []
    for c in range(1 << (e + m)):
        if pow2:
            out.append(Fraction(2) ** (c - bias))
            continue
        E, M = c >> m, c & ((1 << m) - 1)
        out.append(Fraction(M, 1 << m) * Fraction(2) ** (1 - bias) if E == 0
                   else Fraction((1 << m) + M, 1 << m) * Fraction(2) ** (E - bias))
    return out


def _nearest(grid, a: Fraction):
    """index of the grid value nearest a >= 0, ties to the even index, saturating"""
    if a >= grid[-1]:
        return len(grid) - 1
    best = 0
    for k in range(1, len(grid)):
        d, db = abs(a - grid[k]), abs(a - grid[best])
        if d < db or (d == db and k % 2 == 0):
            best = k
    return best


def _brute_block(y32, fmt):
    """Alg. 1 over every valid scale of the format (lexicographic (loss, code) min)."""
    ve, vm, se, sm, bs = fmt
    vals = _grid(ve, vm)
    pow2 = sm == 0
    sg = _grid(se, sm, pow2)[:-1]  # the all-ones code is NaN
    vmax = vals[-1]
    kinv = _rn32(1 / vmax)
    m = max(abs(Fraction(float(v))) for v in y32)
    v = _rn32(m * Fraction(float(kinv)))
    if pow2:
        c0 = next((c for c, s in enumerate(sg) if s >= Fraction(float(v))), len(sg) - 1)
    else:
        c0 = _nearest(sg, Fraction(float(v)))
    cands = [c for c in range(len(sg)) if (c >= 1 or pow2)]
    if not pow2 and c0 == 0:
        cands = [0] + cands
    best = None
    base = None
    for c in sorted(cands):
        s = sg[c]
        rho = Fraction(0) if s == 0 else Fraction(float(_rn32(1 / s)))
        parts = []
        for h in range(bs // 16):
            d = []
            for i in range(16):
                yv = Fraction(float(y32[16 * h + i]))
                t = _rn32(yv * rho)
                q = vals[_nearest(vals, abs(Fraction(float(t))))]
                q = -q if np.signbit(t) else q
                d.append(_rn32(yv - q * s))
            a = _rn32(Fraction(float(d[0])) ** 2)
            for i in range(2, 16, 2):
                a = _rn32(Fraction(float(d[i])) ** 2 + Fraction(float(a)))
            b = _rn32(Fraction(float(d[1])) ** 2)
            for i in range(3, 16, 2):
                b = _rn32(Fraction(float(d[i])) ** 2 + Fraction(float(b)))
            parts.append(_rn32(Fraction(float(a)) + Fraction(float(b))))
        w = 1
        while w < len(parts):
            for h in range(0, len(parts), 2 * w):
                parts[h] = _rn32(Fraction(float(parts[h])) + Fraction(float(parts[h + w])))
            w *= 2
        loss = parts[0]
        if c == c0:
            base = loss
        if best is None or loss < best[0]:
            best = (loss, c)
    return c0, best[1], best[0], base


@pytest.mark.parametrize("fmt", [(3, 0, 3, 2, 16), (1, 2, 5, 1, 16), (2, 1, 6, 0, 32), (2, 2, 3, 3, 16)])
def test_gen_search_matches_exact_brute_force(oracle_lib, fmt):
    ve, vm, se, sm, bs = fmt
    rng = np.random.default_rng(100 + ve * 10 + se)
    maxc = (1 << (se + sm)) - 2
    smax = oracle.gen_scale_value(se, sm, maxc)
    vmax = oracle.gen_value(ve, vm, (1 << (ve + vm)) - 1)
    n_blocks = 40
    for k in range(n_blocks):
        scale = float(np.exp(rng.uniform(np.log(1e-3), np.log(smax * vmax / 4))))
        y = (rng.standard_normal(bs) * scale).astype(np.float32)
        if k % 10 == 0:
            y[:] = 0.0
        if k % 10 == 1:  # grid points and midpoints of one scale
            s = oracle.gen_scale_value(se, sm, int(rng.integers(1, maxc)))
            y = (rng.integers(-8, 9, bs) * 0.25 * s).astype(np.float32)
        r = oracle.search_block_gen(y, fmt, -maxc, maxc)
        c0, cstar, best, base = _brute_block(y, fmt)
        assert (r.c0, r.cstar) == (c0, cstar), (k, y)
        assert np.float32(r.err_best).view(np.uint32) == np.float32(best).view(np.uint32)
        assert np.float32(r.err_base).view(np.uint32) == np.float32(base).view(np.uint32)


def test_gen_invariants(oracle_lib):
    """ScaleSearch never loses to the max-abs scale; a wider window never loses."""
    x = _bf16(16, 256, 4, kind="gauss")
    for fmt in ((3, 2, 4, 3, 16), (1, 2, 5, 2, 16), (2, 1, 5, 0, 16), (4, 3, 4, 3, 16)):
        prev = None
        for r in (0, 1, 2, 4, 8):
            q = oracle.quantize_gen(x, 16, 256, -r, r, fmt, "tensor")
            assert np.all(q.err[:, 0] <= q.err[:, 1])
            if prev is not None:
                assert np.all(q.err[:, 0] <= prev)
            prev = q.err[:, 0].copy()
        q0 = oracle.quantize_gen(x, 16, 256, 0, 0, fmt, "tensor")
        assert np.all(q0.offsets == 0) and np.array_equal(q0.err[:, 0], q0.err[:, 1])
