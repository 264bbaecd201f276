"""Bitwise brute-force pin of the oracle's Algorithm 1 (SPEC S:570 / SURVEY §8(c)
"Brute force": >= 10^4 seeded blocks).

tests/brute/brute_nvfp4.c is an exhaustive search written independently of
oracle/ss_oracle.c (different scale decode, c0 rounding, E2M1 rounding and
selection technique; see its header).  Over 16 384 seeded blocks from eight
families -- Gaussian, Student-t, wide dynamic range, full 24-bit mantissas,
exact E2M1 midpoints at many scales (ties), blocks representable in NVFP4,
underflow to the zero scale, saturation at 448 -- and four windows
(max-abs, the paper's [-2, 6], +-8 and the full range of P:218), the oracle's
c0, c*, f*, both losses (bit patterns) and all 16 nibbles must equal the
brute force's.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "brute", "brute_nvfp4.c")
N_PER_FAMILY = 2048
WINDOWS = [(0, 0), (-2, 6), (-8, 8), (-126, 126)]


@pytest.fixture(scope="module")
def brute(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("brute") / "brute_nvfp4.so")
    subprocess.run(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                    "-o", so, SRC, "-lm"], check=True)
    L = ctypes.CDLL(so)
    P = ctypes.c_void_p
    L.brute_search.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, P, P, P, P]
    return L


def _blocks(seed=2026):
    rng = np.random.default_rng(seed)
    n = N_PER_FAMILY
    grid = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
    s_all = np.array([ldexp_code(c) for c in range(1, 127)], np.float64)
    fam = [
        rng.standard_normal((n, 16)),
        rng.standard_t(3, (n, 16)),
        rng.standard_normal((n, 16)) * np.exp(rng.uniform(-25, 12, (n, 1))),
        (rng.standard_normal((n, 16)) * (1 + rng.uniform(-2 ** -20, 2 ** -20, (n, 16)))),
        # exact E2M1 midpoints / grid points times a scale value: ties everywhere
        rng.choice(np.concatenate([grid, mids]), (n, 16)) * rng.choice([-1, 1], (n, 16))
        * s_all[rng.integers(0, 126, (n, 1))],
        # representable blocks with max |q| in {4, 6}
        np.concatenate([rng.choice(grid, (n, 15)), rng.choice([4.0, 6.0], (n, 1))], 1)
        * rng.choice([-1, 1], (n, 16)) * s_all[rng.integers(0, 126, (n, 1))],
        # underflow: max-abs scale code 0 (zero-scale candidate) and the smallest codes
        rng.standard_normal((n, 16)) * 2.0 ** rng.uniform(-16, -8, (n, 1)),
        # saturation: block maxima above 6 * 448
        rng.standard_normal((n, 16)) * 2.0 ** rng.uniform(9, 13, (n, 1)),
    ]
    return np.concatenate(fam).astype(np.float32)


def ldexp_code(c):
    """UE4M3 code -> value for the test's inputs (a third spelling: frexp-free
    arithmetic on the code's fields in float64)."""
    e, m = c >> 3, c & 7
    return m / 512.0 if e == 0 else (8 + m) * 2.0 ** (e - 10)


@pytest.mark.parametrize("window", WINDOWS, ids=lambda w: "%d:%d" % w)
def test_oracle_equals_independent_brute_force(oracle_lib, brute, window):
    y = np.ascontiguousarray(_blocks())
    n = y.shape[0]
    assert n >= 10_000
    c0 = np.empty(n, np.int32)
    cs = np.empty(n, np.int32)
    best = np.empty(n, np.float32)
    base = np.empty(n, np.float32)
    nib = np.empty((n, 16), np.uint8)
    brute.brute_search(y.ctypes.data, n, window[0], window[1], c0.ctypes.data, cs.ctypes.data,
                       best.ctypes.data, base.ctypes.data, nib.ctypes.data)
    bad = []
    for i in range(n):
        r = oracle_lib.search_block(y[i], *window)
        ok = (r.c0 == c0[i] and r.cstar == cs[i] and r.fstar == cs[i] - c0[i]
              and np.float32(r.err_best).view(np.uint32) == best[i].view(np.uint32)
              and np.float32(r.err_base).view(np.uint32) == base[i].view(np.uint32)
              and np.array_equal(r.nib, nib[i]))
        if not ok:
            bad.append(i)
    assert not bad, "%d of %d blocks differ, first %d: y=%s" % (len(bad), n, bad[0], y[bad[0]].tolist())
    # the families exercise what they are meant to
    assert (c0 == 0).any() and (c0 == 126).any()
    if window == (-126, 126):
        assert len(np.unique(cs - c0)) > 10
