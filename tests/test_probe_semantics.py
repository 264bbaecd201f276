"""Hardware conversion semantics on the B200 versus the CPU oracle.

Runs tools/probes/probe (built here with nvcc) which records every point where
the hardware rounding functions cvt.rn.satfinite.e2m1x2.f32 and
cvt.rn.satfinite.e4m3x2.f32 change value over all 2^32 binary32 patterns, the
unpack cvt.rn.f16x2.e2m1x2 of all 256 bytes, and fma.rn.f32.f16 on 2^20
(q, -s, y) triples.  The oracle encoders (enumeration, R10/R11) must
agree at both ends of every constant run, which fixes the hardware function
exactly because both are monotone step functions of the pattern.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE_DIR = os.path.join(ROOT, "tools", "probes")


def _build_probe():
    exe = os.path.join(PROBE_DIR, "probe")
    src = os.path.join(PROBE_DIR, "probe.cu")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-lineinfo", "-o", exe, src], check=True)
    return exe


@pytest.fixture(scope="module")
def probe_out(tmp_path_factory):
    import json
    exe = _build_probe()
    out = tmp_path_factory.mktemp("probe")
    res = subprocess.run([exe, str(out)], check=True, capture_output=True, text=True, timeout=600)
    info = json.loads(res.stdout)
    dst = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(dst):
        with open(os.path.join(dst, "probe.json"), "w") as f:
            f.write(res.stdout)
    return out, info


def _runs(path):
    t = np.fromfile(path, np.uint32).reshape(-1, 2)
    return t[np.argsort(t[:, 0])]


def _check_runs(trans, lo, hi, oracle_fn, mask):
    """trans: sorted (pattern, code); run k covers [p_k, p_{k+1})."""
    p = trans[:, 0].astype(np.int64)
    ends = np.append(p[1:], hi)
    keep = p < hi
    starts, stops, codes = p[keep], np.minimum(ends[keep], hi), trans[keep, 1] & mask
    assert starts[0] == lo
    pts = np.concatenate([starts, stops - 1]).astype(np.uint32)
    want = np.concatenate([codes, codes]).astype(np.uint8)
    got = oracle_fn(pts.view(np.float32)) & mask
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(hex(int(pts[b])), int(got[b]), int(want[b])) for b in bad[:10]]


@pytest.mark.gpu
def test_e2m1_pack_matches_oracle(oracle_lib, probe_out):
    out, _ = probe_out
    _check_runs(_runs(out / "e2m1_pos_transitions.u32"), 0, 0x7F800001, oracle_lib.e2m1_encode, 0xF)
    _check_runs(_runs(out / "e2m1_neg_transitions.u32"), 0x80000000, 0xFF800001, oracle_lib.e2m1_encode, 0xF)


@pytest.mark.gpu
def test_e4m3_pack_matches_oracle(oracle_lib, probe_out):
    out, _ = probe_out
    _check_runs(_runs(out / "e4m3_pos_transitions.u32"), 0, 0x7F800000, oracle_lib.e4m3_encode, 0xFF)


@pytest.mark.gpu
def test_pair_order(probe_out):
    _, info = probe_out
    assert info["pair_order_e2m1"] == 0x72       # first operand -> high nibble
    assert info["pair_order_e4m3"] == 0x7E38


@pytest.mark.gpu
def test_e2m1_unpack(oracle_lib, probe_out):
    out, _ = probe_out
    h = np.fromfile(out / "e2m1_unpack.u32", np.uint32)
    lo = (h & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
    hi = (h >> 16).astype(np.uint16).view(np.float16).astype(np.float64)
    for b in range(256):
        assert lo[b] == oracle_lib.e2m1_value(b & 15) and hi[b] == oracle_lib.e2m1_value(b >> 4), b
        assert np.signbit(lo[b]) == bool(b & 8) and np.signbit(hi[b]) == bool(b & 0x80)


@pytest.mark.gpu
def test_fhfma_is_single_rounding(probe_out):
    out, _ = probe_out
    a = np.fromfile(out / "fhfma_a.u16", np.uint16).view(np.float16).astype(np.float64)
    b = np.fromfile(out / "fhfma_b.u16", np.uint16).view(np.float16).astype(np.float64)
    c = np.fromfile(out / "fhfma_c.f32", np.float32).astype(np.float64)
    d = np.fromfile(out / "fhfma_d.f32", np.float32)
    ref = (a * b + c).astype(np.float32)      # exact in float64 for these ranges, one rounding
    assert np.array_equal(ref.view(np.uint32), d.view(np.uint32))
