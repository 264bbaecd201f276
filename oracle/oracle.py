"""ctypes marshalling for the C oracle (test infrastructure only; see __init__)."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ss_oracle.c")
_HDR = os.path.join(_HERE, "ss_oracle.h")
_SO = os.path.join(_HERE, "libss_oracle.so")
_LOCK = threading.Lock()
_LIB = None


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile ss_oracle.c with gcc (plain IEEE binary32, no contraction)."""
    fresh = (
        os.path.exists(_SO)
        and os.path.getmtime(_SO) >= os.path.getmtime(_SRC)
        and os.path.getmtime(_SO) >= os.path.getmtime(_HDR)
    )
    if fresh and not force:
        return _SO
    tmp = _SO + ".tmp%d" % os.getpid()
    cmd = [
        "gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
        "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm",
    ]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _SO)
    return _SO


class _BlockResult(ctypes.Structure):
    _fields_ = [
        ("c0", ctypes.c_int32),
        ("cstar", ctypes.c_int32),
        ("fstar", ctypes.c_int32),
        ("n_evaluated", ctypes.c_int32),
        ("err_best", ctypes.c_float),
        ("err_base", ctypes.c_float),
        ("nib", ctypes.c_uint8 * 16),
    ]


def lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            path = build()
            L = ctypes.CDLL(path)
            P = ctypes.c_void_p
            i64 = ctypes.c_int64
            L.so_e2m1_value.restype = ctypes.c_double
            L.so_e2m1_value.argtypes = [ctypes.c_int]
            L.so_e2m1_encode.restype = ctypes.c_int
            L.so_e2m1_encode.argtypes = [ctypes.c_float]
            L.so_e4m3_value.restype = ctypes.c_float
            L.so_e4m3_value.argtypes = [ctypes.c_int]
            L.so_e4m3_encode.restype = ctypes.c_int
            L.so_e4m3_encode.argtypes = [ctypes.c_float]
            L.so_e2m1_encode_array.argtypes = [P, i64, P]
            L.so_e4m3_encode_array.argtypes = [P, i64, P]
            L.so_search_block.restype = ctypes.c_int
            L.so_search_block.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_BlockResult)]
            L.so_tensor_amax.restype = ctypes.c_int
            L.so_tensor_amax.argtypes = [P, i64, P]
            L.so_global_scale.restype = ctypes.c_int
            L.so_global_scale.argtypes = [ctypes.c_int, ctypes.c_uint32, P]
            L.so_quantize.restype = ctypes.c_int
            L.so_quantize.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                                      P, P, P, P, P, P, P, ctypes.c_int]
            L.so_e2m3_value.restype = ctypes.c_double
            L.so_e2m3_value.argtypes = [ctypes.c_int]
            L.so_e2m3_encode.restype = ctypes.c_int
            L.so_e2m3_encode.argtypes = [ctypes.c_float]
            L.so_ue8m0_value.restype = ctypes.c_float
            L.so_ue8m0_value.argtypes = [ctypes.c_int]
            L.so_ue8m0_encode.restype = ctypes.c_int
            L.so_ue8m0_encode.argtypes = [ctypes.c_float]
            L.so_quantize_fmt.restype = ctypes.c_int
            L.so_quantize_fmt.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P, P,
                                          P, P, ctypes.c_int]
            L.so_dequantize_fmt.restype = ctypes.c_int
            L.so_dequantize_fmt.argtypes = [P, P, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            P, ctypes.c_int, P]
            L.so_dequantize.restype = ctypes.c_int
            L.so_dequantize.argtypes = [P, P, i64, i64, ctypes.c_float, P]
            ci = ctypes.c_int
            L.so_gen_value.restype = ctypes.c_double
            L.so_gen_value.argtypes = [ci, ci, ci]
            L.so_gen_encode.restype = ci
            L.so_gen_encode.argtypes = [ci, ci, ctypes.c_float]
            L.so_gen_scale_value.restype = ctypes.c_double
            L.so_gen_scale_value.argtypes = [ci, ci, ci]
            L.so_gen_scale_encode.restype = ci
            L.so_gen_scale_encode.argtypes = [ci, ci, ctypes.c_float]
            L.so_gen_numer.restype = ctypes.c_float
            L.so_gen_numer.argtypes = [ci, ci, ci, ci]
            L.so_search_block_gen.restype = ci
            L.so_search_block_gen.argtypes = [ci, ci, ci, ci, ci, P, ci, ci, ctypes.POINTER(_BlockResultFmt)]
            L.so_quantize_gen.restype = ci
            L.so_quantize_gen.argtypes = [P, i64, i64, ci, ci, ci, P, ci, ci, ci, ci, ci, P, P, P, P, P,
                                          P, P, ci]
            L.so_dequantize_gen.restype = ci
            L.so_dequantize_gen.argtypes = [P, P, i64, i64, ci, ci, ci, ci, ci, ctypes.c_float, P]
            _LIB = L
    return _LIB


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(st):
    if st != 0:
        raise OracleError({1: "invalid argument", 4: "non-finite input",
                           5: "global scale out of range"}.get(st, "status %d" % st))


def e2m1_value(nibble: int) -> float:
    return lib().so_e2m1_value(int(nibble))


def e4m3_value(code: int) -> float:
    return lib().so_e4m3_value(int(code))


def e2m1_encode(t) -> np.ndarray:
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float32).ravel())
    out = np.empty(t.size, np.uint8)
    lib().so_e2m1_encode_array(_ptr(t), t.size, _ptr(out))
    return out


def e4m3_encode(v) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float32).ravel())
    out = np.empty(v.size, np.uint8)
    lib().so_e4m3_encode_array(_ptr(v), v.size, _ptr(out))
    return out


@dataclass
class BlockResult:
    c0: int
    cstar: int
    fstar: int
    n_evaluated: int
    err_best: float
    err_base: float
    nib: np.ndarray


def search_block(y, fmin: int, fmax: int) -> BlockResult:
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float32))
    assert y.shape == (16,)
    r = _BlockResult()
    _check(lib().so_search_block(_ptr(y), int(fmin), int(fmax), ctypes.byref(r)))
    return BlockResult(r.c0, r.cstar, r.fstar, r.n_evaluated, r.err_best, r.err_base,
                       np.frombuffer(bytes(r.nib), np.uint8).copy())


def _as_u16(x) -> np.ndarray:
    """Accept a numpy uint16 array of bf16 bit patterns or a torch bf16 tensor."""
    if hasattr(x, "view") and hasattr(x, "dtype") and "bfloat16" in str(x.dtype):
        import torch  # plumbing only
        return x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    a = np.asarray(x)
    if a.dtype != np.uint16:
        raise TypeError("expected bf16 bit patterns as uint16")
    return np.ascontiguousarray(a)


def tensor_amax(x) -> int:
    x = _as_u16(x)
    out = np.zeros(1, np.uint32)
    _check(lib().so_tensor_amax(_ptr(x), x.size, _ptr(out)))
    return int(out[0])


def global_scale(gmode: int, amax_bits: int) -> float:
    out = np.zeros(1, np.float32)
    _check(lib().so_global_scale(int(gmode), ctypes.c_uint32(amax_bits), _ptr(out)))
    return float(out[0])


@dataclass
class QuantResult:
    codes: np.ndarray    # [rows][cols/2] u8
    scales: np.ndarray   # [rows][cols/16] u8
    offsets: np.ndarray  # [rows*cols/16] i8
    err: np.ndarray      # [rows*cols/16][2] f32
    sums: np.ndarray     # [2] f64
    n_eval: int
    G: float             # [rows] np.float32 array in mode "row"


GMODES = {"none": 0, "tensor": 1, "given": 2, "row": 3}


def quantize(x, rows: int, cols: int, fmin: int, fmax: int, gmode="tensor",
             amax_bits: int | None = None, threads: int = 0) -> QuantResult:
    x = _as_u16(x).reshape(-1)
    assert x.size == rows * cols
    gm = GMODES[gmode] if isinstance(gmode, str) else int(gmode)
    nb = rows * cols // 16
    codes = np.empty((rows, cols // 2), np.uint8)
    scales = np.empty((rows, cols // 16), np.uint8)
    offs = np.empty(nb, np.int8)
    err = np.empty((nb, 2), np.float32)
    sums = np.zeros(2, np.float64)
    neval = np.zeros(1, np.int64)
    G = np.zeros(rows if gm == 3 else 1, np.float32)
    ab = None if amax_bits is None else np.array([amax_bits], np.uint32)
    _check(lib().so_quantize(_ptr(x), rows, cols, int(fmin), int(fmax), gm, _ptr(ab),
                             _ptr(codes), _ptr(scales), _ptr(offs), _ptr(err), _ptr(sums),
                             _ptr(neval), _ptr(G), int(threads)))
    return QuantResult(codes, scales, offs, err, sums, int(neval[0]),
                       G.copy() if gm == 3 else float(G[0]))


def dequantize(codes, scales, rows: int, cols: int, G=1.0) -> np.ndarray:
    """bf16 bit patterns of xhat; G is a scalar or a per-row array (mode "row")."""
    codes = np.ascontiguousarray(codes, np.uint8).reshape(rows, cols // 2)
    scales = np.ascontiguousarray(scales, np.uint8).reshape(rows, cols // 16)
    out = np.empty((rows, cols), np.uint16)
    if np.ndim(G) == 0:
        _check(lib().so_dequantize(_ptr(codes), _ptr(scales), rows, cols, ctypes.c_float(G), _ptr(out)))
        return out
    for r in range(rows):
        c, sc, o = codes[r].copy(), scales[r].copy(), np.empty(cols, np.uint16)
        _check(lib().so_dequantize(_ptr(c), _ptr(sc), 1, cols, ctypes.c_float(float(G[r])), _ptr(o)))
        out[r] = o
    return out


# ---------------------------------------------------------------------------
# Other block formats: name -> (value format, scale format, block)
# ---------------------------------------------------------------------------
FORMATS = {
    "nvfp4": (0, 0, 16),        # E2M1 values, UE4M3 scales, 16-blocks
    "mxfp4": (0, 1, 32),        # E2M1 values, UE8M0 scales, 32-blocks
    "mxfp6_e2m3": (1, 1, 32),   # E2M3 values, UE8M0 scales, 32-blocks
    "nvfp6_e2m3": (1, 0, 16),   # E2M3 values, UE4M3 scales, 16-blocks (value sweep)
    # block-size study (fig:block_size): NVFP4 values and scales
    "nvfp4_b32": (0, 0, 32), "nvfp4_b64": (0, 0, 64), "nvfp4_b128": (0, 0, 128),
    "nvfp4_b256": (0, 0, 256),
}


def e2m3_value(code: int) -> float:
    return lib().so_e2m3_value(int(code))


def e2m3_encode(t: float) -> int:
    return lib().so_e2m3_encode(float(t))


def ue8m0_value(code: int) -> float:
    return lib().so_ue8m0_value(int(code))


def ue8m0_encode(v: float) -> int:
    return lib().so_ue8m0_encode(float(v))


def quantize_fmt(x, rows: int, cols: int, fmin: int, fmax: int, fmt="mxfp4", gmode="none",
                 amax_bits: int | None = None, threads: int = 0) -> QuantResult:
    """so_quantize_fmt; codes are [rows][cols/2] nibbles (E2M1) or [rows][cols] bytes (E2M3)."""
    vf, sf, bs = FORMATS[fmt] if isinstance(fmt, str) else fmt
    x = _as_u16(x).reshape(-1)
    assert x.size == rows * cols
    gm = GMODES[gmode] if isinstance(gmode, str) else int(gmode)
    nb = rows * cols // bs
    codes = np.empty((rows, cols // 2 if vf == 0 else cols), np.uint8)
    scales = np.empty((rows, cols // bs), np.uint8)
    offs = np.empty(nb, np.int8)
    err = np.empty((nb, 2), np.float32)
    sums = np.zeros(2, np.float64)
    neval = np.zeros(1, np.int64)
    G = np.zeros(rows if gm == 3 else 1, np.float32)
    ab = None if amax_bits is None else np.array([amax_bits], np.uint32)
    _check(lib().so_quantize_fmt(_ptr(x), rows, cols, int(fmin), int(fmax), gm, _ptr(ab), vf, sf, bs,
                                 _ptr(codes), _ptr(scales), _ptr(offs), _ptr(err), _ptr(sums),
                                 _ptr(neval), _ptr(G), int(threads)))
    return QuantResult(codes, scales, offs, err, sums, int(neval[0]),
                       G.copy() if gm == 3 else float(G[0]))


def dequantize_fmt(codes, scales, rows: int, cols: int, fmt="mxfp4", G=1.0) -> np.ndarray:
    """bf16 bit patterns of xhat for a format; G scalar or per-row array."""
    vf, sf, bs = FORMATS[fmt] if isinstance(fmt, str) else fmt
    codes = np.ascontiguousarray(codes, np.uint8)
    scales = np.ascontiguousarray(scales, np.uint8)
    g = np.atleast_1d(np.asarray(G, np.float32)).copy()
    out = np.empty((rows, cols), np.uint16)
    _check(lib().so_dequantize_fmt(_ptr(codes), _ptr(scales), rows, cols, vf, sf, bs, _ptr(g),
                                   int(g.size > 1), _ptr(out)))
    return out


# ---------------------------------------------------------------------------
# Generic ExMy formats (fig:nvfp-scale / fig:nvfp-val /
# fig:mxfp P:237-260; reading R21).  A format is
# (value_e, value_m, scale_e, scale_m, block).
# ---------------------------------------------------------------------------
class _BlockResultFmt(ctypes.Structure):
    _fields_ = [("c0", ctypes.c_int32), ("cstar", ctypes.c_int32), ("fstar", ctypes.c_int32),
                ("n_evaluated", ctypes.c_int32), ("err_best", ctypes.c_float),
                ("err_base", ctypes.c_float), ("code", ctypes.c_uint8 * 256)]


def gen_value(e: int, m: int, code: int) -> float:
    return lib().so_gen_value(int(e), int(m), int(code))


def gen_encode(e: int, m: int, t: float) -> int:
    return lib().so_gen_encode(int(e), int(m), float(t))


def gen_scale_value(e: int, m: int, code: int) -> float:
    return lib().so_gen_scale_value(int(e), int(m), int(code))


def gen_scale_encode(e: int, m: int, v: float) -> int:
    return lib().so_gen_scale_encode(int(e), int(m), float(v))


def gen_numer(ve: int, vm: int, se: int, sm: int) -> float:
    return lib().so_gen_numer(int(ve), int(vm), int(se), int(sm))


def search_block_gen(y, fmt, fmin: int, fmax: int) -> BlockResult:
    ve, vm, se, sm, bs = fmt
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float32))
    assert y.shape == (bs,)
    r = _BlockResultFmt()
    _check(lib().so_search_block_gen(ve, vm, se, sm, bs, _ptr(y), int(fmin), int(fmax), ctypes.byref(r)))
    return BlockResult(r.c0, r.cstar, r.fstar, r.n_evaluated, r.err_best, r.err_base,
                       np.frombuffer(bytes(r.code), np.uint8)[:bs].copy())


def quantize_gen(x, rows: int, cols: int, fmin: int, fmax: int, fmt, gmode="tensor",
                 amax_bits: int | None = None, threads: int = 0) -> QuantResult:
    """so_quantize_gen: codes [rows][cols] one per byte, scales [rows][cols/bs]."""
    ve, vm, se, sm, bs = fmt
    x = _as_u16(x).reshape(-1)
    assert x.size == rows * cols
    gm = {"none": 0, "tensor": 1, "given": 2}[gmode] if isinstance(gmode, str) else int(gmode)
    nb = rows * cols // bs
    codes = np.empty((rows, cols), np.uint8)
    scales = np.empty((rows, cols // bs), np.uint8)
    offs = np.empty(nb, np.int8)
    err = np.empty((nb, 2), np.float32)
    sums = np.zeros(2, np.float64)
    neval = np.zeros(1, np.int64)
    G = np.zeros(1, np.float32)
    ab = None if amax_bits is None else np.array([amax_bits], np.uint32)
    _check(lib().so_quantize_gen(_ptr(x), rows, cols, int(fmin), int(fmax), gm, _ptr(ab), ve, vm, se, sm,
                                 bs, _ptr(codes), _ptr(scales), _ptr(offs), _ptr(err), _ptr(sums),
                                 _ptr(neval), _ptr(G), int(threads)))
    return QuantResult(codes, scales, offs, err, sums, int(neval[0]), float(G[0]))


def dequantize_gen(codes, scales, rows: int, cols: int, fmt, G=1.0) -> np.ndarray:
    ve, vm, se, sm, bs = fmt
    codes = np.ascontiguousarray(codes, np.uint8)
    scales = np.ascontiguousarray(scales, np.uint8)
    out = np.empty((rows, cols), np.uint16)
    _check(lib().so_dequantize_gen(_ptr(codes), _ptr(scales), rows, cols, ve, vm, se, sm, bs,
                                   ctypes.c_float(G), _ptr(out)))
    return out
