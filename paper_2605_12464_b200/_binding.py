"""ctypes binding of libss.so (include/ss.h).  Argument marshalling only.

Every step of the quantization runs in the sm_100a kernels behind the C ABI;
there is no Python or CPU compute path.  If the library cannot be loaded, or
the current device is not sm_100, calls raise ``SSError`` -- nothing falls back.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import NamedTuple, Optional

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libss.so")


def use_variant(name: Optional[str]) -> None:
    """Tools only: load libss_<name>.so (a tuning / counting build of the same
    sources, tools/kbench.py) instead of libss.so.  Must precede the first call."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("libss already loaded")
    LIB_PATH = os.path.join(PKG, "libss%s.so" % ("_" + name if name and name != "base" else ""))

SS_OK, SS_ERR_INVALID_ARG, SS_ERR_ALIGNMENT, SS_ERR_CUDA = 0, 1, 2, 3
SS_ERR_NONFINITE, SS_ERR_RANGE, SS_ERR_UNSUPPORTED_DEVICE = 4, 5, 6
GMODES = {"none": 0, "tensor": 1, "device_amax": 2, "row": 3}
SCALE_LAYOUTS = {"linear": 0, "swizzled": 1}
# block formats (ss.h SS_FMT_*): name -> (id, block size, value bytes per element)
FORMATS = {"nvfp4": (0, 16, 0.5), "mxfp4": (1, 32, 0.5), "mxfp6_e2m3": (2, 32, 1.0),
           "nvfp6_e2m3": (3, 16, 1.0), "nvfp4_b32": (4, 32, 0.5), "nvfp4_b64": (5, 64, 0.5),
           "nvfp4_b128": (6, 128, 0.5), "nvfp4_b256": (7, 256, 0.5)}
FLAG_NONFINITE, FLAG_RANGE = 1, 2

_lock = threading.Lock()
_lib = None


class SSError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = "libss: %s" % (status_string(status) if _lib is not None else "status %d" % status)
        super().__init__(msg + (" (%s)" % what if what else ""))


class TensorIO(ctypes.Structure):
    _fields_ = [
        ("in_bf16", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("d_amax_bits", ctypes.c_void_p),
        ("out_codes", ctypes.c_void_p),
        ("out_scales", ctypes.c_void_p),
        ("out_err", ctypes.c_void_p),
        ("out_offset", ctypes.c_void_p),
        ("d_err_sums", ctypes.c_void_p),
        ("d_global_scale", ctypes.c_void_p),
        ("scale_layout", ctypes.c_int),
    ]


class HostTensorIO(ctypes.Structure):
    _fields_ = [
        ("h_in_bf16", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("h_codes", ctypes.c_void_p),
        ("h_scales", ctypes.c_void_p),
        ("h_err", ctypes.c_void_p),
    ]


class QuantArgs(ctypes.Structure):
    _fields_ = [
        ("in_bf16", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("f_min", ctypes.c_int),
        ("f_max", ctypes.c_int),
        ("global_scale_mode", ctypes.c_int),
        ("d_amax_bits", ctypes.c_void_p),
        ("out_codes", ctypes.c_void_p),
        ("out_scales", ctypes.c_void_p),
        ("out_err", ctypes.c_void_p),
        ("out_offset", ctypes.c_void_p),
        ("d_err_sums", ctypes.c_void_p),
        ("d_global_scale", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("scale_layout", ctypes.c_int),
        ("format", ctypes.c_int),
    ]


class Plan(ctypes.Structure):
    """ss_plan: the launches a batched call would make (ss_quantize_plan)."""
    _fields_ = [
        ("amax_fused", ctypes.c_int),
        ("small_path", ctypes.c_int),
        ("row_fused", ctypes.c_int),
        ("launches", ctypes.c_int),
        ("trail_batches", ctypes.c_int),
    ]


class GenFormat(ctypes.Structure):
    """ss_gen_format: value ExMy, scale UExMy, block 16 or 32 (R21)."""
    _fields_ = [
        ("value_e", ctypes.c_int),
        ("value_m", ctypes.c_int),
        ("scale_e", ctypes.c_int),
        ("scale_m", ctypes.c_int),
        ("block", ctypes.c_int),
    ]


MAX_PEERS, IPC_HANDLE_BYTES = 8, 64


class Exchange(ctypes.Structure):
    """ss_exchange: every rank's exchange buffer as mapped in this process."""
    _fields_ = [
        ("world", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("buf", ctypes.c_void_p * MAX_PEERS),
        ("max_tensors", ctypes.c_int),
        ("max_groups", ctypes.c_int),
    ]


class ExchangeGroup(ctypes.Structure):
    _fields_ = [
        ("slot0", ctypes.c_int),
        ("count", ctypes.c_int),
        ("group", ctypes.c_int),
        ("epoch", ctypes.c_uint32),
    ]


class DequantArgs(ctypes.Structure):
    _fields_ = [
        ("codes", ctypes.c_void_p),
        ("scales", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("d_global_scale", ctypes.c_void_p),
        ("g_per_row", ctypes.c_int),
        ("scale_layout", ctypes.c_int),
        ("out_bf16", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("format", ctypes.c_int),
    ]


def lib():
    """Load libss.so (raises if it is missing: there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError("libss.so not built: run `python -m paper_2605_12464_b200.build` "
                                  "or __graft_entry__.build(); there is no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            P, i64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
            L.ss_status_string.restype = ctypes.c_char_p
            L.ss_status_string.argtypes = [I]
            L.ss_version.restype = I
            L.ss_version.argtypes = []
            L.ss_tensor_amax.restype = I
            L.ss_tensor_amax.argtypes = [P, i64, P, I, P]
            L.ss_quantize_nvfp4.restype = I
            L.ss_quantize_nvfp4.argtypes = [P, i64, i64, I, I, P, P, P, P]
            L.ss_tensor_amax_batched.restype = I
            L.ss_tensor_amax_batched.argtypes = [P, P, I, P, I, P]
            L.ss_quantize_nvfp4_batched.restype = I
            L.ss_quantize_nvfp4_batched.argtypes = [ctypes.POINTER(TensorIO), I, I, I, I, P]
            L.ss_quantize_nvfp4_ex.restype = I
            L.ss_quantize_nvfp4_ex.argtypes = [ctypes.POINTER(QuantArgs)]
            L.ss_dequantize_nvfp4_ex.restype = I
            L.ss_dequantize_nvfp4_ex.argtypes = [ctypes.POINTER(DequantArgs)]
            L.ss_scale_bytes.restype = i64
            L.ss_scale_bytes.argtypes = [i64, i64, I]
            L.ss_scale_bytes_fmt.restype = i64
            L.ss_scale_bytes_fmt.argtypes = [i64, i64, I, I]
            L.ss_code_bytes.restype = i64
            L.ss_code_bytes.argtypes = [i64, i64, I]
            L.ss_quantize_batched_fmt.restype = I
            L.ss_quantize_batched_fmt.argtypes = [ctypes.POINTER(TensorIO), I, I, I, I, I, P]
            L.ss_quantize_nvfp4_batched_next_amax.restype = I
            L.ss_quantize_nvfp4_batched_next_amax.argtypes = [ctypes.POINTER(TensorIO), I, I, I, P, P, I, P, P]
            L.ss_quantize_nvfp4_f32.restype = I
            L.ss_quantize_nvfp4_f32.argtypes = [P, i64, i64, I, I, P, P, P, P, P, P]
            L.ss_dequantize_nvfp4.restype = I
            L.ss_dequantize_nvfp4.argtypes = [P, P, i64, i64, P, P, P]
            L.ss_quantize_nvfp4_host.restype = I
            L.ss_quantize_nvfp4_host.argtypes = [P, i64, i64, I, I, I, P, P, P]
            L.ss_quantize_nvfp4_host_batched.restype = I
            L.ss_quantize_nvfp4_host_batched.argtypes = [ctypes.POINTER(HostTensorIO), I, I, I, I]
            L.ss_quantize_plan.restype = I
            L.ss_quantize_plan.argtypes = [ctypes.POINTER(TensorIO), I, I, I, I, I, ctypes.POINTER(Plan)]
            L.ss_quantize_gen.restype = I
            L.ss_quantize_gen.argtypes = [ctypes.POINTER(TensorIO), I, I, I, ctypes.POINTER(GenFormat), P]
            L.ss_dequantize_gen.restype = I
            L.ss_dequantize_gen.argtypes = [P, P, i64, i64, ctypes.POINTER(GenFormat), P, P, P]
            L.ss_exchange_bytes.restype = i64
            L.ss_exchange_bytes.argtypes = [I, I]
            L.ss_exchange_init.restype = I
            L.ss_exchange_init.argtypes = [P, I, I, P]
            L.ss_exchange_alloc.restype = I
            L.ss_exchange_alloc.argtypes = [I, I, ctypes.POINTER(ctypes.c_void_p)]
            L.ss_exchange_free.restype = I
            L.ss_exchange_free.argtypes = [P]
            L.ss_ipc_handle.restype = I
            L.ss_ipc_handle.argtypes = [P, P]
            L.ss_ipc_open.restype = I
            L.ss_ipc_open.argtypes = [P, ctypes.POINTER(ctypes.c_void_p)]
            L.ss_ipc_close.restype = I
            L.ss_ipc_close.argtypes = [P]
            L.ss_exchange_publish.restype = I
            L.ss_exchange_publish.argtypes = [ctypes.POINTER(Exchange), ctypes.POINTER(ExchangeGroup), P, P]
            L.ss_quantize_nvfp4_exchange.restype = I
            L.ss_quantize_nvfp4_exchange.argtypes = [ctypes.POINTER(TensorIO), I, I, I, ctypes.POINTER(Exchange),
                                                     ctypes.POINTER(ExchangeGroup), P, P, I, P,
                                                     ctypes.POINTER(ExchangeGroup), P]
            L.ss_get_device_status.restype = I
            L.ss_get_device_status.argtypes = [ctypes.POINTER(ctypes.c_int), P]
            _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().ss_status_string(int(status)).decode()


def _check(st: int, what: str = ""):
    if st != SS_OK:
        raise SSError(st, what)


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _window(radius, fmin, fmax):
    if fmin is None and fmax is None:
        r = 8 if radius is None else int(radius)
        if r < 0:
            raise ValueError("radius must be >= 0")
        return -min(r, 126), min(r, 126)
    if radius is not None:
        raise ValueError("give either radius or (fmin, fmax)")
    return int(fmin), int(fmax)


class QuantOut(NamedTuple):
    codes: "torch.Tensor"            # [rows][cols/2] uint8
    scales: "torch.Tensor"           # [rows][cols/16] uint8 (E4M3 codes)
    err: "Optional[torch.Tensor]"    # [nb][2] float32 {best, base}
    offsets: "Optional[torch.Tensor]"  # [nb] int8
    sums: "Optional[torch.Tensor]"   # [2] float64
    G: "Optional[torch.Tensor]"      # [1] float32


def tensor_amax(x, out=None, accumulate: bool = False, stream=None):
    """Device u32 tensor holding the FP32 bits of max|x| (ss_tensor_amax)."""
    import torch
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous()
    if out is None:
        out = torch.zeros(1, dtype=torch.int32, device=x.device)
    _check(lib().ss_tensor_amax(_ptr(x), x.numel(), _ptr(out), int(accumulate), _stream_ptr(stream)),
           "ss_tensor_amax")
    return out


def quantize(x, radius=None, fmin=None, fmax=None, gmode: str = "tensor", amax=None,
             want_err: bool = True, want_offsets: bool = True, want_sums: bool = True,
             want_g: bool = True, out: Optional[QuantOut] = None, scale_layout: str = "linear",
             fmt: str = "nvfp4", stream=None) -> QuantOut:
    """ScaleSearch NVFP4 quantization of a [rows][cols] bf16 CUDA tensor (ss_quantize_nvfp4_ex)."""
    import torch
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous() and x.dim() == 2
    rows, cols = x.shape
    lo, hi = _window(radius, fmin, fmax)
    gm = GMODES[gmode]
    if gm == 2 and amax is None:
        raise ValueError("gmode='device_amax' needs amax (device int32/uint32 tensor)")
    if out is None:
        out = alloc_out(x, want_err, want_offsets, want_sums, want_g, scale_layout, gmode, fmt)
    a = QuantArgs(_ptr(x), rows, cols, lo, hi, gm, _ptr(amax), _ptr(out.codes), _ptr(out.scales),
                  _ptr(out.err), _ptr(out.offsets), _ptr(out.sums), _ptr(out.G), _stream_ptr(stream),
                  SCALE_LAYOUTS[scale_layout], FORMATS[fmt][0])
    _check(lib().ss_quantize_nvfp4_ex(ctypes.byref(a)), "ss_quantize_nvfp4_ex")
    return out


def tensor_amax_batched(xs, out=None, accumulate: bool = False, stream=None):
    """Device int32 [len(xs)] of FP32 amax bits, one launch (ss_tensor_amax_batched)."""
    import torch
    n = len(xs)
    for x in xs:
        assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous()
    if out is None:
        out = torch.zeros(n, dtype=torch.int32, device=xs[0].device if n else "cuda")
    ptrs = (ctypes.c_void_p * max(n, 1))(*[x.data_ptr() for x in xs])
    ns = (ctypes.c_int64 * max(n, 1))(*[x.numel() for x in xs])
    _check(lib().ss_tensor_amax_batched(ptrs, ns, n, _ptr(out), int(accumulate), _stream_ptr(stream)),
           "ss_tensor_amax_batched")
    return out


def scale_bytes(rows: int, cols: int, scale_layout: str = "linear", fmt: str = "nvfp4") -> int:
    return int(lib().ss_scale_bytes_fmt(rows, cols, SCALE_LAYOUTS[scale_layout], FORMATS[fmt][0]))


def alloc_out(x, want_err=True, want_offsets=True, want_sums=True, want_g=True,
              scale_layout: str = "linear", gmode: str = "tensor", fmt: str = "nvfp4") -> QuantOut:
    """Output buffers for ``x`` in block format ``fmt``: codes [rows][cols/2]
    (E2M1) or [rows][cols] (E2M3); scales [rows][cols/bs] (linear) or the flat
    swizzled tile buffer; per-block errors/offsets; G [1] or [rows] (gmode 'row')."""
    import torch
    rows, cols = x.shape
    _, bs, vbytes = FORMATS[fmt]
    nsb = rows * cols // bs
    dev = x.device
    scales = (torch.empty(rows, cols // bs, dtype=torch.uint8, device=dev)
              if scale_layout == "linear" else
              torch.empty(scale_bytes(rows, cols, scale_layout, fmt), dtype=torch.uint8, device=dev))
    return QuantOut(
        torch.empty(rows, int(cols * vbytes), dtype=torch.uint8, device=dev),
        scales,
        torch.empty(nsb, 2, dtype=torch.float32, device=dev) if want_err else None,
        torch.empty(nsb, dtype=torch.int8, device=dev) if want_offsets else None,
        torch.empty(2, dtype=torch.float64, device=dev) if want_sums else None,
        torch.empty(rows if gmode == "row" else 1, dtype=torch.float32, device=dev)
        if (want_g or gmode == "row") else None,
    )


def quantize_batched(xs, outs, radius=None, fmin=None, fmax=None, gmode: str = "tensor",
                     amax=None, scale_layout: str = "linear", fmt: str = "nvfp4", stream=None):
    """All tensors of ``xs`` into ``outs`` (QuantOut each) in one call
    (ss_quantize_nvfp4_batched).  ``amax``: device int32 [len(xs)] for
    gmode='device_amax' (e.g. after the NCCL max all-reduce)."""
    import torch
    lo, hi = _window(radius, fmin, fmax)
    gm = GMODES[gmode]
    n = len(xs)
    if gm == 2:
        if amax is None or amax.numel() < n:
            raise ValueError("gmode='device_amax' needs amax with one slot per tensor")
    arr = (TensorIO * max(n, 1))()
    for i, (x, o) in enumerate(zip(xs, outs)):
        assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous() and x.dim() == 2
        rows, cols = x.shape
        arr[i] = TensorIO(_ptr(x), rows, cols, amax.data_ptr() + 4 * i if gm == 2 else None,
                          _ptr(o.codes), _ptr(o.scales), _ptr(o.err), _ptr(o.offsets), _ptr(o.sums),
                          _ptr(o.G), SCALE_LAYOUTS[scale_layout])
    if fmt == "nvfp4":
        _check(lib().ss_quantize_nvfp4_batched(arr, n, lo, hi, gm, _stream_ptr(stream)),
               "ss_quantize_nvfp4_batched")
    else:
        _check(lib().ss_quantize_batched_fmt(arr, n, lo, hi, gm, FORMATS[fmt][0], _stream_ptr(stream)),
               "ss_quantize_batched_fmt")
    return outs


def quantize_f32(x, radius=None, fmin=None, fmax=None, G=None, want_err: bool = True,
                 want_offsets: bool = True, stream=None):
    """FP32 [rows][cols] CUDA tensor through the one-thread block routine
    (ss_quantize_nvfp4_f32); ``G``: device float32 [1] global scale or None (G = 1).
    Returns QuantOut (sums / G fields None)."""
    import torch
    assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous() and x.dim() == 2
    rows, cols = x.shape
    lo, hi = _window(radius, fmin, fmax)
    dev = x.device
    out = QuantOut(torch.empty(rows, cols // 2, dtype=torch.uint8, device=dev),
                   torch.empty(rows, cols // 16, dtype=torch.uint8, device=dev),
                   torch.empty(rows * cols // 16, 2, dtype=torch.float32, device=dev) if want_err else None,
                   torch.empty(rows * cols // 16, dtype=torch.int8, device=dev) if want_offsets else None,
                   None, None)
    _check(lib().ss_quantize_nvfp4_f32(_ptr(x), rows, cols, lo, hi, _ptr(G), _ptr(out.codes),
                                       _ptr(out.scales), _ptr(out.err), _ptr(out.offsets),
                                       _stream_ptr(stream)), "ss_quantize_nvfp4_f32")
    return out


def quantize_batched_next_amax(xs, outs, amax, next_xs, next_amax, radius=None, fmin=None, fmax=None,
                               stream=None):
    """Quantize ``xs`` with their (all-reduced) ``amax`` and compute, in the same
    launch, the local amax of ``next_xs`` into ``next_amax`` (device int32
    [len(next_xs)], overwritten) -- ss_quantize_nvfp4_batched_next_amax."""
    import torch
    lo, hi = _window(radius, fmin, fmax)
    n, m = len(xs), len(next_xs)
    arr = (TensorIO * max(n, 1))()
    for i, (x, o) in enumerate(zip(xs, outs)):
        assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous() and x.dim() == 2
        rows, cols = x.shape
        arr[i] = TensorIO(_ptr(x), rows, cols, amax.data_ptr() + 4 * i, _ptr(o.codes), _ptr(o.scales),
                          _ptr(o.err), _ptr(o.offsets), _ptr(o.sums), _ptr(o.G), SCALE_LAYOUTS["linear"])
    for x in next_xs:
        assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous()
    ptrs = (ctypes.c_void_p * max(m, 1))(*[x.data_ptr() for x in next_xs])
    ns = (ctypes.c_int64 * max(m, 1))(*[x.numel() for x in next_xs])
    _check(lib().ss_quantize_nvfp4_batched_next_amax(arr, n, lo, hi, ptrs, ns, m, _ptr(next_amax),
                                                      _stream_ptr(stream)),
           "ss_quantize_nvfp4_batched_next_amax")
    return outs


def quantize_simple(x, radius: int, gmode: str, codes, scales, err=None, stream=None):
    """The three-output entry point of the north star (ss_quantize_nvfp4)."""
    rows, cols = x.shape
    _check(lib().ss_quantize_nvfp4(_ptr(x), rows, cols, int(radius), GMODES[gmode], _ptr(codes),
                                   _ptr(scales), _ptr(err), _stream_ptr(stream)), "ss_quantize_nvfp4")


def dequantize(codes, scales, rows: int, cols: int, G=None, out=None, stream=None,
               scale_layout: str = "linear", fmt: str = "nvfp4"):
    """bf16 [rows][cols] reconstruction (ss_dequantize_nvfp4_ex); G is a device
    f32 [1], a per-row [rows] (gmode 'row'), or None (G = 1)."""
    import torch
    if out is None:
        out = torch.empty(rows, cols, dtype=torch.bfloat16, device=codes.device)
    per_row = G is not None and G.numel() == rows and rows > 1
    a = DequantArgs(_ptr(codes), _ptr(scales), rows, cols, _ptr(G), int(per_row),
                    SCALE_LAYOUTS[scale_layout], _ptr(out), _stream_ptr(stream), FORMATS[fmt][0])
    _check(lib().ss_dequantize_nvfp4_ex(ctypes.byref(a)), "ss_dequantize_nvfp4_ex")
    return out


def quantize_host(h_x, rows: int, cols: int, fmin: int, fmax: int, gmode: str,
                  h_codes, h_scales, h_err=None):
    """End to end from host memory (ss_quantize_nvfp4_host); synchronous."""
    _check(lib().ss_quantize_nvfp4_host(_ptr(h_x), rows, cols, int(fmin), int(fmax), GMODES[gmode],
                                        _ptr(h_codes), _ptr(h_scales), _ptr(h_err)),
           "ss_quantize_nvfp4_host")


def quantize_host_batched(h_xs, h_codes, h_scales, h_errs=None, radius=None, fmin=None,
                          fmax=None, gmode: str = "tensor"):
    """End to end from host memory for a list of tensors (ss_quantize_nvfp4_host_batched);
    synchronous.  Host tensors should be pinned."""
    lo, hi = _window(radius, fmin, fmax)
    n = len(h_xs)
    arr = (HostTensorIO * max(n, 1))()
    for i, x in enumerate(h_xs):
        rows, cols = x.shape
        arr[i] = HostTensorIO(_ptr(x), rows, cols, _ptr(h_codes[i]), _ptr(h_scales[i]),
                              _ptr(h_errs[i]) if h_errs is not None else None)
    _check(lib().ss_quantize_nvfp4_host_batched(arr, n, lo, hi, GMODES[gmode]),
           "ss_quantize_nvfp4_host_batched")


def device_status(stream=None) -> int:
    f = ctypes.c_int(0)
    _check(lib().ss_get_device_status(ctypes.byref(f), _stream_ptr(stream)), "ss_get_device_status")
    return f.value


def plan(shapes, radius=None, fmin=None, fmax=None, gmode: str = "tensor", fmt: str = "nvfp4",
         want_err: bool = True, want_sums: bool = True, scale_layout: str = "linear") -> Plan:
    """The library's launch plan for a batched call over tensors of these
    (rows, cols) shapes (ss_quantize_plan; no device needed, nothing runs)."""
    lo, hi = _window(radius, fmin, fmax)
    n = len(shapes)
    dummy = 1 << 20                     # aligned placeholder: the plan never reads pointers
    arr = (TensorIO * max(n, 1))()
    gm = GMODES[gmode]
    for i, (rows, cols) in enumerate(shapes):
        arr[i] = TensorIO(dummy, rows, cols, dummy if gm == 2 else None, dummy, dummy,
                          dummy if want_err else None, None, dummy if want_sums else None,
                          dummy if gm == 3 else None, SCALE_LAYOUTS[scale_layout])
    out = Plan()
    _check(lib().ss_quantize_plan(arr, n, lo, hi, gm, FORMATS[fmt][0], ctypes.byref(out)), "ss_quantize_plan")
    return out


def quantize_gen(x, fmt, radius=None, fmin=None, fmax=None, gmode: str = "tensor", amax=None,
                 want_err: bool = True, want_offsets: bool = True, want_sums: bool = True,
                 want_g: bool = True, stream=None) -> QuantOut:
    """ScaleSearch over a generic ExMy format ``fmt`` = (value_e, value_m,
    scale_e, scale_m, block) (ss_quantize_gen).  Codes [rows][cols], one per byte."""
    import torch
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous() and x.dim() == 2
    rows, cols = x.shape
    ve, vm, se, sm, bs = fmt
    lim = (1 << (se + sm)) - 2
    if fmin is None and fmax is None:
        r = 8 if radius is None else int(radius)
        lo, hi = -min(r, lim), min(r, lim)
    else:
        lo, hi = int(fmin), int(fmax)
    gm = GMODES[gmode]
    if gm == 2 and amax is None:
        raise ValueError("gmode='device_amax' needs amax")
    dev = x.device
    nb = rows * cols // bs
    out = QuantOut(torch.empty(rows, cols, dtype=torch.uint8, device=dev),
                   torch.empty(rows, cols // bs, dtype=torch.uint8, device=dev),
                   torch.empty(nb, 2, dtype=torch.float32, device=dev) if want_err else None,
                   torch.empty(nb, dtype=torch.int8, device=dev) if want_offsets else None,
                   torch.empty(2, dtype=torch.float64, device=dev) if want_sums else None,
                   torch.empty(1, dtype=torch.float32, device=dev) if want_g else None)
    t = TensorIO(_ptr(x), rows, cols, _ptr(amax) if gm == 2 else None, _ptr(out.codes), _ptr(out.scales),
                 _ptr(out.err), _ptr(out.offsets), _ptr(out.sums), _ptr(out.G), 0)
    f = GenFormat(ve, vm, se, sm, bs)
    _check(lib().ss_quantize_gen(ctypes.byref(t), lo, hi, gm, ctypes.byref(f), _stream_ptr(stream)),
           "ss_quantize_gen")
    return out


def dequantize_gen(codes, scales, rows: int, cols: int, fmt, G=None, out=None, stream=None):
    """bf16 [rows][cols] from ss_quantize_gen outputs (ss_dequantize_gen)."""
    import torch
    if out is None:
        out = torch.empty(rows, cols, dtype=torch.bfloat16, device=codes.device)
    f = GenFormat(*fmt)
    _check(lib().ss_dequantize_gen(_ptr(codes), _ptr(scales), rows, cols, ctypes.byref(f), _ptr(G),
                                   _ptr(out), _stream_ptr(stream)), "ss_dequantize_gen")
    return out


# ---------------------------------------------------------------------------
# Peer-memory amax exchange (include/ss.h)
# ---------------------------------------------------------------------------
def exchange_bytes(max_tensors: int, max_groups: int) -> int:
    return int(lib().ss_exchange_bytes(int(max_tensors), int(max_groups)))


def exchange_alloc(max_tensors: int, max_groups: int) -> int:
    """A zeroed exchange buffer in its own cudaMalloc allocation (device pointer;
    the current device); free with exchange_free."""
    out = ctypes.c_void_p()
    _check(lib().ss_exchange_alloc(int(max_tensors), int(max_groups), ctypes.byref(out)), "ss_exchange_alloc")
    return int(out.value)


def exchange_free(ptr: int) -> None:
    _check(lib().ss_exchange_free(ctypes.c_void_p(ptr)), "ss_exchange_free")


def ipc_handle(ptr: int) -> bytes:
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(lib().ss_ipc_handle(ctypes.c_void_p(ptr), h), "ss_ipc_handle")
    return h.raw


def ipc_open(handle: bytes) -> int:
    out = ctypes.c_void_p()
    _check(lib().ss_ipc_open(ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES), ctypes.byref(out)),
           "ss_ipc_open")
    return int(out.value)


def ipc_close(ptr: int) -> None:
    _check(lib().ss_ipc_close(ctypes.c_void_p(ptr)), "ss_ipc_close")


def make_exchange(world: int, rank: int, ptrs, max_tensors: int, max_groups: int) -> Exchange:
    x = Exchange()
    x.world, x.rank, x.max_tensors, x.max_groups = world, rank, max_tensors, max_groups
    for r, p_ in enumerate(ptrs):
        x.buf[r] = p_
    return x


def exchange_publish(x: Exchange, slot0: int, group: int, epoch: int, local_amax, stream=None):
    g = ExchangeGroup(slot0, local_amax.numel(), group, epoch)
    _check(lib().ss_exchange_publish(ctypes.byref(x), ctypes.byref(g), _ptr(local_amax), _stream_ptr(stream)),
           "ss_exchange_publish")


def quantize_exchange(xs, outs, x: Exchange, slot0: int, group: int, epoch: int, next_xs=None,
                      next_amax=None, next_slot0: int = 0, radius=None, fmin=None, fmax=None, stream=None):
    """Quantize ``xs`` (a group of row shards; zero-row shards included) with G
    from the ranks' amaxes in the exchange, and publish the local amaxes of
    ``next_xs`` (computed in the same launch into ``next_amax``) as group
    ``group + 1`` (ss_quantize_nvfp4_exchange)."""
    lo, hi = _window(radius, fmin, fmax)
    n = len(xs)
    arr = (TensorIO * max(n, 1))()
    for i, (t, o) in enumerate(zip(xs, outs)):
        rows, cols = t.shape
        arr[i] = TensorIO(_ptr(t) if t.numel() else None, rows, cols, None, _ptr(o.codes) if t.numel() else None,
                          _ptr(o.scales) if t.numel() else None, _ptr(o.err) if t.numel() else None,
                          _ptr(o.offsets) if t.numel() else None, _ptr(o.sums), _ptr(o.G), 0)
    gin = ExchangeGroup(slot0, n, group, epoch)
    nn = len(next_xs) if next_xs else 0
    ptrs = (ctypes.c_void_p * max(nn, 1))(*[t.data_ptr() if t.numel() else None for t in (next_xs or [])])
    ns = (ctypes.c_int64 * max(nn, 1))(*[t.numel() for t in (next_xs or [])])
    gout = ExchangeGroup(next_slot0, nn, group + 1, epoch)
    _check(lib().ss_quantize_nvfp4_exchange(arr, n, lo, hi, ctypes.byref(x), ctypes.byref(gin), ptrs, ns, nn,
                                            _ptr(next_amax) if nn else None, ctypes.byref(gout) if nn else None,
                                            _stream_ptr(stream)), "ss_quantize_nvfp4_exchange")
    return outs
