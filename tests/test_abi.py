"""The C-ABI library builds, loads and exports every symbol include/ss.h declares;
argument errors are synchronous; without an sm_100 device nothing falls back."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ss.h")


@pytest.fixture(scope="module")
def L():
    from paper_2605_12464_b200 import build, _binding
    build.build()
    return _binding.lib()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert {"ss_tensor_amax", "ss_quantize_nvfp4", "ss_dequantize_nvfp4"} <= set(names)
    for n in names:
        assert hasattr(L, n), n
    nm = os.popen("nm -D --defined-only %s" % os.path.join(ROOT, "paper_2605_12464_b200", "libss.so")).read()
    exported = set(re.findall(r"\bT (ss_\w+)", nm))
    assert set(names) == exported, (set(names) ^ exported)


def test_status_strings(L):
    assert L.ss_version() == 500
    for s in range(7):
        assert L.ss_status_string(s)
    assert L.ss_status_string(6).decode().startswith("unsupported device")


def test_argument_errors_are_synchronous(L):
    from paper_2605_12464_b200 import _binding as B
    P = ctypes.c_void_p
    buf = ctypes.create_string_buffer(1024 + 64)
    base = (ctypes.addressof(buf) + 63) // 64 * 64
    # cols % 16 != 0
    assert L.ss_quantize_nvfp4(P(base), 4, 24, 8, 1, P(base), P(base), None, None) == B.SS_ERR_INVALID_ARG
    # negative radius / rows
    assert L.ss_quantize_nvfp4(P(base), 4, 32, -1, 1, P(base), P(base), None, None) == B.SS_ERR_INVALID_ARG
    assert L.ss_quantize_nvfp4(P(base), -1, 32, 8, 1, P(base), P(base), None, None) == B.SS_ERR_INVALID_ARG
    # null outputs
    assert L.ss_quantize_nvfp4(P(base), 4, 32, 8, 1, None, P(base), None, None) == B.SS_ERR_INVALID_ARG
    # misaligned input
    assert L.ss_quantize_nvfp4(P(base + 2), 4, 32, 8, 1, P(base), P(base), None, None) == B.SS_ERR_ALIGNMENT
    # f_min > 0 in the extended form; DEVICE_AMAX without a pointer
    a = B.QuantArgs(base, 4, 32, 1, 8, 0, None, base, base, None, None, None, None, None)
    assert L.ss_quantize_nvfp4_ex(ctypes.byref(a)) == B.SS_ERR_INVALID_ARG
    a = B.QuantArgs(base, 4, 32, -2, 6, 2, None, base, base, None, None, None, None, None)
    assert L.ss_quantize_nvfp4_ex(ctypes.byref(a)) == B.SS_ERR_INVALID_ARG
    assert L.ss_tensor_amax(P(base), -5, P(base), 0, None) == B.SS_ERR_INVALID_ARG
    assert L.ss_dequantize_nvfp4(P(base), P(base), 4, 20, None, P(base), None) == B.SS_ERR_INVALID_ARG
    # batched forms: bad shape / window / missing amax / misalignment, all before any launch
    io = (B.TensorIO * 2)()
    io[0] = B.TensorIO(base, 4, 32, None, base, base, None, None, None, None)
    io[1] = B.TensorIO(base, 4, 24, None, base, base, None, None, None, None)
    assert L.ss_quantize_nvfp4_batched(io, 2, -8, 8, 1, None) == B.SS_ERR_INVALID_ARG
    io[1] = B.TensorIO(base, 4, 32, None, base, base, None, None, None, None)
    assert L.ss_quantize_nvfp4_batched(io, 2, 1, 8, 1, None) == B.SS_ERR_INVALID_ARG
    assert L.ss_quantize_nvfp4_batched(io, 2, -8, 8, 2, None) == B.SS_ERR_INVALID_ARG
    io[1] = B.TensorIO(base + 2, 4, 32, None, base, base, None, None, None, None)
    assert L.ss_quantize_nvfp4_batched(io, 2, -8, 8, 1, None) == B.SS_ERR_ALIGNMENT
    ptrs = (P * 2)(base, base + 8)
    ns = (ctypes.c_int64 * 2)(64, 64)
    assert L.ss_tensor_amax_batched(ptrs, ns, 2, P(base), 0, None) == B.SS_ERR_ALIGNMENT
    ns[1] = -1
    ptrs[1] = base
    assert L.ss_tensor_amax_batched(ptrs, ns, 2, P(base), 0, None) == B.SS_ERR_INVALID_ARG
    # FP32 block-routine entry point (ss_quantize_nvfp4_f32)
    F = L.ss_quantize_nvfp4_f32
    assert F(P(base), 4, 24, -8, 8, None, P(base), P(base), None, None, None) == B.SS_ERR_INVALID_ARG
    assert F(P(base), 4, 32, 1, 8, None, P(base), P(base), None, None, None) == B.SS_ERR_INVALID_ARG
    assert F(P(base), 4, 32, -8, 8, None, None, P(base), None, None, None) == B.SS_ERR_INVALID_ARG
    assert F(P(base + 4), 4, 32, -8, 8, None, P(base), P(base), None, None, None) == B.SS_ERR_ALIGNMENT
    assert F(P(base), 4, 32, -8, 8, P(base + 2), P(base), P(base), None, None, None) == B.SS_ERR_ALIGNMENT


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is None and
                    os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_fallback_without_device(L):
    # valid arguments on a host without an sm_100 device: an error, never a CPU result
    from paper_2605_12464_b200 import _binding as B
    P = ctypes.c_void_p
    buf = ctypes.create_string_buffer(4096)
    base = (ctypes.addressof(buf) + 63) // 64 * 64
    st = L.ss_quantize_nvfp4(P(base), 2, 32, 8, 1, P(base + 1024), P(base + 2048), None, None)
    assert st == B.SS_ERR_UNSUPPORTED_DEVICE
    assert L.ss_tensor_amax(P(base), 64, P(base + 1024), 0, None) == B.SS_ERR_UNSUPPORTED_DEVICE
    io = (B.TensorIO * 1)(B.TensorIO(base, 2, 32, None, base + 1024, base + 2048, None, None, None,
                                     None))
    assert L.ss_quantize_nvfp4_batched(io, 1, -8, 8, 1, None) == B.SS_ERR_UNSUPPORTED_DEVICE
    assert L.ss_quantize_nvfp4_f32(P(base), 2, 32, -8, 8, None, P(base + 1024), P(base + 2048), None, None,
                                   None) == B.SS_ERR_UNSUPPORTED_DEVICE


def test_binding_raises_not_falls_back():
    from paper_2605_12464_b200 import _binding as B
    e = B.SSError(B.SS_ERR_UNSUPPORTED_DEVICE, "x")
    assert isinstance(e, RuntimeError)


def test_device_header_compiles_standalone(tmp_path):
    """include/ss_device.cuh is usable from a user's own kernel (nvcc, sm_100a),
    with no library symbols needed."""
    import shutil
    import subprocess
    if not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    src = tmp_path / "user.cu"
    src.write_text(
        '#include "ss_device.cuh"\n'
        "__global__ void user_kernel(const float* x, uint2* codes, unsigned char* scales) {\n"
        "  float y[16];\n"
        "  for (int i = 0; i < 16; i++) y[i] = x[16 * threadIdx.x + i];\n"
        "  if (threadIdx.x & 1) return;   // divergent callers are fine\n"
        "  ss::Nvfp4Block r = ss::search_nvfp4_block<8, 8>(y);\n"
        "  ss::Nvfp4Block q = ss::search_nvfp4_block<-1, -1>(y, -2, 6);\n"
        "  codes[threadIdx.x] = r.codes;\n"
        "  scales[threadIdx.x] = (unsigned char)(r.scale ^ q.scale);\n"
        "}\n")
    res = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-c",
                          "-I", os.path.join(ROOT, "include"), "-o", str(tmp_path / "user.o"), str(src)],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def test_quantize_plan_trail(L):
    """The trailing-amax chain of DESIGN.md §4.2c as ss_quantize_plan reports
    it: per-tensor-G calls of >= 2^26 elements and >= 2 tensors; batch 0
    ~1/64 of the elements, each later batch at most twice its predecessor and
    at most 64 tensors; one quantize (+ error-sum) launch per batch."""
    import ssgen
    from paper_2605_12464_b200 import _binding as B
    specs = ssgen.workload("c2_qwen3_8b_weights")
    shapes = [(s.rows, s.cols) for s in specs]
    p = B.plan(shapes, radius=8)
    assert p.amax_fused == 1 and p.trail_batches == 8 and p.launches == 16
    assert B.plan(shapes, radius=8, want_sums=False).launches == 8
    assert B.plan(shapes, radius=8, gmode="device_amax").trail_batches == 0     # amax given
    assert B.plan(shapes, radius=1).trail_batches == 0                           # HBM-bound window
    assert B.plan([(4096, 4096)] * 3, radius=8).trail_batches == 0               # < 2^26 elements
    assert B.plan([(16384, 8192)], radius=8).trail_batches == 0                  # one tensor
    p = B.plan([(64, 64)] * 300 + [(4096, 4096)] * 4, radius=8)                  # <= 64 tensors per batch
    assert p.trail_batches >= 300 // 64
    p = B.plan([(1, 16)] * 30 + [(16384, 4096)], radius=8)                      # huge after tiny: own amax
    assert p.amax_fused == 1 and p.trail_batches == 2 and p.launches == 4


def test_quantize_plan(L):
    """ss_quantize_plan (no device needed): the fused-amax rule (>= 4 offsets,
    first tensor <= half of the batch), the small-tensor path,
    row fusion and the launch counts bench.py reports."""
    from paper_2605_12464_b200 import _binding as B
    p = B.plan([(10, 160), (10, 160)], radius=8)
    assert p.amax_fused == 1 and p.small_path == 0 and p.launches == 2          # quant + sums
    assert B.plan([(0, 16), (10, 160), (10, 160)], fmin=-2, fmax=1).amax_fused == 1
    p = B.plan([(11, 160), (10, 160)], radius=8)                                  # first dominates
    assert p.amax_fused == 0 and p.launches == 3                                  # amax + quant + sums
    p = B.plan([(10, 160)], radius=8)                                             # one small tensor
    assert p.amax_fused == 0 and p.small_path == 1 and p.launches == 3
    assert B.plan([(10, 160)], radius=8, want_sums=False).launches == 2
    p = B.plan([(4096, 4096)] * 2, radius=1)                                      # HBM-bound window
    assert p.amax_fused == 0 and p.launches == 3
    assert B.plan([], radius=8).launches == 0
    p = B.plan([(64, 64)] * 130, radius=8)                                        # 2 launches of <= 128
    assert p.amax_fused == 1 and p.launches == 4
    p = B.plan([(64, 64)] * 130, radius=8, gmode="device_amax", want_sums=False)
    assert p.launches == 2
    p = B.plan([(8, 4096), (8, 256)], radius=8, gmode="row")                      # one row-fused tensor
    assert p.row_fused == 1 and p.launches == 1 + 1 + 1                            # rowscale + quant + sums
    assert B.plan([(8, 4096)], radius=1, gmode="row").row_fused == 0              # narrow: two-pass
    with pytest.raises(B.SSError):
        B.plan([(4, 24)], radius=8)


def test_e2m3_codes_need_16_byte_alignment(L):
    """E2M3 codes are stored as 16-B vectors: 8-B aligned code buffers are
    rejected synchronously (quantize and dequantize), E2M1 ones accepted."""
    from paper_2605_12464_b200 import _binding as B
    buf = ctypes.create_string_buffer(8192)
    base = (ctypes.addressof(buf) + 255) // 256 * 256
    for fmt, want in (("nvfp6_e2m3", B.SS_ERR_ALIGNMENT), ("mxfp6_e2m3", B.SS_ERR_ALIGNMENT)):
        io = (B.TensorIO * 1)(B.TensorIO(base, 2, 32, None, base + 1024 + 8, base + 2048, None, None, None,
                                         None, 0))
        assert L.ss_quantize_batched_fmt(io, 1, -1, 1, 0, B.FORMATS[fmt][0], None) == want
        d = B.DequantArgs(base + 8, base + 2048, 2, 32, None, 0, 0, base + 4096, None, B.FORMATS[fmt][0])
        assert L.ss_dequantize_nvfp4_ex(ctypes.byref(d)) == want
    # an 8-B aligned E2M1 code buffer passes validation (then: no device here, or it runs)
    io = (B.TensorIO * 1)(B.TensorIO(base, 2, 32, None, base + 1024 + 8, base + 2048, None, None, None,
                                     None, 0))
    assert L.ss_quantize_batched_fmt(io, 1, -1, 1, 0, B.FORMATS["mxfp4"][0], None) != B.SS_ERR_ALIGNMENT


def test_piece_limit_plan(L):
    """Tensors over the kernels' 32-bit half-block index are accepted (they run
    as row pieces, never with the fused amax); a single row (or, swizzled, a
    128-row band) over the piece limit is rejected synchronously."""
    from paper_2605_12464_b200 import _binding as B
    big = (1 << 20) + 1024, 32768                      # 2^31 + 2^21 half-blocks
    p = B.plan([(4096, 4096), big], radius=8)       # would fuse without the split
    assert p.amax_fused == 0
    assert B.plan([(4096, 4096), (4096, 4096)], radius=8).amax_fused == 1
    with pytest.raises(B.SSError):
        B.plan([(2, 1 << 36)], radius=8)                # one row of 2^32 half-blocks
    with pytest.raises(B.SSError):                      # 128 rows of 2^25 half-blocks: no swizzled piece
        B.plan([(256, 1 << 29)], radius=8, scale_layout="swizzled")


def test_generic_and_exchange_argument_errors(L):
    """ss_quantize_gen / ss_dequantize_gen and the peer-exchange entry points
    reject bad arguments synchronously (no device needed)."""
    from paper_2605_12464_b200 import _binding as B
    P = ctypes.c_void_p
    buf = ctypes.create_string_buffer(4096 + 64)
    base = (ctypes.addressof(buf) + 63) // 64 * 64
    io = B.TensorIO(base, 4, 64, None, base, base, None, None, None, None, 0)
    for fmt in ((0, 3, 4, 3, 16), (2, 6, 4, 3, 16), (2, 1, 8, 1, 16), (2, 1, 4, 3, 48), (2, 1, 9, 0, 16)):
        f = B.GenFormat(*fmt)
        assert L.ss_quantize_gen(ctypes.byref(io), -2, 2, 0, ctypes.byref(f), None) == B.SS_ERR_INVALID_ARG
    f = B.GenFormat(2, 1, 8, 0, 32)     # UE8M0: no global scale (vmax * smax overflows binary32)
    assert L.ss_quantize_gen(ctypes.byref(io), -2, 2, 1, ctypes.byref(f), None) == B.SS_ERR_INVALID_ARG
    f = B.GenFormat(2, 1, 4, 3, 16)
    assert L.ss_quantize_gen(ctypes.byref(io), 1, 2, 0, ctypes.byref(f), None) == B.SS_ERR_INVALID_ARG
    bad = B.TensorIO(base, 4, 64, None, base + 8, base, None, None, None, None, 0)  # codes not 16-B aligned
    assert L.ss_quantize_gen(ctypes.byref(bad), -2, 2, 0, ctypes.byref(f), None) == B.SS_ERR_ALIGNMENT
    assert L.ss_dequantize_gen(P(base), P(base), 4, 40, ctypes.byref(f), None, P(base), None) == B.SS_ERR_INVALID_ARG
    # exchange geometry and descriptors
    assert L.ss_exchange_bytes(0, 1) == 0
    assert L.ss_exchange_bytes(252, 8) == 4 * (2 * 252 * 8 + 8 * 8)
    assert L.ss_exchange_init(None, 4, 2, None) == B.SS_ERR_INVALID_ARG
    x = B.make_exchange(2, 0, [base, base + 1024], 4, 2)
    g = B.ExchangeGroup(0, 2, 0, 1)
    assert L.ss_exchange_publish(ctypes.byref(x), ctypes.byref(g), None, None) == B.SS_ERR_INVALID_ARG
    g0 = B.ExchangeGroup(3, 2, 0, 1)    # slot0 + count > max_tensors
    assert L.ss_exchange_publish(ctypes.byref(x), ctypes.byref(g0), P(base), None) == B.SS_ERR_INVALID_ARG
    g0 = B.ExchangeGroup(0, 2, 0, 0)    # epoch 0 is reserved (a zeroed buffer)
    assert L.ss_exchange_publish(ctypes.byref(x), ctypes.byref(g0), P(base), None) == B.SS_ERR_INVALID_ARG
    x9 = B.make_exchange(9, 0, [base] * 8, 4, 2)
    assert L.ss_exchange_publish(ctypes.byref(x9), ctypes.byref(g), P(base), None) == B.SS_ERR_INVALID_ARG
    ios = (B.TensorIO * 2)(io, io)
    gin = B.ExchangeGroup(0, 3, 0, 1)   # count differs from the call's
    assert L.ss_quantize_nvfp4_exchange(ios, 2, -8, 8, ctypes.byref(x), ctypes.byref(gin), None, None, 0, None,
                                        None, None) == B.SS_ERR_INVALID_ARG
    assert L.ss_ipc_handle(None, P(base)) == B.SS_ERR_INVALID_ARG
    assert L.ss_ipc_open(None, ctypes.byref(ctypes.c_void_p())) == B.SS_ERR_INVALID_ARG
