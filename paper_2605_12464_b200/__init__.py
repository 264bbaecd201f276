"""ScaleSearch NVFP4 quantization on B200 (arxiv 2605.12464), B200-native.

The compute path is libss.so (include/ss.h): hand-written sm_100a kernels for
the amax, search-quantize and dequantize steps.  This package is the thin
Python binding (argument marshalling only) plus the row-shard driver that
runs one process per GPU over torch.distributed/NCCL.
"""
from ._binding import (  # noqa: F401
    FLAG_NONFINITE,
    FLAG_RANGE,
    GMODES,
    SCALE_LAYOUTS,
    FORMATS,
    QuantOut,
    SSError,
    alloc_out,
    dequantize,
    device_status,
    lib,
    plan,
    quantize,
    quantize_batched,
    quantize_batched_next_amax,
    quantize_f32,
    quantize_gen,
    dequantize_gen,
    quantize_host,
    quantize_host_batched,
    quantize_simple,
    scale_bytes,
    status_string,
    tensor_amax,
    tensor_amax_batched,
)

__all__ = [
    "lib", "tensor_amax", "tensor_amax_batched", "quantize_batched", "quantize_batched_next_amax", "quantize_f32", "quantize_gen", "dequantize_gen",
    "alloc_out", "quantize", "quantize_simple", "dequantize", "quantize_host", "quantize_host_batched",
    "device_status", "scale_bytes", "plan", "SCALE_LAYOUTS", "FORMATS", "status_string", "SSError", "QuantOut", "GMODES",
]
