"""CPU oracle for ScaleSearch NVFP4 quantization (arxiv 2605.12464, Algorithm 1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2605_12464_b200`` never imports it and
shares no code with it.

The arithmetic lives in plain C (``ss_oracle.c``); this module only builds the
shared library with gcc and marshals numpy arrays through ctypes.
"""
from .oracle import (  # noqa: F401
    build,
    lib,
    e2m1_value,
    e2m1_encode,
    e4m3_value,
    e4m3_encode,
    search_block,
    tensor_amax,
    global_scale,
    quantize,
    dequantize,
    FORMATS,
    e2m3_value,
    e2m3_encode,
    ue8m0_value,
    ue8m0_encode,
    quantize_fmt,
    dequantize_fmt,
    OracleError,
    gen_value,
    gen_encode,
    gen_scale_value,
    gen_scale_encode,
    gen_numer,
    search_block_gen,
    quantize_gen,
    dequantize_gen,
)
