// ss_kernels.cuh — sm_100a device code for ScaleSearch NVFP4 quantization
// (umbrella header).
//
// Hot path = Algorithm 1 of arxiv 2605.12464 applied to
// every block of a bf16 tensor, under the FP32 contract of include/ss.h
// (readings R1-R20 in DESIGN.md §3).  Not a contraction, so no tensor cores:
// plain FP32 plus the Blackwell FP4/FP6/FP8 conversion instructions.
//
//   ss_common.cuh        tuning macros, launch constants, block-format traits
//   ss_ptx.cuh           PTX wrappers (f32x2 FMUL/FFMA, cvt e2m1/e2m3/e4m3/ue8m0,
//                        mixed-precision FHFMA, cp.async)
//   ss_search.cuh        candidate table, global scale, row / swizzle indexing,
//                        batch descriptors, per-candidate loss, exact lower
//                        bound and the selection steps
//   ss_fused_amax.cuh    the amax warps of the fused-amax quantize kernel (a2)
//   ss_quant_kernel.cuh  the search-quantize kernel (a1, a3-a7)
//   ss_aux_kernels.cuh   amax (a2), error sums, per-row scale, dequantize (a8)
//   ss_block.cuh         the one-thread block-search routine (include/ss_device.cuh)
//                        and the FP32-input kernel built on it
//
// Work decomposition: a WARP TASK is 64 consecutive
// 16-element blocks of one tensor, two per lane; a launch covers a batch of up
// to kMaxTensors tensors whose tasks warps draw dynamically from 256 atomic
// counters.  Each warp stages its next task in shared memory with per-lane
// 16-B cp.async (LDGSTS) — no barrier after the prologue.  Per-warp 1-D TMA
// bulk copies were measured first and collapse beyond ~64 outstanding
// operations per SM (tools/probes/bwprobe.cu).
//
// Inner loop per PAIR of elements and candidate (3 issue slots per
// element-candidate; the candidate's {rho, rho, -s | code<<16} comes from one
// LDS.128 of a padded, pre-clamped candidate table):
//   FMUL2  t = y * rho                     (mul.rn.f32x2)
//   F2FP   E2M1 pack of (t0, t1)           (cvt.rn.satfinite.e2m1x2.f32)
//   F2FP   unpack to f16x2 (q0, q1)        (cvt.rn.f16x2.e2m1x2)
//   FHFMA  d0 = y0 + q0 * (-s)             (fma.rn.f32.f16; q*s exact, one rounding)
//   FHFMA  d1 = y1 + q1 * (-s)
//   FFMA2  {a, b} += {d0^2, d1^2}          (fma.rn.f32x2: the even / odd chains of R12)
// Negative offsets f <= -3 are first tested against an exact lower bound
// and skipped by the whole warp when no lane can win (bit-identical outputs).
#pragma once
#include "ss_common.cuh"
#include "ss_ptx.cuh"
#include "ss_search.cuh"
#include "ss_quant_kernel.cuh"
#include "ss_aux_kernels.cuh"
#include "ss_block.cuh"
#include "ss_gen_kernel.cuh"
