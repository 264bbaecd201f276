/* ss_device.cuh — device-side API of the ScaleSearch library (sm_100a).
 *
 * The block-search routine of Algorithm 1 ("NVFP4 Scale Search", arxiv
 * 2605.12464, §4) for one 16-element block that a
 * thread holds in registers, for kernels that quantize their own FP32 data
 * in place (the paper reuses the search inside FP4 attention to quantize P,
 * P:313).  Header-only; include it from a .cu compiled with
 *   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17
 *
 *   ss::Nvfp4Block r = ss::search_nvfp4_block<8, 8>(y);      // window [-8, 8]
 *   ss::Nvfp4Block r = ss::search_nvfp4_block<-1, -1>(y, fmin, fmax);  // run time
 *
 * y[16]: the block multiplied by the caller's global scale, y = RN(x * G)
 *        (G = RN(2688 / amax) for per-tensor scaling, R9; G = 1 for none).
 * Result: packed E2M1 nibbles (element 2j in the low nibble of byte j), the
 *        UE4M3 scale code c* (0..126), f* = c* - c0, the loss of c* and of
 *        the max-abs scale c0, in y units.
 * Contract: the FP32 arithmetic of include/ss.h (readings R3-R12 of
 *        DESIGN.md §3), so for the same y the result is bit-identical to
 *        ss_quantize_nvfp4* (tests/test_device_routine_gpu.py).
 * Thread-level: no shared memory, no barriers, no warp collectives; safe in
 *        divergent code.  Non-finite y give undefined codes (the caller's
 *        amax should have caught them, R14).
 * Cost: about 3 issue slots per element and candidate (FMUL2, F2FP pack and
 *        unpack, 2 FHFMA, FFMA2 per pair), plus an IEEE reciprocal per
 *        candidate; negative offsets f <= -3 are skipped by an exact bound.
 */
#pragma once
#include "../paper_2605_12464_b200/csrc/ss_block.cuh"
