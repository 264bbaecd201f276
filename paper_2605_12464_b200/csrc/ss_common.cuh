// ss_common.cuh — tuning macros, launch constants and block-format traits.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef SS_MIN_BLOCKS
#define SS_MIN_BLOCKS 4
#endif
#ifndef SS_BPL
#define SS_BPL 2         // NVFP4 blocks per lane per warp task
#endif
#ifndef SS_CILP
#define SS_CILP 2        // candidates whose loss loops are interleaved (fixed windows)
#endif
namespace ss {

constexpr int kWarps = 8;                     // warps per CTA
constexpr int kThreads = 32 * kWarps;
constexpr int kBPL = SS_BPL;                  // 16-element blocks per lane per task
constexpr int kTaskBlocks = 32 * kBPL;        // NVFP4 blocks per warp task
constexpr int kTaskBytes = kTaskBlocks * 32;  // bf16 input bytes per task
constexpr int kStages = kBPL >= 4 ? 2 : 4 / kBPL;  // per-warp smem buffers (tasks in flight)
#ifndef SS_SEG_TASKS
#define SS_SEG_TASKS 512  // C1 call 58.5 -> 56.3 us, C3 -2 % (4096 before; profiles/r02/c1ab_seg.md)
#endif
constexpr int kSegTasks = SS_SEG_TASKS;       // partials per CTA of the error-sum kernel
constexpr int kCounters = 256;                // task counters of the dynamic scheduler
#ifndef SS_PRUNE_FROM
#define SS_PRUNE_FROM 3
#endif
constexpr int kPruneFrom = SS_PRUNE_FROM;     // exact pruning for offsets f <= -kPruneFrom
constexpr int kMaxTensors = 128;              // tensors per launch (kernel-parameter space)
constexpr int kAmaxVecs = 8;                  // 16-B vectors per thread per amax chunk
constexpr int kAmaxChunk = kThreads * kAmaxVecs;  // 16-B vectors per amax chunk (32 KiB)
#ifndef SS_AMAX_PDL_TRIGGER
// 1: the amax / row-scale grids let the quantize grid launch early (PDL
// trigger).  Measured slower (C3 r = 8: 339 vs 313 us per amax + quantize call),
// so the quantize grid launches when they complete; its own PDL launch still
// hides the launch gap (C1 r = 8 quantize: 52 -> 47 us).
#define SS_AMAX_PDL_TRIGGER 0
#endif
#ifndef SS_AMAX_WARPS
#define SS_AMAX_WARPS 2  // fused amax: 1 -> +0.8 %, 2 -> +4.6 %, 3 slower (C2 step, r = 8)
#endif

// fused amax (quant_kernel<..., AF>): warps per CTA that start as amax warps,
// and the 16-B vectors of one amax unit (32 KiB)
constexpr int kAmaxWarps = SS_AMAX_WARPS;
#ifndef SS_AMAX_UNIT
#define SS_AMAX_UNIT 2048
#endif
#ifndef SS_AMAXW_VECS
#define SS_AMAXW_VECS 8
#endif
constexpr int kAmaxUnitVecs = SS_AMAX_UNIT;    // 16-B vectors per amax unit (32 KiB)
constexpr int kAmaxWarpVecs = SS_AMAXW_VECS;  // 16-B loads in flight per lane of an amax warp
constexpr int kTrailVecs = 256;               // 16-B vectors per trailing-amax unit (4 KiB, 8 per lane)


constexpr uint32_t kOneSixthBits = 0x3E2AAAABu;  // RN(1/6) (Alg. 1 line 2; R8)
constexpr float kGlobalNumer = 2688.0f;          // 6 * 448: largest NVFP4 magnitude (R9)

// Block formats: value format VF
// (0 E2M1, 1 E2M3), scale format SF (0 UE4M3, 1 UE8M0, R19), block BS (16..256).
// Formats 4-7: NVFP4 values and scales on 32..256-element blocks (the
// block-size study of fig:block_size).
enum : int {
  kFmtNVFP4 = 0, kFmtMXFP4 = 1, kFmtMXFP6E2M3 = 2, kFmtNVFP6E2M3 = 3,
  kFmtNVFP4B32 = 4, kFmtNVFP4B64 = 5, kFmtNVFP4B128 = 6, kFmtNVFP4B256 = 7
};
template <int FMT>
struct Fmt {
  static constexpr int VF = (FMT == kFmtMXFP6E2M3 || FMT == kFmtNVFP6E2M3) ? 1 : 0;
  static constexpr int SF = (FMT == kFmtMXFP4 || FMT == kFmtMXFP6E2M3) ? 1 : 0;
  static constexpr int BS = FMT >= kFmtNVFP4B32 ? (32 << (FMT - kFmtNVFP4B32)) : (SF ? 32 : 16);
  static constexpr uint32_t kInvVmaxBits = VF ? 0x3E088889u : kOneSixthBits;  // RN(1/7.5), RN(1/6)
  static constexpr int kMaxCode = SF ? 254 : 126;
};
__host__ __device__ constexpr float global_numer(int vf) { return vf ? 3360.0f : kGlobalNumer; }

enum : uint32_t { kFlagNonFinite = 1u, kFlagRange = 2u, kFlagAmaxTimeout = 4u, kFlagExchangeTimeout = 8u };
constexpr int kMaxPeers = 8;  // ranks of a peer-memory amax exchange (one NVLink domain)

}  // namespace ss
