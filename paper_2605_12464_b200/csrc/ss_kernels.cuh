// ss_kernels.cuh — sm_100a device code for ScaleSearch NVFP4 quantization.
//
// Hot path = Algorithm 1 of arxiv 2605.12464 applied to
// every 16-element block, under the FP32 contract of include/ss.h (readings
// R1-R18 in DESIGN.md §3).  Not a contraction, so no tensor cores: the work is
// plain FP32 plus the Blackwell FP4/FP8 conversion instructions.
//
// Work decomposition.  The unit of scheduling is a WARP TASK
// of 32 consecutive NVFP4 blocks (1 KiB of bf16), one block per lane.  A
// launch covers a BATCH of up to kMaxTensors tensors whose tasks are numbered
// consecutively, so one persistent grid walks every tensor of a step with no
// per-tensor tail.  Each warp keeps kStages tasks in flight in shared memory:
// every lane stages its own 32-B block with two 16-B LDGSTS (cp.async) and
// reads back only its own bytes, so no barrier of any kind exists after the
// prologue.  (Per-warp 1-D TMA bulk copies were measured first: beyond ~64
// outstanding bulk operations per SM their throughput collapses to ~2.4 TB/s,
// tools/probes/bwprobe.cu; per-lane LDGSTS streams at the full 7.3 TB/s.)
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
#ifndef SS_AMAX_MODE
#define SS_AMAX_MODE 1   // 0: 32 KiB chunk per CTA iteration; 1: grid-stride, 4 loads in flight
#endif

namespace ss {

constexpr int kWarps = 8;                     // warps per CTA
constexpr int kThreads = 32 * kWarps;
constexpr int kBPL = SS_BPL;                  // NVFP4 blocks per lane per task
constexpr int kTaskBlocks = 32 * kBPL;        // NVFP4 blocks per warp task
constexpr int kTaskBytes = kTaskBlocks * 32;  // bf16 input bytes per task
constexpr int kStages = kBPL >= 4 ? 2 : 4 / kBPL;  // per-warp smem buffers (tasks in flight)
constexpr int kSegTasks = 4096;               // tasks per CTA of the error-sum kernel
constexpr int kCounters = 256;                // task counters of the dynamic scheduler
constexpr int kPruneFrom = 3;                 // exact pruning for offsets f <= -kPruneFrom
constexpr int kMaxTensors = 128;              // tensors per launch (kernel-parameter space)
constexpr int kAmaxVecs = 8;                  // 16-B vectors per thread per amax chunk
constexpr int kAmaxChunk = kThreads * kAmaxVecs;  // 16-B vectors per amax chunk (32 KiB)

constexpr uint32_t kOneSixthBits = 0x3E2AAAABu;  // RN(1/6) (Alg. 1 line 2; R8)
constexpr float kGlobalNumer = 2688.0f;          // 6 * 448: largest NVFP4 magnitude (R9)

// Block formats: value format VF
// (0 E2M1, 1 E2M3), scale format SF (0 UE4M3, 1 UE8M0, R19), block BS (16/32).
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

enum : uint32_t { kFlagNonFinite = 1u, kFlagRange = 2u };

// ---------------------------------------------------------------------------
// Small PTX wrappers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t pack2u(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
#ifndef SS_SCALAR_FP32
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
#else  // tuning variant: the same arithmetic as scalar FMUL / FFMA pairs
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  float a0, a1, b0, b1;
  unpack2(a, a0, a1);
  unpack2(b, b0, b1);
  return pack2(__fmul_rn(a0, b0), __fmul_rn(a1, b1));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  float a0, a1, b0, b1, c0, c1;
  unpack2(a, a0, a1);
  unpack2(b, b0, b1);
  unpack2(c, c0, c1);
  return pack2(__fmaf_rn(a0, b0, c0), __fmaf_rn(a1, b1, c1));
}
#endif
// E2M1 nibbles of (lo, hi) -> f16x2 (q_lo, q_hi).
__device__ __forceinline__ uint32_t e2m1_round_f16x2(float lo, float hi) {
  uint32_t h;
  asm("{\n\t.reg .b8 q;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 q, %2, %1;\n\t"
      "cvt.rn.f16x2.e2m1x2 %0, q;\n\t}"
      : "=r"(h) : "f"(lo), "f"(hi));
  return h;
}
// E2M3 codes of (lo, hi) -> f16x2 (q_lo, q_hi) (MXFP6 values).
__device__ __forceinline__ uint32_t e2m3_round_f16x2(float lo, float hi) {
  uint32_t h;
  asm("{\n\t.reg .b16 q;\n\t"
      "cvt.rn.satfinite.e2m3x2.f32 q, %2, %1;\n\t"
      "cvt.rn.f16x2.e2m3x2 %0, q;\n\t}"
      : "=r"(h) : "f"(lo), "f"(hi));
  return h;
}
// Two E2M3 codes of (lo, hi), one per byte (lo in the low byte).
__device__ __forceinline__ uint32_t e2m3_pack2(float lo, float hi) {
  uint16_t q;
  asm("cvt.rn.satfinite.e2m3x2.f32 %0, %2, %1;" : "=h"(q) : "f"(lo), "f"(hi));
  return q;
}
// UE8M0 code of v >= 0: the smallest power of two >= v, saturating (R19).
__device__ __forceinline__ uint32_t ue8m0_code(float v) {
  uint16_t h;
  asm("cvt.rp.satfinite.ue8m0x2.f32 %0, %1, %2;" : "=h"(h) : "f"(0.0f), "f"(v));
  return h & 0xFFu;
}
// 2^(c - 127) for a UE8M0 code c (c = 0 is the subnormal 2^-127).
__device__ __forceinline__ uint32_t ue8m0_bits(uint32_t c) { return c ? c << 23 : 0x00400000u; }

// 8 E2M1 nibbles of 8 floats packed into one word, element 0 in the low nibble.
__device__ __forceinline__ uint32_t e2m1_pack8(float v0, float v1, float v2, float v3,
                                               float v4, float v5, float v6, float v7) {
  uint32_t w;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
      : "=r"(w)
      : "f"(v0), "f"(v1), "f"(v2), "f"(v3), "f"(v4), "f"(v5), "f"(v6), "f"(v7));
  return w;
}
// d = y + q * negs  (q, negs f16; exact product, one rounding)
__device__ __forceinline__ float fhfma(uint16_t q, uint16_t negs, float y) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(q), "h"(negs), "f"(y));
  return d;
}
// UE4M3 code of v >= 0, RNE, satfinite (Alg. 1 line 2).
__device__ __forceinline__ uint32_t e4m3_code(float v) {
  uint16_t h;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(0.0f), "f"(v));
  return h & 0xFFu;
}
// E4M3 code -> f16 bits (exact) via the hardware unpack.
__device__ __forceinline__ uint16_t e4m3_to_f16(uint32_t code) {
  uint32_t h;
  asm("{\n\t.reg .b16 c;\n\tcvt.u16.u32 c, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, c;\n\t}"
      : "=r"(h) : "r"(code));
  return (uint16_t)(h & 0xFFFFu);
}
__device__ __forceinline__ float f16_to_f32(uint16_t h) {
  float f;
  asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
  return f;
}

// ---- shared-memory staging -------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Per-lane asynchronous 16-B global -> shared copies (LDGSTS), grouped.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// Candidate table.  Two halves of TabW = 127 + 2*Pad entries (Pad = the
// largest |f| of the kernel's window); entry i of a half stands for the
// unclamped candidate code k = i - Pad:
//   half 0 (used when c0 == 0): code = 0 for k <= 0 (the zero-scale candidate,
//            R3), else min(k, 126);
//   half 1 (c0 >= 1):           code = clamp(k, 1, 126).
// A block's candidates are base[f] with base = half + Pad + c0, so
// out-of-range offsets become duplicates of the nearest valid code, which
// never change the lexicographic (loss, code) minimum (R2, R4): no branches.
// Entry = {rho, rho, (-s as f16) | code << 16, 0} with rho = RN(1/s) (R7);
// code 0 has rho = 0 and -s = -0.
// ---------------------------------------------------------------------------
// UE8M0 (SF = 1): one half of 255 + 2*Pad entries, code = clamp(k, 0, 254),
// entry = {rho, rho, code << 16, bits(-s)} (every code is a scale, R19).
template <int Pad, int SF>
__device__ __forceinline__ void build_cand_table(uint4* tab) {
  if constexpr (SF == 1) {
    constexpr int TabW = 255 + 2 * Pad;
    for (int i = threadIdx.x; i < TabW; i += blockDim.x) {
      const int k = i - Pad;
      const uint32_t code = (uint32_t)(k < 0 ? 0 : (k > 254 ? 254 : k));
      const uint32_t rho = ue8m0_bits(254u - code);  // 2^(127 - c), exact
      tab[i] = make_uint4(rho, rho, code << 16, ue8m0_bits(code) ^ 0x80000000u);
    }
    return;
  }
  constexpr int TabW = 127 + 2 * Pad;
  for (int i = threadIdx.x; i < 2 * TabW; i += blockDim.x) {
    const int half = i / TabW;
    const int k = i - half * TabW - Pad;
    int code = half == 0 ? (k <= 0 ? 0 : k) : (k < 1 ? 1 : k);
    code = code > 126 ? 126 : code;
    uint4 e;
    if (code == 0) {
      e = make_uint4(0u, 0u, 0x8000u, 0u);
    } else {
      const uint16_t sh = e4m3_to_f16((uint32_t)code);
      const float rho = __frcp_rn(f16_to_f32(sh));  // IEEE RN(1/s), not MUFU (R7)
      e = make_uint4(__float_as_uint(rho), __float_as_uint(rho),
                     (uint32_t)(sh ^ 0x8000u) | ((uint32_t)code << 16), 0u);
    }
    tab[i] = e;
  }
}

// Global scale from the amax bit pattern (R9); flags non-finite / overflow.
__device__ __forceinline__ float global_scale(uint32_t ab, uint32_t* flags, bool report,
                                              float numer = kGlobalNumer) {
  if (ab >= 0x7F800000u) {  // NaN / Inf in the input (R14)
    if (report) atomicOr(flags, kFlagNonFinite);
    return 1.0f;
  }
  const float A = __uint_as_float(ab);
  if (A == 0.0f) return 1.0f;
  const float G = __fdiv_rn(numer, A);
  if (!isfinite(G)) {
    if (report) atomicOr(flags, kFlagRange);
    return 1.0f;
  }
  return G;
}

// Row of flat block b (b < 2^31) for nbr blocks per row: multiply-high by
// floor((2^32-1)/nbr) is exact or one short; one correction step.
__device__ __forceinline__ uint32_t div_rows(uint32_t b, uint32_t nbr, uint32_t magic) {
  uint32_t q = __umulhi(b, magic);
  if (b - q * nbr >= nbr) q++;
  return q;
}

// Byte offset of scale (row r, scale column j) in the tensor-core layout of
// block-scaled MMA (cuBLAS / CUTLASS Sm1xx "128x4" scale-factor atom,
// R15b): 512-B tiles of 128 rows x 4 scale columns, tiles row-band-major,
// inside a tile (r % 32) * 16 + ((r / 32) % 4) * 4 + j % 4.
__device__ __forceinline__ uint32_t swizzled_scale_offset(uint32_t r, uint32_t j, uint32_t nkt) {
  return ((r >> 7) * nkt + (j >> 2)) * 512u + (r & 31u) * 16u + ((r >> 5) & 3u) * 4u + (j & 3u);
}

// ---------------------------------------------------------------------------
// Batch descriptors (kernel parameters; __grid_constant__).
// ---------------------------------------------------------------------------
struct QTensor {
  const uint8_t* in;        // bf16 [nb][16]
  uint2* codes;             // [nb] 8 B
  uint8_t* scales;          // [nb]
  float2* err;              // nullable [nb]
  int8_t* offsets;          // nullable [nb]
  double* sums;             // nullable [2]
  float* g_out;             // nullable
  const uint32_t* amax;     // gmode 1: FP32 bits of the tensor amax
  const float* g_row;       // gmode 2: per-row global scales [rows]
  int64_t nb;               // NVFP4 blocks
  int64_t task0;            // first global task of this tensor
  int64_t seg0;             // first global segment (error-sum kernel CTA) of this tensor
  uint32_t nbr;             // blocks per row (cols / 16)
  uint32_t nbr_magic;       // floor((2^32 - 1) / nbr): row = div_rows(block)
  uint32_t nkt;             // swizzled layout: ceil(nbr / 4) scale tiles per 128-row band
  int swz;                  // scale layout: 0 linear [rows][nbr], 1 128x4 swizzled (R15b)
};

struct QuantBatch {
  int n;                    // tensors in this launch
  int fmin, fmax;           // window (runtime loop variant only)
  int gmode;                // 0: G = 1; 1: G from t[i].amax; 2: per-row G from t[i].g_row
  float g_numer;            // vmax * 448 (2688 for E2M1, 3360 for E2M3 values)
  int64_t ntasks;           // total tasks of the batch
  int64_t nsegs;            // total error-sum segments of the batch
  double2* part1;           // per task {sum best, sum base}   (when any sums wanted)
  double2* part2;           // per segment
  uint32_t* tick;           // per tensor, zero and self re-arming
  uint32_t* ctr;            // [kCounters + 1] task counters + done count, zero and self re-arming
  uint32_t* flags;
  unsigned long long* evals;  // SS_COUNT_EVALS builds: block-candidate evaluations executed
  QTensor t[kMaxTensors];
};

struct ATensor {
  const uint4* in;          // 16-B vectors
  int64_t nvec;             // whole 16-B vectors
  int ntail;                // trailing bf16 elements (< 8)
  int64_t chunk0;           // first global chunk
  uint32_t* out;            // amax slot (FP32 bits)
};

struct AmaxBatch {
  int n;
  int64_t nchunks;
  ATensor t[kMaxTensors];
};

// Index of the tensor holding task/chunk `k`, searching forward from `from`
// (warp-uniform; the tasks of one warp increase monotonically).
__device__ __forceinline__ int locate_task(const QuantBatch& p, int64_t k, int from) {
  int i = from;
  while (i + 1 < p.n && p.t[i + 1].task0 <= k) i++;
  return i;
}

// ---------------------------------------------------------------------------
// Amax kernel: unsigned max of |x| bf16 bit patterns (exact, NaN-propagating).
// One 32 KiB chunk per CTA iteration, 8 independent 16-B loads per thread.
// ---------------------------------------------------------------------------
// CTA b owns the contiguous global chunk range [b*per, (b+1)*per) (chunk =
// kAmaxChunk 16-B vectors of one tensor, kAmaxVecs independent coalesced loads
// per thread).  The running max is kept per thread while the tensor stays the
// same and reduced (warp redux + smem) into ONE atomicMax per (CTA, tensor).
__global__ void __launch_bounds__(kThreads) amax_kernel(const __grid_constant__ AmaxBatch p) {
  __shared__ uint32_t red[kWarps];
  const uint32_t M = 0x7FFF7FFFu;
  const int64_t per = (p.nchunks + gridDim.x - 1) / gridDim.x;
  const int64_t c_lo = (int64_t)blockIdx.x * per;
  const int64_t c_hi = min(p.nchunks, c_lo + per);
  if (c_lo >= c_hi) return;  // CTA-uniform
  int ti = 0;
  while (ti + 1 < p.n && p.t[ti + 1].chunk0 <= c_lo) ti++;
  uint32_t m = 0;
  for (int64_t ch = c_lo; ch < c_hi; ch++) {
    const ATensor& T = p.t[ti];
    const int64_t v0 = (ch - T.chunk0) * kAmaxChunk + threadIdx.x;
    uint4 v[kAmaxVecs];
#pragma unroll
    for (int k = 0; k < kAmaxVecs; k++) {
      const int64_t i = v0 + (int64_t)k * kThreads;
      v[k] = i < T.nvec ? __ldcs(T.in + i) : make_uint4(0, 0, 0, 0);
    }
    uint32_t mm = m;
#pragma unroll
    for (int k = 0; k < kAmaxVecs; k++)
      mm = __vmaxu2(mm, __vmaxu2(__vmaxu2(v[k].x & M, v[k].y & M), __vmaxu2(v[k].z & M, v[k].w & M)));
    m = mm;
    // trailing elements: handled by the chunk that holds the last vector
    if (T.ntail && (ch - T.chunk0) == (T.nvec / kAmaxChunk) && threadIdx.x < T.ntail) {
      const uint16_t* tail = reinterpret_cast<const uint16_t*>(T.in + T.nvec);
      m = __vmaxu2(m, (uint32_t)(tail[threadIdx.x] & 0x7FFFu));
    }
    const bool flush = ch + 1 == c_hi || (ti + 1 < p.n && p.t[ti + 1].chunk0 <= ch + 1);
    if (flush) {  // CTA-uniform
      uint32_t r = __reduce_max_sync(0xFFFFFFFFu, max(m & 0xFFFFu, m >> 16));
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps; w++) r = max(r, red[w]);
        r = max(r, red[0]);
        if (r) atomicMax(T.out, r << 16);  // bf16 bits -> FP32 bits (exact)
      }
      __syncthreads();
      m = 0;
      while (ti + 1 < p.n && p.t[ti + 1].chunk0 <= ch + 1) ti++;
    }
  }
}

// ---------------------------------------------------------------------------
// Error sums.  The quantize kernel stores one {sum best, sum base} partial per
// warp task (a fixed lane tree); sums_kernel then reduces each tensor's task
// partials in a fixed order: CTA k sums segment k (kSegTasks tasks) and the
// last CTA of a tensor (ticket counter) sums the tensor's segment partials.
// Deterministic for any grid of either kernel.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Fixed-order CTA sum of n double2 values at src (thread-strided, then tree).
__device__ __forceinline__ double2 cta_sum(const double2* src, int64_t n, double2* red) {
  double a = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const double2 v = __ldcg(src + i);
    a += v.x;
    c += v.y;
  }
  a = warp_sum(a);
  c = warp_sum(c);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(a, c);
  __syncthreads();
  double2 r = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int w = 0; w < kWarps; w++) {
      r.x += red[w].x;
      r.y += red[w].y;
    }
  return r;  // valid in thread 0
}

__global__ void __launch_bounds__(kThreads) sums_kernel(const __grid_constant__ QuantBatch p) {
  __shared__ double2 red[kWarps];
  __shared__ uint32_t last;
  int ti = 0;
  for (int64_t sg = blockIdx.x; sg < p.nsegs; sg += gridDim.x) {
    while (ti + 1 < p.n && p.t[ti + 1].seg0 <= sg) ti++;
    const QTensor& T = p.t[ti];
    if (!T.sums) continue;  // CTA-uniform
    const int64_t ntask = (T.nb + kTaskBlocks - 1) / kTaskBlocks;
    const int64_t nseg = (ntask + kSegTasks - 1) / kSegTasks;
    const int64_t k = sg - T.seg0;
    const int64_t t0 = k * kSegTasks;
    const double2 r = cta_sum(p.part1 + T.task0 + t0, min((int64_t)kSegTasks, ntask - t0), red);
    if (threadIdx.x == 0) {
      p.part2[sg] = r;
      __threadfence();
      last = atomicAdd(p.tick + ti, 1u) == (uint32_t)(nseg - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const double2 f = cta_sum(p.part2 + T.seg0, nseg, red);
      if (threadIdx.x == 0) {
        T.sums[0] = f.x;
        T.sums[1] = f.y;
        p.tick[ti] = 0u;  // re-arm
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Search-quantize kernel.
// ---------------------------------------------------------------------------

// Loss of one candidate (Alg. 1 lines 7-9) for the 16 values y (8 f32 pairs).
__device__ __forceinline__ float cand_loss(const uint64_t (&y2)[8], const float (&y)[16],
                                           const uint4 e) {
  const uint64_t rr = pack2u(e.x, e.y);
  const uint16_t negs = (uint16_t)(e.z & 0xFFFFu);
  uint64_t acc = 0;  // {even chain a, odd chain b}
#pragma unroll
  for (int k = 0; k < 8; k++) {
    float t0, t1;
    unpack2(fmul2(y2[k], rr), t0, t1);
    const uint32_t q = e2m1_round_f16x2(t0, t1);
    const float d0 = fhfma((uint16_t)(q & 0xFFFFu), negs, y[2 * k]);
    const float d1 = fhfma((uint16_t)(q >> 16), negs, y[2 * k + 1]);
    const uint64_t d = pack2(d0, d1);
    acc = ffma2(d, d, acc);
  }
  float a, b;
  unpack2(acc, a, b);
  return __fadd_rn(a, b);
}

// Losses of CN candidates with their pair loops interleaved (independent
// FFMA2 accumulation chains); each loss is computed exactly as cand_loss.
template <int CN>
__device__ __forceinline__ void cand_loss_n(const uint64_t (&y2)[8], const float (&y)[16],
                                            const uint4 (&e)[CN], float (&loss)[CN]) {
  uint64_t acc[CN];
#pragma unroll
  for (int c = 0; c < CN; c++) acc[c] = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
#pragma unroll
    for (int c = 0; c < CN; c++) {
      float t0, t1;
      unpack2(fmul2(y2[k], pack2u(e[c].x, e[c].y)), t0, t1);
      const uint32_t q = e2m1_round_f16x2(t0, t1);
      const uint16_t negs = (uint16_t)(e[c].z & 0xFFFFu);
      const float d0 = fhfma((uint16_t)(q & 0xFFFFu), negs, y[2 * k]);
      const float d1 = fhfma((uint16_t)(q >> 16), negs, y[2 * k + 1]);
      const uint64_t d = pack2(d0, d1);
      acc[c] = ffma2(d, d, acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < CN; c++) {
    float a, b;
    unpack2(acc[c], a, b);
    loss[c] = __fadd_rn(a, b);
  }
}

// Loss of one candidate for the 16 values of this lane in format FMT: the
// NVFP4 sequence, E2M3 rounding for VF = 1, and for UE8M0 scales (s outside
// f16) the residual as FFMA2 with q widened to f32.  A block of BS = 16 * 2^k
// elements spans 2^k lanes; their part losses are summed by an xor butterfly,
// which every lane evaluates as the same pairwise tree (R20; FADD commutes
// bit-exactly).
template <int FMT>
__device__ __forceinline__ float block_loss(const uint64_t (&y2)[8], const float (&y)[16],
                                            const uint4 e) {
  using F = Fmt<FMT>;
  float l;
  if constexpr (F::VF == 0 && F::SF == 0) {
    l = cand_loss(y2, y, e);
  } else {
    const uint64_t rr = pack2u(e.x, e.y);
    const uint16_t negs = (uint16_t)(e.z & 0xFFFFu);
    const uint64_t ns2 = pack2u(e.w, e.w);
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      float t0, t1;
      unpack2(fmul2(y2[k], rr), t0, t1);
      const uint32_t q = F::VF ? e2m3_round_f16x2(t0, t1) : e2m1_round_f16x2(t0, t1);
      uint64_t d;
      if constexpr (F::SF == 0) {
        d = pack2(fhfma((uint16_t)(q & 0xFFFFu), negs, y[2 * k]),
                  fhfma((uint16_t)(q >> 16), negs, y[2 * k + 1]));
      } else {
        const uint64_t qf = pack2(f16_to_f32((uint16_t)(q & 0xFFFFu)), f16_to_f32((uint16_t)(q >> 16)));
        d = ffma2(qf, ns2, y2[k]);
      }
      acc = ffma2(d, d, acc);
    }
    float a, b;
    unpack2(acc, a, b);
    l = __fadd_rn(a, b);
  }
#pragma unroll
  for (int o = 1; o < Fmt<FMT>::BS / 16; o <<= 1) l = __fadd_rn(l, __shfl_xor_sync(0xFFFFFFFFu, l, o));
  return l;
}

// Exact lower bound of a candidate's computed loss: RN(d^2) of the block's
// max-magnitude element (|y| = m), computed with the same instructions as its
// term of the loss.  Each FMA step adds a non-negative value and RN is
// monotone, so the computed loss >= RN(d_j^2) for every element j; a
// candidate whose bound exceeds the incumbent can never be selected, and
// skipping it changes no output bit.
//
// `sat` reports t = m * rho >= vmax: the max element then rounds to vmax for
// this and every smaller scale, and d = m - vmax * s >= 0 grows as s shrinks,
// so the bound only increases along the negative side from here on.
template <int FMT>
__device__ __forceinline__ float cand_lb(float m, const uint4 e, bool& sat) {
  using F = Fmt<FMT>;
  const float t = __fmul_rn(m, __uint_as_float(e.x));
  sat = t >= (F::VF ? 7.5f : 6.0f);
  const uint32_t q = F::VF ? e2m3_round_f16x2(t, t) : e2m1_round_f16x2(t, t);
  float d;
  if constexpr (F::SF == 0) {
    d = fhfma((uint16_t)(q & 0xFFFFu), (uint16_t)(e.z & 0xFFFFu), m);
  } else {
    d = __fmaf_rn(f16_to_f32((uint16_t)(q & 0xFFFFu)), __uint_as_float(e.w), m);
  }
  return __fmul_rn(d, d);
}

// Candidate order (equivalent to Alg. 1's ascending strict-< scan, R4): f = 0
// first (it is also err_base), then f = 1, 2, ... with strict "<" (ties keep
// the smaller code), then f = -1, -2, ... with "<=" (a tie moves to the
// smaller code; smaller codes always come later in this order).  Clamped
// duplicates carry the same code, so they never change the result.  The
// negative side runs last because the incumbent is then final or nearly so:
// a warp skips a negative candidate when no lane's cand_lb reaches it.
// SS_COUNT_EVALS (tools only): count the candidate evaluations a warp executes.
#ifdef SS_COUNT_EVALS
#define SS_COUNT(n) (n_evals += (n))
#else
#define SS_COUNT(n) ((void)0)
#endif

// Negative-side update with exact pruning (cand_lb, warp vote).
#ifndef SS_NO_PRUNE
// Used inside the negative-side loop: `break`s once every lane is pruned AND
// saturated (no further negative offset can win, cand_lb).
#define SS_TAKE_NEG(F)                                                   \
  {                                                                      \
    const uint4 e_ = base[F];                                            \
    bool sat_;                                                           \
    const bool prune_ = cand_lb<FMT>(m, e_, sat_) > best;                \
    if (__all_sync(0xFFFFFFFFu, prune_ && sat_)) break;                  \
    if (!__all_sync(0xFFFFFFFFu, prune_)) {                              \
      SS_COUNT(1);                                                       \
      const float l_ = block_loss<FMT>(y2, y, e_);                       \
      const bool t_ = l_ <= best;                                        \
      best = t_ ? l_ : best;                                             \
      bsel = t_ ? e_.z : bsel;                                           \
    }                                                                    \
  }
#else
#define SS_TAKE_NEG(F) SS_TAKE(F, <=)
#endif

// Runtime-window updates (scan order of R4, see above).
#define SS_TAKE(F, CMP)                                      \
  {                                                          \
    SS_COUNT(1);                                             \
    const uint4 e_ = base[F];                                \
    const float l_ = block_loss<FMT>(y2, y, e_);             \
    const bool t_ = l_ CMP best;                             \
    best = t_ ? l_ : best;                                   \
    bsel = t_ ? e_.z : bsel;                                 \
  }

// NEG/POS >= 0: compile-time window [-NEG, POS]; NEG < 0: runtime [fmin, fmax].
// RI: the batch needs each block's row (per-row G or the swizzled scale
// layout); without it those per-block steps are compiled out.  FMT: block
// format (Fmt<>); fixed windows (NEG >= 0) exist for NVFP4 only.  Units:
// `b`/`j` index 16-element HALF-blocks (one per lane); a 32-element block is
// the lane pair (2i, 2i + 1), whose even lane writes its scale, offset and
// errors.
template <int NEG, int POS, bool RI, int FMT>
__global__ void __launch_bounds__(kThreads, SS_MIN_BLOCKS) quant_kernel(const __grid_constant__ QuantBatch p) {
  using F = Fmt<FMT>;
  static_assert(FMT == kFmtNVFP4 || NEG < 0, "fixed windows are compiled for NVFP4 only");
  constexpr int Pad = NEG < 0 ? F::kMaxCode : (NEG > POS ? NEG : POS);
  constexpr int TabW = F::SF ? 255 + 2 * Pad : 127 + 2 * Pad;
  constexpr int kHalves = F::BS / 16;  // lanes per scale block
  __shared__ __align__(16) uint4 tab[F::SF ? TabW : 2 * TabW];
  __shared__ __align__(128) uint4 buf[kWarps][kStages][kTaskBytes / 16];

  build_cand_table<Pad, F::SF>(tab);
  __syncthreads();

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + w;

  const float kinv = __uint_as_float(F::kInvVmaxBits);  // RN(1 / vmax) (R8)
  // Stage s of this warp holds one task.  Lane l copies its own blocks
  // l, l+32, ... (2 x 16-B LDGSTS each) and later reads back only what it
  // copied, so no cross-lane sync is needed; one commit group per stage
  // (empty groups past the end keep the group count uniform).
  // Task indices are 32-bit: a batch holds < 2^31 tasks (2^41 elements).
  auto issue = [&](int tk, int ti, int s) {
    const QTensor& T = p.t[ti];
    const int b0 = (tk - (int)T.task0) * kTaskBlocks;
    const int nblk = (int)min((int64_t)kTaskBlocks, T.nb - b0);
    const uint8_t* src = T.in + (int64_t)b0 * 32;
#pragma unroll
    for (int u = 0; u < kBPL; u++) {
      const int j = u * 32 + lane;
      if (j < nblk) {
        cp_async16(&buf[w][s][2 * j], src + j * 32);
        cp_async16(&buf[w][s][2 * j + 1], src + j * 32 + 16);
      }
    }
  };
  auto gscale = [&](int ti, bool report) -> float {
    if (p.gmode != 1) return 1.0f;  // 0: G = 1; 2: per-row G, read per block
    return global_scale(__ldg(p.t[ti].amax), p.flags, report, p.g_numer);
  };
  // Dynamic scheduling: counter c hands out tasks c, c + kCounters, ... ; warp
  // gw draws from counter gw % kCounters, so warps the arbiter favours simply
  // take more tasks and every warp finishes at about the same time.  Each
  // warp's tasks increase, so the tensor lookup only moves forward.
  const int cidx = gw % kCounters;
  bool exhausted = false;
  const int ntasks = (int)p.ntasks;
  auto grab = [&]() -> int {
    if (exhausted) return -1;
    uint32_t idx = 0;
    if (lane == 0) idx = atomicAdd(p.ctr + cidx, 1u);
    idx = __shfl_sync(0xFFFFFFFFu, idx, 0);
    const int64_t t = cidx + (int64_t)idx * kCounters;
    if (t >= ntasks) {
      exhausted = true;
      return -1;
    }
    return t;
  };

  // prologue: kStages tasks in flight
  int q_task[kStages];
  int q_ti[kStages];
  int tj = 0;
#pragma unroll
  for (int k = 0; k < kStages; k++) {
    const int t = grab();
    if (t >= 0) {
      tj = locate_task(p, t, tj);
      issue(t, tj, k);
    }
    q_task[k] = t;
    q_ti[k] = tj;
    cp_async_commit();
  }
  int s = 0;
#ifdef SS_COUNT_EVALS
  unsigned long long n_evals = 0;  // per warp (all lanes count the same)
#endif
  // global scale of the current task's tensor, recomputed when the tensor changes
  int cur_ti = -1;
  float G = 1.0f;
  while (q_task[0] >= 0) {
    const int task = q_task[0];
    const int ti = q_ti[0];
    const QTensor& T = p.t[ti];
    if (ti != cur_ti) {  // warp-uniform
      cur_ti = ti;
      G = gscale(ti, task == (int)T.task0 && lane == 0);
    }
    const int b0 = (task - (int)T.task0) * kTaskBlocks;   // first block of the task
    const int nblk = (int)min((int64_t)kTaskBlocks, T.nb - b0);

    cp_async_wait<kStages - 1>();  // this lane's copies of stage s have landed
    int8_t* offsets = T.offsets ? T.offsets + b0 / kHalves : nullptr;
    float2* err = T.err ? T.err + b0 / kHalves : nullptr;
    double sb = 0.0, sc = 0.0;
    const uint64_t GG = pack2(G, G);

#pragma unroll 1
    for (int u = 0; u < kBPL; u++) {
      const int j = u * 32 + lane;          // half-block within the task
      const bool active = j < nblk;
      const bool writer = (lane & (kHalves - 1)) == 0;  // owns the scale block
      // scale-block index within the tensor; its row (per-row G, swizzled layout)
      const uint32_t sbk = (uint32_t)(b0 + min(j, nblk - 1)) / kHalves;
      uint32_t row = 0;
      uint64_t Gb = GG;
      if (RI && (T.g_row || T.swz)) {  // warp-uniform
        row = div_rows(sbk, T.nbr, T.nbr_magic);
        if (T.g_row) {
          const float gr = __ldg(T.g_row + row);
          Gb = pack2(gr, gr);
        }
      }
      // a1 + a3: bf16 -> f32 is exact; y = RN(x * G)
      const uint4 v0 = buf[w][s][2 * j], v1 = buf[w][s][2 * j + 1];
      const uint32_t wd[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      float y[16];
      uint64_t y2[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        y2[k] = fmul2(pack2u(wd[k] << 16, wd[k] & 0xFFFF0000u), Gb);
        unpack2(y2[k], y[2 * k], y[2 * k + 1]);
      }
      // a4: block max-abs scale code c0 (Alg. 1 lines 1-2)
      float m = 0.0f;
#pragma unroll
      for (int i = 0; i < 16; i++) m = fmaxf(m, fabsf(y[i]));
#pragma unroll
      for (int o = 1; o < kHalves; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
      const float v = __fmul_rn(m, kinv);
      const int c0 = F::SF ? (int)ue8m0_code(v) : (int)e4m3_code(v);
      const uint4* base = F::SF ? tab + Pad + c0 : tab + (c0 ? TabW : 0) + Pad + c0;

      // a5 + a6: candidate search (Alg. 1 lines 5-10)
      float best, loss0;
      uint32_t bsel;
      if constexpr (NEG >= 0) {
        // f = 0, 1, ..., POS in chunks of CI interleaved candidates (the
        // selection updates applied in scan order), then the negative side
        constexpr int NC = 1 + POS;
        constexpr int CI = SS_CILP < NC ? SS_CILP : NC;
#pragma unroll
        for (int i0 = 0; i0 < NC; i0 += CI) {
          uint4 e[CI];
          float l[CI];
#pragma unroll
          for (int c = 0; c < CI; c++) e[c] = base[i0 + c < NC ? i0 + c : NC - 1];
          cand_loss_n<CI>(y2, y, e, l);
          SS_COUNT(NC - i0 < CI ? NC - i0 : CI);
#pragma unroll
          for (int c = 0; c < CI; c++) {
            const int i = i0 + c;
            if (i >= NC) break;
            if (i == 0) {
              best = l[c];
              loss0 = l[c];  // err_base: the max-abs scale (f = 0)
              bsel = e[c].z;
            } else {
              const bool t_ = l[c] < best;
              best = t_ ? l[c] : best;
              bsel = t_ ? e[c].z : bsel;
            }
          }
        }
#pragma unroll
        for (int f = 1; f <= NEG; f++) {
          if (f < kPruneFrom) {  // near offsets almost never prune for a whole warp
            SS_TAKE(-f, <=)
          } else {
            SS_TAKE_NEG(-f)
          }
        }
      } else {
        best = block_loss<FMT>(y2, y, base[0]);
        SS_COUNT(1);
        loss0 = best;  // err_base: the max-abs scale (f = 0)
        bsel = base[0].z;
        // runtime window; skip offsets that are clamped duplicates for every lane
        const int lo = __reduce_min_sync(0xFFFFFFFFu, F::SF ? -c0 : (c0 ? 1 : 0) - c0);
        const int hi = __reduce_max_sync(0xFFFFFFFFu, F::kMaxCode - c0);
        const int fneg = max(p.fmin, lo), fpos = min(p.fmax, hi);
#pragma unroll 1
        for (int f = 1; f <= fpos; f++) SS_TAKE(f, <)
#pragma unroll 1
        for (int f = -1; f >= fneg; f--) {
          if (f > -kPruneFrom) {
            SS_TAKE(f, <=)
          } else {
            SS_TAKE_NEG(f)
          }
        }
      }

      // a7: emit the winner: codes of t = y * rho*, scale byte, offset, errors
      const uint32_t code = bsel >> 16;
      const float rs = __uint_as_float(
          (F::SF ? tab[Pad + code] : tab[(code ? TabW : 0) + Pad + code]).x);
      const uint64_t rr = pack2(rs, rs);
      float t[16];
#pragma unroll
      for (int k = 0; k < 8; k++) unpack2(fmul2(y2[k], rr), t[2 * k], t[2 * k + 1]);
      if (active) {
        const int64_t hb = b0 + j;  // half-block index within the tensor
        if constexpr (F::VF == 0) {
          uint2 cw;
          cw.x = e2m1_pack8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
          cw.y = e2m1_pack8(t[8], t[9], t[10], t[11], t[12], t[13], t[14], t[15]);
          __stcs(T.codes + hb, cw);
        } else {  // E2M3: one code per byte
          uint32_t cw[4];
#pragma unroll
          for (int k = 0; k < 4; k++)
            cw[k] = e2m3_pack2(t[4 * k], t[4 * k + 1]) | (e2m3_pack2(t[4 * k + 2], t[4 * k + 3]) << 16);
          __stcs(reinterpret_cast<uint4*>(T.codes) + hb, make_uint4(cw[0], cw[1], cw[2], cw[3]));
        }
        if (writer) {
          if (!RI || !T.swz) {
            T.scales[sbk] = (uint8_t)code;
          } else {
            T.scales[swizzled_scale_offset(row, sbk - row * T.nbr, T.nkt)] = (uint8_t)code;
          }
          const int jb = j / kHalves;  // scale block within the task
          if (offsets) offsets[jb] = (int8_t)((int)code - c0);
          if (err) __stcs(err + jb, make_float2(best, loss0));
          sb += (double)best;
          sc += (double)loss0;
        }
      }
    }
    {  // refill stage s with the next task drawn (always commit: uniform group count)
      const int t = grab();
      if (t >= 0) {
        tj = locate_task(p, t, tj);
        issue(t, tj, s);
      }
      cp_async_commit();
#pragma unroll
      for (int k = 0; k + 1 < kStages; k++) {
        q_task[k] = q_task[k + 1];
        q_ti[k] = q_ti[k + 1];
      }
      q_task[kStages - 1] = t;
      q_ti[kStages - 1] = tj;
    }
    if (T.sums) {  // per-task partial (fixed lane tree); reduced by sums_kernel
      sb = warp_sum(sb);
      sc = warp_sum(sc);
      if (lane == 0) p.part1[task] = make_double2(sb, sc);
    }
    if (T.g_out && b0 == 0 && lane == 0 && p.gmode != 2) *T.g_out = G;

    s = s + 1 == kStages ? 0 : s + 1;
  }
#ifdef SS_COUNT_EVALS
  if (lane == 0 && p.evals) atomicAdd(p.evals, n_evals * 32ull / (unsigned long long)kHalves);
#endif
  // the last warp of the grid to finish re-arms the counters for the next launch
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(p.ctr + kCounters, 1u) == gridDim.x * kWarps - 1) {
      for (int c = 0; c < kCounters; c++) p.ctr[c] = 0u;
      p.ctr[kCounters] = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// Per-row global scale (SS_GLOBAL_ROW; "after per-row scaling"):
// g_row[r] = RN(2688 / max_k |x_rk|), 1 for an all-zero row, flags as the
// per-tensor scale (R9, R14).  A warp task covers 32 / lpr rows with lpr
// lanes per row (a power of two <= the row's 16-B vector count, <= 32);
// lanes stride the row, a segmented xor-shuffle max finishes it.
// ---------------------------------------------------------------------------
struct RTensor {
  const uint4* in;          // [rows][rowvec] 16-B vectors
  float* g_row;             // [rows] output
  int64_t rows;
  int32_t rowvec;           // 16-B vectors per row (cols / 8)
  int32_t lpr;              // lanes per row
  int64_t task0;            // first global warp task
};

struct RowBatch {
  int n;
  int64_t ntasks;
  uint32_t* flags;
  float g_numer;
  RTensor t[kMaxTensors];
};

__global__ void __launch_bounds__(kThreads) rowscale_kernel(const __grid_constant__ RowBatch p) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * kWarps;
  int ti = 0;
  for (int64_t task = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); task < p.ntasks; task += W) {
    while (ti + 1 < p.n && p.t[ti + 1].task0 <= task) ti++;
    const RTensor& T = p.t[ti];
    const int lpr = T.lpr;
    const int64_t r = (task - T.task0) * (32 / lpr) + lane / lpr;
    const int sub = lane % lpr;
    uint32_t m = 0;
    if (r < T.rows) {
      const uint4* src = T.in + r * T.rowvec;
      const uint32_t M = 0x7FFF7FFFu;
      for (int v = sub; v < T.rowvec; v += lpr) {
        const uint4 a = __ldcs(src + v);
        m = __vmaxu2(m, __vmaxu2(__vmaxu2(a.x & M, a.y & M), __vmaxu2(a.z & M, a.w & M)));
      }
    }
    uint32_t mx = max(m & 0xFFFFu, m >> 16);
    for (int o = lpr >> 1; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (sub == 0 && r < T.rows) T.g_row[r] = global_scale(mx << 16, p.flags, true, p.g_numer);
  }
}

// ---------------------------------------------------------------------------
// Dequantize kernel: xhat = RNE_bf16(RN((q * s) / G)).
// ---------------------------------------------------------------------------
struct DequantParams {
  const uint8_t* codes;     // E2M1: 8 B per 16 elements; E2M3: 16 B per 16 elements
  const uint8_t* scales;
  int64_t nb;               // 16-element half-blocks
  const float* g;           // nullable: G = 1; per tensor [1] or per row [rows]
  int g_per_row;
  uint32_t nbr, nbr_magic, nkt;  // scale blocks per row
  int swz;                  // scale layout (0 linear, 1 swizzled)
  uint4* out;
};

// xhat = RNE_bf16(RN((q * s) / G)) per element, any format (FMT).
template <int FMT>
__global__ void __launch_bounds__(256) dequant_kernel(const __grid_constant__ DequantParams p) {
  using F = Fmt<FMT>;
  constexpr int kHalves = F::BS / 16;
  const float G0 = (p.g && !p.g_per_row) ? *p.g : 1.0f;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < p.nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t sbk = (uint32_t)(b / kHalves);
    float G = G0;
    uint8_t sc;
    if (p.g_per_row || p.swz) {
      const uint32_t r = div_rows(sbk, p.nbr, p.nbr_magic);
      if (p.g_per_row) G = p.g[r];
      sc = p.swz ? p.scales[swizzled_scale_offset(r, sbk - r * p.nbr, p.nkt)] : p.scales[sbk];
    } else {
      sc = p.scales[sbk];
    }
    const float s = F::SF ? __uint_as_float(ue8m0_bits(sc)) : f16_to_f32(e4m3_to_f16(sc));
    float q[16];
    if constexpr (F::VF == 0) {
      const uint2 cw = __ldcs(reinterpret_cast<const uint2*>(p.codes) + b);
      const uint32_t words[2] = {cw.x, cw.y};
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t h;
        asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
            "mov.b32 {b0, b1, b2, b3}, %1;\n\t"
            "cvt.rn.f16x2.e2m1x2 %0, b0;\n\t}"
            : "=r"(h) : "r"(words[k >> 2] >> (8 * (k & 3))));
        q[2 * k] = f16_to_f32((uint16_t)(h & 0xFFFFu));
        q[2 * k + 1] = f16_to_f32((uint16_t)(h >> 16));
      }
    } else {
      const uint4 cw = __ldcs(reinterpret_cast<const uint4*>(p.codes) + b);
      const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t h;
        asm("{\n\t.reg .b16 c;\n\tcvt.u16.u32 c, %1;\n\tcvt.rn.f16x2.e2m3x2 %0, c;\n\t}"
            : "=r"(h) : "r"(words[k >> 1] >> (16 * (k & 1))));
        q[2 * k] = f16_to_f32((uint16_t)(h & 0xFFFFu));
        q[2 * k + 1] = f16_to_f32((uint16_t)(h >> 16));
      }
    }
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const float x0 = __fdiv_rn(__fmul_rn(q[2 * k], s), G);
      const float x1 = __fdiv_rn(__fmul_rn(q[2 * k + 1], s), G);
      uint32_t r;
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x1), "f"(x0));
      o[k] = r;
    }
    __stcs(p.out + 2 * b, make_uint4(o[0], o[1], o[2], o[3]));
    __stcs(p.out + 2 * b + 1, make_uint4(o[4], o[5], o[6], o[7]));
  }
}

}  // namespace ss
