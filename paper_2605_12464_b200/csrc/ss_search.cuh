// ss_search.cuh — the candidate table, global scale, row/swizzle indexing, batch descriptors, and the per-candidate loss, bound and selection steps of Algorithm 1.
#pragma once
#include "ss_ptx.cuh"

namespace ss {

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
// UE4M3 candidate for unclamped code k: half 0 (c0 == 0) maps k <= 0 to the
// zero scale, half 1 clamps to [1, 126]; both clamp at 126.
__device__ __forceinline__ int clamp_code(int half, int k) {
  const int code = half == 0 ? (k <= 0 ? 0 : k) : (k < 1 ? 1 : k);
  return code > 126 ? 126 : code;
}
// {rho, rho, (-s as f16) | code << 16, 0} of UE4M3 code 0..126 (code 0: the zero scale)
__device__ __forceinline__ uint4 cand_entry(int code) {
  if (code == 0) return make_uint4(0u, 0u, 0x8000u, 0u);
  const uint16_t sh = e4m3_to_f16((uint32_t)code);
  const float rho = __frcp_rn(f16_to_f32(sh));  // IEEE RN(1/s), not MUFU (R7)
  return make_uint4(__float_as_uint(rho), __float_as_uint(rho),
                    (uint32_t)(sh ^ 0x8000u) | ((uint32_t)code << 16), 0u);
}

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
    tab[i] = cand_entry(clamp_code(half, i - half * TabW - Pad));
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
  int64_t task0;            // first global scheduling unit of this tensor
  int64_t seg0;             // first global segment (error-sum kernel CTA) of this tensor
  uint32_t nbr;             // blocks per row (cols / 16)
  uint32_t nbr_magic;       // floor((2^32 - 1) / nbr): row = div_rows(block)
  uint32_t nkt;             // swizzled layout: ceil(nbr / 4) scale tiles per 128-row band
  int swz;                  // scale layout: 0 linear [rows][nbr], 1 128x4 swizzled (R15b)
  // row-fused per-row G (gmode 2 with the row amax inside the quantize pass):
  // hpr > 0 marks it.  A row is cpr chunks of <= kTaskBlocks half-blocks; a
  // scheduling unit is cpu chunks of one row (upr units per row); G_r goes to
  // g_out[row].  hpr == 0: plain tensor, units = items of kTaskBlocks.
  // (16-bit: hpr <= 512, cpr <= 8; small fields keep the launch parameters small)
  int16_t hpr, cpr, upr, cpu;
  int32_t part0;            // first error-sum partial (one per work item) of this tensor
  int32_t npart;            // error-sum partials of this tensor
  // fused amax (AF launches): the search of this tensor waits until
  // QuantBatch::done[i] == na (0: G needs no in-launch amax)
  int32_t na;
  int32_t xslot;            // gmode 3: the tensor's slot in QuantBatch::xin
};

// A tensor whose amax the AF amax warps compute: units [a0, next a0) of
// kAmaxUnitVecs 16-B vectors, folded into *slot (atomicMax of FP32 bits) and,
// when done >= 0, counted into QuantBatch::done[done].
struct AmaxTask {
  const uint4* in;
  int64_t nvec;             // 16-B vectors (2 per 16-element block)
  uint32_t* slot;
  int32_t a0;
  int32_t done;
};

struct QuantBatch {
  int n;                    // tensors in this launch
  int fmin, fmax;           // window (runtime loop variant only)
  int gmode;                // 0: G = 1; 1: G from t[i].amax; 2: per-row G from t[i].g_row
  float g_numer;            // vmax * 448 (2688 for E2M1, 3360 for E2M3 values)
  int64_t ntasks;           // total scheduling units of the batch
  int32_t ipu;              // plain tensors: work items per scheduling unit (and per error-sum partial)
  int64_t nsegs;            // total error-sum segments of the batch
  double2* part1;           // per task {sum best, sum base}   (when any sums wanted)
  double2* part2;           // per segment
  uint32_t* tick;           // per tensor, zero and self re-arming
  uint32_t* ctr;            // [kCounters + 1] task counters + done count, zero and self re-arming
  uint32_t* flags;
  uint32_t* done;           // AF launches: [kMaxTensors] finished amax units per tensor, then the
                            // amax unit counter (zero, re-armed)
  int32_t namax;            // AF launches: amax units of the batch
  int32_t nam;              // AF launches: amax tasks (am[0..nam))
  // Trailing amax (AF launches of a pipelined per-tensor-G call, DESIGN.md
  // §4.2c): the NEXT launch's tensors are am[tr0..nam), cut into ntrail
  // units of kTrailVecs 16-B vectors numbered by AmaxTask::a0 from 0; the
  // search warp finishing scheduling unit u folds trail units
  // [u * tpu, u * tpu + tpu) into their tensors' slots.  Nobody waits on them
  // in this launch; the next launch reads the slots (stream order).
  int32_t tr0, ntrail, tpu;
  AmaxTask am[kMaxTensors];
  unsigned long long* evals;  // SS_COUNT_EVALS builds: block-candidate evaluations executed
  // Peer-memory amax exchange.  Consumer, gmode 3: G of
  // tensor i from max_r xin[xslot_i * kMaxPeers + r] once every rank's flag
  // xin_flag[r] >= xepoch_in (mod 2^32).  Producer: when the launch's xunits_out
  // next-group amax units are done (counted in done[kMaxTensors + 1]), the
  // finishing warp stores the xcount_out local amaxes (xlocal) into every
  // rank's buffer (xout[p] + j * kMaxPeers) and releases xout_flag[p] =
  // xepoch_out.
  int32_t xw;               // ranks
  uint32_t xepoch_in, xepoch_out;
  int32_t xcount_out, xunits_out;
  const uint32_t* xin;
  const uint32_t* xin_flag;
  const uint32_t* xlocal;
  uint32_t* xout[kMaxPeers];
  uint32_t* xout_flag[kMaxPeers];
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

// Per-row global scale of row `row` of a row-fused tensor, computed by one
// warp (identical in every lane): G_r = RN(numer / max_k |x_rk|) exactly as
// rowscale_kernel (R9b), from one coalesced pass over the row's 16-B vectors
// (8 loads in flight per lane).  The row stays in L2 for the quantize reads.
__device__ __forceinline__ float row_global_scale(const QTensor& T, uint32_t row, int lane,
                                                  uint32_t* flags, float numer) {
  const uint4* src = reinterpret_cast<const uint4*>(T.in) + (int64_t)row * T.hpr * 2;
  const int nv = T.hpr * 2;
  const uint32_t M = 0x7FFF7FFFu;
  uint32_t m = 0;
  int v = lane;
  for (; v + 224 < nv; v += 256) {  // 8 loads in flight per lane
    uint4 a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = __ldg(src + v + 32 * k);
#pragma unroll
    for (int k = 0; k < 8; k++)
      m = __vmaxu2(m, __vmaxu2(__vmaxu2(a[k].x & M, a[k].y & M), __vmaxu2(a[k].z & M, a[k].w & M)));
  }
  for (; v < nv; v += 32) {
    const uint4 a = __ldg(src + v);
    m = __vmaxu2(m, __vmaxu2(__vmaxu2(a.x & M, a.y & M), __vmaxu2(a.z & M, a.w & M)));
  }
  const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, max(m & 0xFFFFu, m >> 16));
  return global_scale(mx << 16, flags, lane == 0, numer);
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
      bidx = t_ ? (F) : bidx;                                            \
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
    bidx = t_ ? (F) : bidx;                                  \
  }

// NEG/POS >= 0: compile-time window [-NEG, POS]; NEG < 0: runtime [fmin, fmax].
// Sum of a double over the 32 lanes (fixed xor tree, identical in every lane).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

}  // namespace ss
