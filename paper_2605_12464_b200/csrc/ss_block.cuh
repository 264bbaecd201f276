// ss_block.cuh — Algorithm 1 (NVFP4 Scale Search) for ONE
// 16-element block held in registers by ONE thread: the block-search device
// routine a fused kernel reuses (e.g. quantizing attention's P tile, P:313,
// P:538-539).  Public entry: include/ss_device.cuh.
//
// Same FP32 contract as quant_kernel (R3-R12), hence bit-identical results
// for the same y: c0 from RN(max|y| * RN(1/6)) (R8); candidates
// c = clamp(c0 + f) with the zero scale for c0 = 0 (R2, R3); t = RN(y * RN(1/s))
// (R7); E2M1 RNE (R10, R11); d = RN(y - q s); even/odd FMA chains, RN(a + b)
// (R12); lexicographic (loss, code) minimum (R4).  Differences from the
// kernel's inner loop, none of which changes a result bit: candidate
// entries are computed in registers (no shared table), and negative offsets
// are pruned per thread with the same exact bound (cand_lb), so the routine
// has no warp collectives and may be called from divergent code.
#pragma once
#include "ss_search.cuh"

namespace ss {

struct Nvfp4Block {
  uint2 codes;      // 16 E2M1 nibbles, element 2j in the low nibble of byte j (R15)
  uint32_t scale;   // UE4M3 code c* (0..126)
  int offset;       // f* = c* - c0 (R5)
  float err_best;   // loss of c* (y units, R13)
  float err_base;   // loss of the max-abs scale c0 (f = 0)
};

// Search over [fmin, fmax] (fmin <= 0 <= fmax; |f| <= 126).  NEG/POS >= 0
// fix the window at compile time (loops unrolled), NEG < 0 takes it at run time.
template <int NEG, int POS>
__device__ __forceinline__ Nvfp4Block search_nvfp4_block(const float (&y)[16], int fmin = -NEG,
                                                         int fmax = POS) {
  if constexpr (NEG >= 0) {
    fmin = -NEG;
    fmax = POS;
  }
  uint64_t y2[8];
#pragma unroll
  for (int k = 0; k < 8; k++) y2[k] = pack2(y[2 * k], y[2 * k + 1]);
  float m = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; i++) m = fmaxf(m, fabsf(y[i]));
  const int c0 = (int)e4m3_code(__fmul_rn(m, __uint_as_float(kOneSixthBits)));
  const int half = c0 ? 1 : 0;

  const uint4 e0 = cand_entry(clamp_code(half, c0));
  float best = cand_loss(y2, y, e0);
  const float loss0 = best;
  uint32_t bsel = e0.z;
  const int hi = min(fmax, 126 - c0);         // beyond: clamped duplicates of code 126
  const int lo = max(fmin, (c0 ? 1 : 0) - c0);  // below: duplicates of code 1 (or 0)
  auto take_pos = [&](int f) {
    const uint4 e = cand_entry(clamp_code(half, c0 + f));
    const float l = cand_loss(y2, y, e);
    if (l < best) {  // ties keep the smaller code (R4)
      best = l;
      bsel = e.z;
    }
  };
  // false once no further negative offset can win (pruned and saturated)
  auto take_neg = [&](int f) -> bool {
    const uint4 e = cand_entry(clamp_code(half, c0 - f));
    if (f >= kPruneFrom) {  // exact bound (cand_lb): skip, or stop once saturated
      bool sat;
      if (cand_lb<kFmtNVFP4>(m, e, sat) > best) return !sat;
    }
    const float l = cand_loss(y2, y, e);
    if (l <= best) {  // a tie moves to the smaller code (R4)
      best = l;
      bsel = e.z;
    }
    return true;
  };
  if constexpr (NEG >= 0) {
#pragma unroll
    for (int f = 1; f <= POS; f++)
      if (f <= hi) take_pos(f);
#pragma unroll
    for (int f = 1; f <= NEG; f++)
      if (-f < lo || !take_neg(f)) break;
  } else {
#pragma unroll 1
    for (int f = 1; f <= hi; f++) take_pos(f);
#pragma unroll 1
    for (int f = 1; -f >= lo; f++)
      if (!take_neg(f)) break;
  }

  Nvfp4Block r;
  r.scale = bsel >> 16;
  r.offset = (int)r.scale - c0;
  r.err_best = best;
  r.err_base = loss0;
  const float rs = __uint_as_float(cand_entry((int)r.scale).x);
  const uint64_t rr = pack2(rs, rs);
  float t[16];
#pragma unroll
  for (int k = 0; k < 8; k++) unpack2(fmul2(y2[k], rr), t[2 * k], t[2 * k + 1]);
  r.codes.x = e2m1_pack8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
  r.codes.y = e2m1_pack8(t[8], t[9], t[10], t[11], t[12], t[13], t[14], t[15]);
  return r;
}

// ---------------------------------------------------------------------------
// FP32-input quantize kernel built on the routine (ss_quantize_nvfp4_f32):
// one thread per block, grid-stride; y = RN(x * G) with G given on the device
// (attention quantizes P with a fixed global scale).  Non-finite inputs set
// the sticky flag (R14) and are otherwise unchecked.
// ---------------------------------------------------------------------------
struct F32Params {
  const float4* in;       // [nb][4] float4
  int64_t nb;
  int fmin, fmax;
  const float* g;         // nullable: G = 1
  uint2* codes;
  uint8_t* scales;
  float2* err;            // nullable
  int8_t* offsets;        // nullable
  uint32_t* flags;
};

template <int NEG, int POS>
__global__ void __launch_bounds__(256) quant_f32_kernel(const __grid_constant__ F32Params p) {
  const float G = p.g ? *p.g : 1.0f;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < p.nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    float y[16];
    uint32_t nonfinite = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const float4 v = __ldcs(p.in + 4 * b + k);
      const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        nonfinite |= (__float_as_uint(xs[j]) & 0x7F800000u) == 0x7F800000u;
        y[4 * k + j] = __fmul_rn(xs[j], G);
      }
    }
    if (nonfinite) atomicOr(p.flags, kFlagNonFinite);
    const Nvfp4Block r = search_nvfp4_block<NEG, POS>(y, p.fmin, p.fmax);
    __stcs(p.codes + b, r.codes);
    p.scales[b] = (uint8_t)r.scale;
    if (p.err) __stcs(p.err + b, make_float2(r.err_best, r.err_base));
    if (p.offsets) p.offsets[b] = (int8_t)r.offset;
  }
}

// ---------------------------------------------------------------------------
// Small-tensor bf16 kernel (quantize_core picks it for one NVFP4 tensor of at
// most kSmallMaxBlocks blocks, linear scales, G per tensor or 1): one thread
// per block through the same routine, so a small tensor spreads over every
// resident thread (48 registers) instead of 2 blocks per lane of the
// persistent grid, and no candidate table is built.  Outputs equal
// quant_kernel's bit for bit; the FP64 error sums are reduced per 256-block
// chunk (fixed tree) and then by sums_kernel.
// ---------------------------------------------------------------------------
struct SmallParams {
  const uint4* in;        // [nb][2] uint4 (16 bf16)
  int64_t nb;
  int fmin, fmax;
  int gmode;              // 0: G = 1; 1: G from *amax
  const uint32_t* amax;
  float g_numer;
  uint2* codes;
  uint8_t* scales;
  float2* err;            // nullable
  int8_t* offsets;        // nullable
  float* g_out;           // nullable
  double2* part1;         // nullable: per 256-block chunk {sum best, sum base}
  uint32_t* flags;
};

template <int NEG, int POS>
__global__ void __launch_bounds__(256) quant_small_kernel(const __grid_constant__ SmallParams p) {
  __shared__ double2 red[8];
  pdl_wait();  // the amax grid (PDL predecessor) has completed
  pdl_launch_dependents();
  const float G = p.gmode == 1 ? global_scale(*p.amax, p.flags, blockIdx.x == 0 && threadIdx.x == 0, p.g_numer)
                               : 1.0f;
  if (p.g_out && blockIdx.x == 0 && threadIdx.x == 0) *p.g_out = G;
  const uint64_t GG = pack2(G, G);
  for (int64_t c = blockIdx.x; c * 256 < p.nb; c += gridDim.x) {  // CTA-uniform chunks of 256 blocks
    const int64_t b = c * 256 + threadIdx.x;
    double sb = 0.0, sc = 0.0;
    if (b < p.nb) {
      const uint4 v0 = __ldcs(p.in + 2 * b), v1 = __ldcs(p.in + 2 * b + 1);
      const uint32_t wd[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      float y[16];
#pragma unroll
      for (int k = 0; k < 8; k++)  // a1 + a3: exact bf16 -> f32, y = RN(x * G)
        unpack2(fmul2(pack2u(wd[k] << 16, wd[k] & 0xFFFF0000u), GG), y[2 * k], y[2 * k + 1]);
      const Nvfp4Block r = search_nvfp4_block<NEG, POS>(y, p.fmin, p.fmax);
      __stcs(p.codes + b, r.codes);
      p.scales[b] = (uint8_t)r.scale;
      if (p.err) __stcs(p.err + b, make_float2(r.err_best, r.err_base));
      if (p.offsets) p.offsets[b] = (int8_t)r.offset;
      sb = r.err_best;
      sc = r.err_base;
    }
    if (p.part1) {  // fixed-order CTA tree: lanes, then warps 0..7
      sb = warp_sum(sb);
      sc = warp_sum(sc);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(sb, sc);
      __syncthreads();
      if (threadIdx.x == 0) {
        double2 t = red[0];
        for (int w = 1; w < 8; w++) {
          t.x += red[w].x;
          t.y += red[w].y;
        }
        p.part1[c] = t;
      }
      __syncthreads();
    }
  }
}

}  // namespace ss
