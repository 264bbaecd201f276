// ss_kernels.cuh — sm_100a device code for ScaleSearch NVFP4 quantization.
//
// Hot path = Algorithm 1 of arxiv 2605.12464 applied to
// every 16-element block, under the FP32 contract of include/ss.h (readings
// R1-R15 in DESIGN.md §3).  Not a contraction, so no tensor cores: the work is
// plain FP32 + the Blackwell FP4/FP8 conversion instructions, one NVFP4 block
// per thread, the candidate loop unrolled in registers.
//
// Per element and candidate the inner loop issues, per PAIR of elements:
//   FMUL2  t = y * rho                     (mul.rn.f32x2, scalar-broadcast rho)
//   F2FP   E2M1 pack of (t0, t1)           (cvt.rn.satfinite.e2m1x2.f32)
//   F2FP   unpack to f16x2 (q0, q1)        (cvt.rn.f16x2.e2m1x2)
//   FHFMA  d0 = y0 + q0 * (-s)             (fma.rn.f32.f16; q*s exact, one rounding)
//   FHFMA  d1 = y1 + q1 * (-s)
//   FFMA2  {a, b} += {d0^2, d1^2}          (fma.rn.f32x2: the even / odd chains of R12)
// = 3 issue slots per element-candidate.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ss {

constexpr int kThreads = 256;           // threads per CTA = NVFP4 blocks per CTA tile
constexpr uint32_t kOneSixthBits = 0x3E2AAAABu;  // RN(1/6) (Alg. 1 line 2; R8)
constexpr float kGlobalNumer = 2688.0f;  // 6 * 448: largest NVFP4 magnitude (R9)

enum : uint32_t { kFlagNonFinite = 1u, kFlagRange = 2u };

// ---------------------------------------------------------------------------
// Small PTX wrappers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fmul2_bcast(uint64_t a, float b) {
  uint64_t r, bb = pack2(b, b);
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(bb));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// E2M1 nibbles of (lo, hi) -> f16x2 (q_lo, q_hi); also returns the packed byte.
__device__ __forceinline__ uint32_t e2m1_round_f16x2(float lo, float hi) {
  uint32_t h;
  asm("{\n\t.reg .b8 q;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 q, %2, %1;\n\t"
      "cvt.rn.f16x2.e2m1x2 %0, q;\n\t}"
      : "=r"(h) : "f"(lo), "f"(hi));
  return h;
}
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

// ---------------------------------------------------------------------------
// Candidate table: for every UE4M3 code c, rho = RN(1/s_c) and -s_c as f16.
// Entry 0 is the zero-scale candidate (rho = 0, s = 0; R3); entry 127 (NaN)
// is never selected (masked as invalid).
// ---------------------------------------------------------------------------
struct __align__(8) Cand {
  float rho;
  uint32_t negs;  // f16 bits of -s in the low half
};

__device__ __forceinline__ void build_cand_table(Cand* tab) {
  for (int c = threadIdx.x; c < 128; c += blockDim.x) {
    Cand e;
    if (c == 0 || c == 127) {
      e.rho = 0.0f;
      e.negs = 0x8000u;  // -0
    } else {
      uint16_t sh = e4m3_to_f16((uint32_t)c);
      float s = f16_to_f32(sh);
      e.rho = __frcp_rn(s);          // RN(1/s) (R7), IEEE reciprocal
      e.negs = (uint32_t)(sh ^ 0x8000u);
    }
    tab[c] = e;
  }
}

// Global scale from the amax bit pattern (R9); flags non-finite / overflow.
__device__ __forceinline__ float global_scale(int gmode, const uint32_t* amax_bits,
                                              uint32_t* flags, bool report) {
  if (gmode == 0) return 1.0f;
  uint32_t ab = *amax_bits;
  if (ab >= 0x7F800000u) {  // NaN / Inf in the input
    if (report) atomicOr(flags, kFlagNonFinite);
    return 1.0f;
  }
  float A = __uint_as_float(ab);
  if (A == 0.0f) return 1.0f;
  float G = __fdiv_rn(kGlobalNumer, A);
  if (!isfinite(G)) {
    if (report) atomicOr(flags, kFlagRange);
    return 1.0f;
  }
  return G;
}

// ---------------------------------------------------------------------------
// Amax kernel: unsigned max of |x| bf16 bit patterns (exact, NaN-propagating).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t umax2(uint32_t a, uint32_t b) {
  return __vmaxu2(a, b);  // per-halfword unsigned max
}

__global__ void __launch_bounds__(256) amax_kernel(const uint4* __restrict__ in, int64_t n16,
                                                   const uint16_t* __restrict__ tail, int n_tail,
                                                   uint32_t* __restrict__ out) {
  uint32_t m = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // 4 independent 16-B loads in flight per thread per iteration
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = in[i], b = in[i + stride];  // default policy: keep in L2 for the quantize pass
    uint4 c = in[i + 2 * stride], d = in[i + 3 * stride];
    const uint32_t M = 0x7FFF7FFFu;
    uint32_t x0 = umax2(umax2(a.x & M, a.y & M), umax2(a.z & M, a.w & M));
    uint32_t x1 = umax2(umax2(b.x & M, b.y & M), umax2(b.z & M, b.w & M));
    uint32_t x2 = umax2(umax2(c.x & M, c.y & M), umax2(c.z & M, c.w & M));
    uint32_t x3 = umax2(umax2(d.x & M, d.y & M), umax2(d.z & M, d.w & M));
    m = umax2(m, umax2(umax2(x0, x1), umax2(x2, x3)));
  }
  for (; i < n16; i += stride) {
    uint4 a = in[i];
    const uint32_t M = 0x7FFF7FFFu;
    m = umax2(m, umax2(umax2(a.x & M, a.y & M), umax2(a.z & M, a.w & M)));
  }
  uint32_t r = max(m & 0xFFFFu, m >> 16);
  if (blockIdx.x == 0 && threadIdx.x < n_tail) r = max(r, (uint32_t)(tail[threadIdx.x] & 0x7FFFu));
  for (int o = 16; o > 0; o >>= 1) r = max(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
  __shared__ uint32_t red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    for (int o = 16; o > 0; o >>= 1) r = max(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
    if (threadIdx.x == 0) atomicMax(out, r << 16);  // bf16 bits -> FP32 bits (exact)
  }
}

// ---------------------------------------------------------------------------
// Search-quantize kernel.
// ---------------------------------------------------------------------------
struct QuantParams {
  const uint4* in;          // bf16 blocks, 2 x uint4 per NVFP4 block
  int64_t nb;               // number of 16-element blocks
  int fmin, fmax;           // runtime window (NC == fmax - fmin + 1 when NC > 0)
  int gmode;
  const uint32_t* amax_bits;
  uint2* codes;             // 8 B per block
  uint8_t* scales;
  int8_t* offsets;          // nullable
  float2* err;              // nullable
  double2* partials;        // nullable: per-CTA {sum best, sum base}
  double* sums;             // receives the fixed-order total when partials != null
  uint32_t* ticket;         // zero-initialised counter for the last-CTA reduction
  float* g_out;             // nullable
  uint32_t* flags;
};

// Loss of one candidate (Alg. 1 lines 7-9) for the 16 values y (as 8 f32 pairs).
__device__ __forceinline__ float cand_loss(const uint64_t (&y2)[8], const float (&y)[16],
                                           float rho, uint16_t negs) {
  uint64_t acc = 0;  // {even chain a, odd chain b}
#pragma unroll
  for (int k = 0; k < 8; k++) {
    float t0, t1;
    unpack2(fmul2_bcast(y2[k], rho), t0, t1);
    uint32_t q = e2m1_round_f16x2(t0, t1);
    float d0 = fhfma((uint16_t)(q & 0xFFFFu), negs, y[2 * k]);
    float d1 = fhfma((uint16_t)(q >> 16), negs, y[2 * k + 1]);
    uint64_t d = pack2(d0, d1);
    acc = ffma2(d, d, acc);
  }
  float a, b;
  unpack2(acc, a, b);
  return __fadd_rn(a, b);
}

template <int NC>  // NC > 0: unrolled window of NC candidates; NC == 0: runtime loop
__global__ void __launch_bounds__(kThreads) quant_kernel(QuantParams p) {
  __shared__ Cand tab[128];
  __shared__ double2 red[kThreads / 32];
  build_cand_table(tab);
  const float G = global_scale(p.gmode, p.amax_bits, p.flags, blockIdx.x == 0 && threadIdx.x == 0);
  if (p.g_out && blockIdx.x == 0 && threadIdx.x == 0) *p.g_out = G;
  __syncthreads();

  const float k6 = __uint_as_float(kOneSixthBits);
  const int fmin = p.fmin;
  const int nc = NC > 0 ? NC : (p.fmax - p.fmin + 1);
  double sum_best = 0.0, sum_base = 0.0;

  for (int64_t b = (int64_t)blockIdx.x * kThreads + threadIdx.x; b < p.nb;
       b += (int64_t)gridDim.x * kThreads) {
    // a1: load 16 bf16 (32 B) and widen exactly; a3: y = RN(x * G)
    const uint4 v0 = __ldcs(p.in + 2 * b), v1 = __ldcs(p.in + 2 * b + 1);
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    float y[16];
    uint64_t y2[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      y2[k] = fmul2_bcast(pack2(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xFFFF0000u)), G);
      unpack2(y2[k], y[2 * k], y[2 * k + 1]);
    }
    // a4: block max-abs scale code c0 (Alg. 1 lines 1-2)
    float m = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; i++) m = fmaxf(m, fabsf(y[i]));
    const int c0 = (int)e4m3_code(__fmul_rn(m, k6));

    // a5: candidate search (Alg. 1 lines 5-10), lexicographic (loss, code)
    float best = __int_as_float(0x7FFFFFFF);  // NaN: first valid candidate is taken
    float base = 0.0f;
    int bc = c0;
#pragma unroll
    for (int j = 0; j < (NC > 0 ? NC : 1); j++) {
      // (NC == 0 runs the generic loop below instead)
      if (NC == 0) break;
      const int f = fmin + j;
      const int c = c0 + f;
      const bool valid = (f == 0) || ((unsigned)(c - 1) < 126u);
      const Cand e = tab[c & 127];
      const float loss = cand_loss(y2, y, e.rho, (uint16_t)e.negs);
      const bool take = valid && !(loss >= best);
      best = take ? loss : best;
      bc = take ? c : bc;
      if (f == 0) base = loss;
    }
    if (NC == 0) {
#pragma unroll 1
      for (int j = 0; j < nc; j++) {
        const int f = fmin + j;
        const int c = c0 + f;
        const bool valid = (f == 0) || ((unsigned)(c - 1) < 126u);
        if (!__any_sync(__activemask(), valid)) continue;  // warp-uniform skip
        const Cand e = tab[c & 127];
        const float loss = cand_loss(y2, y, e.rho, (uint16_t)e.negs);
        const bool take = valid && !(loss >= best);
        best = take ? loss : best;
        bc = take ? c : bc;
        if (f == 0) base = loss;
      }
    }

    // a7: emit the winner: nibbles of t = y * rho*, scale byte, offset, errors
    const float rs = tab[bc].rho;
    float t[16];
#pragma unroll
    for (int k = 0; k < 8; k++) unpack2(fmul2_bcast(y2[k], rs), t[2 * k], t[2 * k + 1]);
    uint2 code;
    code.x = e2m1_pack8(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
    code.y = e2m1_pack8(t[8], t[9], t[10], t[11], t[12], t[13], t[14], t[15]);
    __stcs(p.codes + b, code);
    p.scales[b] = (uint8_t)bc;
    if (p.offsets) p.offsets[b] = (int8_t)(bc - c0);
    if (p.err) __stcs(p.err + b, make_float2(best, base));
    sum_best += (double)best;
    sum_base += (double)base;
  }

  if (p.partials) {  // fixed-order CTA reduction (deterministic for a fixed grid)
    for (int o = 16; o > 0; o >>= 1) {
      sum_best += __shfl_xor_sync(0xFFFFFFFFu, sum_best, o);
      sum_base += __shfl_xor_sync(0xFFFFFFFFu, sum_base, o);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(sum_best, sum_base);
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 s = red[0];
      for (int i = 1; i < kThreads / 32; i++) {
        s.x += red[i].x;
        s.y += red[i].y;
      }
      p.partials[blockIdx.x] = s;
      // The last CTA to finish sums the partials in CTA order (deterministic
      // for a fixed grid) and re-arms the ticket: no separate finalize launch.
      __threadfence();
      const uint32_t done = atomicAdd(p.ticket, 1u);
      if (done == gridDim.x - 1) {
        __threadfence();
        double a = 0.0, c = 0.0;
        for (unsigned i = 0; i < gridDim.x; i++) {
          const double2 v = __ldcg(p.partials + i);
          a += v.x;
          c += v.y;
        }
        p.sums[0] = a;
        p.sums[1] = c;
        *p.ticket = 0u;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Dequantize kernel: xhat = RNE_bf16(RN((q * s) / G)).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dequant_kernel(const uint2* __restrict__ codes,
                                                      const uint8_t* __restrict__ scales,
                                                      int64_t nb, const float* __restrict__ g,
                                                      uint4* __restrict__ out) {
  const float G = g ? *g : 1.0f;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint2 cw = __ldcs(codes + b);
    const float s = f16_to_f32(e4m3_to_f16(scales[b]));
    uint32_t o[8];
    const uint32_t words[2] = {cw.x, cw.y};
#pragma unroll
    for (int h = 0; h < 2; h++) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        uint32_t q;
        asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
            "mov.b32 {b0, b1, b2, b3}, %1;\n\t"
            "cvt.rn.f16x2.e2m1x2 %0, b0;\n\t}"
            : "=r"(q) : "r"(words[h] >> (8 * k)));
        const float x0 = __fdiv_rn(__fmul_rn(f16_to_f32((uint16_t)(q & 0xFFFFu)), s), G);
        const float x1 = __fdiv_rn(__fmul_rn(f16_to_f32((uint16_t)(q >> 16)), s), G);
        uint32_t r;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x1), "f"(x0));
        o[h * 4 + k] = r;
      }
    }
    __stcs(out + 2 * b, make_uint4(o[0], o[1], o[2], o[3]));
    __stcs(out + 2 * b + 1, make_uint4(o[4], o[5], o[6], o[7]));
  }
}

}  // namespace ss
