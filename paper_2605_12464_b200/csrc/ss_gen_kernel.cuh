// ss_gen_kernel.cuh — ScaleSearch for generic ExMy block formats (SURVEY
// NEXT(2): the "hypothetical block quantization formats" of fig:nvfp-scale,
// fig:nvfp-val and fig:mxfp; reading R21).
//
// No conversion instruction exists for most of these formats, so both
// roundings are software RNE: |t| is scaled onto its binade's quantum grid
// with an exact power-of-two ldexp in FP64 and rounded to nearest, ties to
// the even code (R10).  The candidate arithmetic is the FP32
// contract of the NVFP4 path: t = RN(y * RN(1/s)) (R7), d = RN(y - q*s) with
// q*s exact (at most vm + sm + 2 <= 24 significant bits), R12 chains, R20
// tree for 32-element blocks.  One thread per block; a study kernel, not a
// tuned one.
#pragma once
#include <cuda_bf16.h>

#include "ss_search.cuh"

namespace ss {

struct GenFmt {
  int ve, vm;      // value format ExMy (sign bit above the ve + vm magnitude bits)
  int se, sm;      // scale format UExMy
  float vmax;      // largest value magnitude
  float kinv;      // RN(1 / vmax) (R8)
  int vemin;       // exponent of the value format's smallest normal (1 - bias)
  int semin;       // same for the scale format (sm >= 1)
  int sbias;       // scale exponent bias
  int smaxc;       // largest finite scale code (the all-ones code is NaN)
  float smax;      // its value
};

struct GenParams {
  const uint4* in;     // [nb][BS / 8] 16-B vectors
  int64_t nb;          // blocks
  int fmin, fmax;
  int gmode;           // 0: G = 1; 1: G from *amax
  const uint32_t* amax;
  float g_numer;       // vmax * smax
  uint4* codes;        // [nb][BS / 16] 16-B vectors: one value code per byte
  uint8_t* scales;     // [nb]
  float2* err;         // nullable
  int8_t* offsets;     // nullable (clamped to int8)
  float* g_out;        // nullable
  double2* part1;      // nullable: per 256-block chunk {sum best, sum base}
  uint32_t* flags;
  GenFmt f;
};

// Magnitude code of a >= 0 on an ExMy grid with smallest-normal exponent
// emin: RNE on the binade's quantum grid (subnormals share the first normal
// binade's quantum).  The caller saturates.
__device__ __forceinline__ int gen_rne_code(double a, int m, int emin) {
  if (a == 0.0) return 0;
  const int e = max(ilogb(a), emin);
  const double x = ldexp(a, m - e);  // exact scaling onto the quantum grid
  const double fl = floor(x);
  const int lo = ((e - emin) << m) + (int)fl;  // fl == 2^(m+1) - 1 + 1 carries into the next binade
  // nearest; a tie goes to the even CODE (R10) -- for m = 0 the code's parity
  // is the exponent's, not the quantum count's, so rint alone is not enough
  return x - fl > 0.5 ? lo + 1 : (x - fl < 0.5 ? lo : lo + (lo & 1));
}
// Value of magnitude code c on that grid (exact).
__device__ __forceinline__ float gen_mag_value(int c, int m, int emin) {
  const int E = c >> m, M = c & ((1 << m) - 1);
  return E == 0 ? (float)ldexp((double)M, emin - m) : (float)ldexp((double)((1 << m) + M), E + emin - 1 - m);
}
// Value code (sign bit, magnitude) of t (R10, R11, R21): satfinite.
__device__ __forceinline__ int gen_value_code(float t, const GenFmt& f) {
  const int sign = signbit(t) ? (1 << (f.ve + f.vm)) : 0;
  const double a = fabs((double)t);
  const int mag = a < (double)f.vmax ? gen_rne_code(a, f.vm, f.vemin) : (1 << (f.ve + f.vm)) - 1;
  return sign | mag;
}
__device__ __forceinline__ float gen_value_of(int code, const GenFmt& f) {
  const int nm = 1 << (f.ve + f.vm);
  const float v = gen_mag_value(code & (nm - 1), f.vm, f.vemin);
  return (code & nm) ? -v : v;
}
// Scale code of v >= 0 (Alg. 1 line 2): sm >= 1 nearest (ties even) satfinite;
// sm == 0 the smallest power of two >= v, saturating (R19).
__device__ __forceinline__ int gen_scale_code(float v, const GenFmt& f) {
  const double a = (double)v;
  if (f.sm == 0) {
    if (a == 0.0) return 0;
    const int e = ilogb(a);
    const int c = e + f.sbias + (ldexp(1.0, e) < a ? 1 : 0);
    return min(max(c, 0), f.smaxc);
  }
  if (!(a < (double)f.smax)) return f.smaxc;
  return gen_rne_code(a, f.sm, f.semin);
}
__device__ __forceinline__ float gen_scale_of(int c, const GenFmt& f) {
  if (f.sm == 0) return (float)ldexp(1.0, c - f.sbias);
  return gen_mag_value(c, f.sm, f.semin);
}

// R12 loss of one 16-element part for scale s (rho = RN(1/s), 0 for s = 0).
__device__ __forceinline__ float gen_part_loss(const float* y, float s, float rho, const GenFmt& f) {
  float d[16];
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const float t = __fmul_rn(y[i], rho);
    const float q = gen_value_of(gen_value_code(t, f), f);
    d[i] = __fmaf_rn(-q, s, y[i]);
  }
  float a = __fmul_rn(d[0], d[0]), b = __fmul_rn(d[1], d[1]);
#pragma unroll
  for (int i = 2; i < 16; i += 2) {
    a = __fmaf_rn(d[i], d[i], a);
    b = __fmaf_rn(d[i + 1], d[i + 1], b);
  }
  return __fadd_rn(a, b);
}

template <int BS>
__global__ void __launch_bounds__(256) quant_gen_kernel(const __grid_constant__ GenParams p) {
  constexpr int NV = BS / 8;  // 16-B input vectors per block
  __shared__ float tab_s[256], tab_r[256];
  __shared__ double2 red[8];
  const GenFmt& f = p.f;
  for (int c = threadIdx.x; c <= f.smaxc; c += blockDim.x) {
    const float s = gen_scale_of(c, f);
    tab_s[c] = s;
    tab_r[c] = s == 0.0f ? 0.0f : __frcp_rn(s);  // IEEE RN(1/s) (R7)
  }
  __syncthreads();
  pdl_wait();  // the amax grid (PDL predecessor) has completed
  pdl_launch_dependents();
  const float G = p.gmode == 1 ? global_scale(*p.amax, p.flags, blockIdx.x == 0 && threadIdx.x == 0, p.g_numer)
                               : 1.0f;
  if (p.g_out && blockIdx.x == 0 && threadIdx.x == 0) *p.g_out = G;
  const int cmin = f.sm == 0 ? 0 : 1;
  for (int64_t ch = blockIdx.x; ch * 256 < p.nb; ch += gridDim.x) {  // CTA-uniform chunks
    const int64_t b = ch * 256 + threadIdx.x;
    double sb = 0.0, sc = 0.0;
    if (b < p.nb) {
      float y[BS];
#pragma unroll
      for (int v = 0; v < NV; v++) {  // a1 + a3: exact bf16 -> f32, y = RN(x * G)
        const uint4 w = __ldcs(p.in + NV * b + v);
        const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
          y[8 * v + 2 * k] = __fmul_rn(__uint_as_float(wd[k] << 16), G);
          y[8 * v + 2 * k + 1] = __fmul_rn(__uint_as_float(wd[k] & 0xFFFF0000u), G);
        }
      }
      float m = 0.0f;
#pragma unroll
      for (int i = 0; i < BS; i++) m = fmaxf(m, fabsf(y[i]));
      const int c0 = gen_scale_code(__fmul_rn(m, f.kinv), f);  // a4
      const int lo = max(p.fmin, cmin - c0), hi = min(p.fmax, f.smaxc - c0);
      float best = 0.0f, base = 0.0f;
      int cbest = -1;
      const bool zero_cand = f.sm > 0 && c0 == 0;  // R3
      for (int fo = zero_cand ? 0 : lo; fo <= hi; fo++) {  // a5: ascending, strict "<" (R4)
        const int c = c0 + fo;
        const float s = tab_s[c], rho = tab_r[c];
        float l = gen_part_loss(y, s, rho, f);
        if (BS == 32) l = __fadd_rn(l, gen_part_loss(y + 16, s, rho, f));  // R20
        if (fo == 0) base = l;                                               // a6
        if (cbest < 0 || l < best) {
          best = l;
          cbest = c;
        }
      }
      // a7: emit the winner's codes, one per byte
      const float rho = tab_r[cbest];
#pragma unroll
      for (int v = 0; v < BS / 16; v++) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          uint32_t word = 0;
#pragma unroll
          for (int j = 0; j < 4; j++)
            word |= (uint32_t)gen_value_code(__fmul_rn(y[16 * v + 4 * k + j], rho), f) << (8 * j);
          w[k] = word;
        }
        __stcs(p.codes + (BS / 16) * b + v, make_uint4(w[0], w[1], w[2], w[3]));
      }
      p.scales[b] = (uint8_t)cbest;
      if (p.offsets) p.offsets[b] = (int8_t)max(-128, min(127, cbest - c0));
      if (p.err) __stcs(p.err + b, make_float2(best, base));
      sb = best;
      sc = base;
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
        p.part1[ch] = t;
      }
      __syncthreads();
    }
  }
}

// a8 for generic formats: xhat = RNE_bf16(RN((q * s) / G)); q * s exact.
__global__ void __launch_bounds__(256) dequant_gen_kernel(const uint8_t* __restrict__ codes,
                                                          const uint8_t* __restrict__ scales, int64_t n,
                                                          int bs, const float* g, GenFmt f,
                                                          __nv_bfloat16* __restrict__ out) {
  const float G = g ? *g : 1.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int sc = scales[i / bs];
    const float s = (f.sm > 0 && sc == 0) ? 0.0f : gen_scale_of(sc, f);
    const float q = gen_value_of(codes[i], f);
    out[i] = __float2bfloat16_rn(__fdiv_rn(__fmul_rn(q, s), G));
  }
}

}  // namespace ss
