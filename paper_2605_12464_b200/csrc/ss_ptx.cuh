// ss_ptx.cuh — PTX wrappers: packed FP32, FP4/FP6/FP8 conversions, cp.async.
#pragma once
#include "ss_common.cuh"

namespace ss {

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
// bf16 pair word -> (lo as f32 bits, hi as f32 bits): exact widening.  The
// low half moves up with a byte permute (integer ALU pipe) instead of a
// shift the compiler may place on the FMA pipe as IMAD.
__device__ __forceinline__ uint64_t bf16x2_to_f32x2(uint32_t w) {
#ifdef SS_PRMT_WIDEN
  uint32_t lo;
  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lo) : "r"(w));
  return pack2u(lo, w & 0xFFFF0000u);
#else
  return pack2u(w << 16, w & 0xFFFF0000u);
#endif
}
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

// ---- programmatic dependent launch (PDL) ------------------------------------
// The dependent grid may start before its predecessor finishes; pdl_wait()
// blocks until the predecessor grid has completed and its writes are visible
// (a no-op without the launch attribute).  pdl_launch_dependents() lets the
// next grid in the stream launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- inter-warp signalling (the fused amax of quant_kernel<..., AF>) -------
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// ---- peer-memory exchange (system scope: peers are other GPUs / processes) --
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// TMA bulk prefetch of [p, p + bytes) into L2 (bytes % 16 == 0); no registers, no smem
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace ss
