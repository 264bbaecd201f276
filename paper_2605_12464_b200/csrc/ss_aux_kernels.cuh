// ss_aux_kernels.cuh — the amax, error-sum, row-scale and dequantize kernels.
#pragma once
#include "ss_search.cuh"

namespace ss {

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
#if SS_AMAX_PDL_TRIGGER
  pdl_launch_dependents();  // the quantize grid may launch now; it waits for this one (pdl_wait)
#endif
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
  pdl_wait();  // launched early (PDL): the quantize grid's partials must be complete
  int ti = 0;
  for (int64_t sg = blockIdx.x; sg < p.nsegs; sg += gridDim.x) {
    while (ti + 1 < p.n && p.t[ti + 1].seg0 <= sg) ti++;
    const QTensor& T = p.t[ti];
    if (!T.sums) continue;  // CTA-uniform
    const int64_t nseg = (T.npart + kSegTasks - 1) / kSegTasks;
    const int64_t k = sg - T.seg0;
    const int64_t t0 = k * kSegTasks;
    const double2 r = cta_sum(p.part1 + T.part0 + t0, min((int64_t)kSegTasks, T.npart - t0), red);
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
#if SS_AMAX_PDL_TRIGGER
  pdl_launch_dependents();
#endif
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
