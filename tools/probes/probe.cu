// probe.cu — B200 (sm_100a) probes that fix the kernel's instruction choice.
//
//  (A) semantics of the conversion instructions the hot loop relies on:
//      cvt.rn.satfinite.e2m1x2.f32 (F2FP...E2M1 PACK), cvt.rn.f16x2.e2m1x2
//      (F2FP...UNPACK), cvt.rn.satfinite.e4m3x2.f32, fma.rn.f32.f16 (FHFMA).
//      Outputs are written to files and compared with the CPU oracle by
//      tests/test_probe_semantics.py (the probe computes nothing itself).
//  (B) issue throughput of each instruction and of the per-element sequence.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o probe probe.cu
// Run:   ./probe <outdir>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t e2m1_pair(float lo, float hi) {
  uint32_t v;
  asm volatile("{\n .reg .b8 b0;\n cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n"
               " cvt.u32.u8 %0, b0;\n}" : "=r"(v) : "f"(lo), "f"(hi));
  return v;
}
__device__ __forceinline__ uint32_t e4m3_pair(float lo, float hi) {
  uint16_t v;
  asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %2, %1;" : "=h"(v) : "f"(lo), "f"(hi));
  return v;
}

// ---- (A) transitions of the hardware rounding functions ------------------
// For patterns p in [lo, hi) of one sign, record p whenever code(p) != code(p-1).
__global__ void e2m1_transitions(uint32_t base, uint64_t n, uint32_t* out, uint32_t* cnt) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint32_t p = base + (uint32_t)i;
    uint32_t c = e2m1_pair(__uint_as_float(p), 0.0f) & 15;
    uint32_t cp = (i == 0) ? 0xFFu : (e2m1_pair(__uint_as_float(p - 1), 0.0f) & 15);
    if (c != cp) {
      uint32_t k = atomicAdd(cnt, 1u);
      if (k < 4096) { out[2 * k] = p; out[2 * k + 1] = c; }
    }
  }
}
__global__ void e4m3_transitions(uint32_t base, uint64_t n, uint32_t* out, uint32_t* cnt) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint32_t p = base + (uint32_t)i;
    uint32_t c = e4m3_pair(__uint_as_float(p), 0.0f) & 0xFF;
    uint32_t cp = (i == 0) ? 0xFFFu : (e4m3_pair(__uint_as_float(p - 1), 0.0f) & 0xFF);
    if (c != cp) {
      uint32_t k = atomicAdd(cnt, 1u);
      if (k < 4096) { out[2 * k] = p; out[2 * k + 1] = c; }
    }
  }
}
// all 256 bytes through the unpack
__global__ void e2m1_unpack_all(uint32_t* out) {
  uint32_t b = threadIdx.x;
  uint32_t h;
  asm volatile("{\n .reg .b8 b0;\n cvt.u8.u32 b0, %1;\n cvt.rn.f16x2.e2m1x2 %0, b0;\n}" : "=r"(h) : "r"(b));
  out[b] = h;
}
// pair order check: which input lands in the low nibble
__global__ void e2m1_pair_order(uint32_t* out) {
  out[0] = e2m1_pair(1.0f, 6.0f);   // expect lo nibble 2 (1.0), hi nibble 7 (6.0)
  out[1] = e4m3_pair(1.0f, 448.0f); // expect lo byte 0x38, hi byte 0x7E
}
// fma.rn.f32.f16 on (q, -s, y) triples
__global__ void fhfma_check(const uint16_t* a, const uint16_t* b, const float* c, float* d, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float r;
    asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(r) : "h"(a[i]), "h"(b[i]), "f"(c[i]));
    d[i] = r;
  }
}

// ---- (B) throughput -------------------------------------------------------
#define NITER 4096
template <int OP>
__global__ void __launch_bounds__(256) tput(float* sink, float seed, long long* cycles) {
  float x[8];
  uint32_t u[8];
  unsigned long long X[4];
#pragma unroll
  for (int k = 0; k < 8; k++) { x[k] = seed + threadIdx.x * 1e-3f + k; u[k] = __float_as_uint(x[k]) & 0x77777777u; }
#pragma unroll
  for (int k = 0; k < 4; k++) asm volatile("mov.b64 %0, {%1,%2};" : "=l"(X[k]) : "f"(x[2*k]), "f"(x[2*k+1]));
  long long t0 = clock64();
  for (int it = 0; it < NITER; it++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (OP == 0) {        // FFMA 3-reg
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(x[(k + 1) & 7]), "f"(x[(k + 3) & 7]));
      } else if (OP == 1) { // FFMA2
        if (k < 4) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(X[k]) : "l"(X[(k + 1) & 3]), "l"(X[(k + 2) & 3]));
      } else if (OP == 2) { // FMUL2
        if (k < 4) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(X[k]) : "l"(X[(k + 1) & 3]));
      } else if (OP == 3) { // F2FP e2m1 pack
        uint32_t v;
        asm volatile("{\n .reg .b8 b0;\n cvt.rn.satfinite.e2m1x2.f32 b0, %1, %2;\n cvt.u32.u8 %0, b0;\n}" : "=r"(v) : "f"(x[k]), "f"(x[(k+1)&7]));
        x[k] = __uint_as_float(__float_as_uint(x[k]) ^ v);
      } else if (OP == 4) { // F2FP e2m1 unpack
        uint32_t h;
        asm volatile("{\n .reg .b8 b0;\n cvt.u8.u32 b0, %1;\n cvt.rn.f16x2.e2m1x2 %0, b0;\n}" : "=r"(h) : "r"(u[k]));
        u[k] = h;
      } else if (OP == 5) { // FHFMA
        asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(x[k]) : "h"((uint16_t)u[k]), "h"((uint16_t)(u[k] >> 16)));
      } else if (OP == 6) { // FMUL scalar
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[k]) : "f"(x[(k + 1) & 7]));
      } else if (OP == 7) { // integer/logic on alu pipe (LOP3)
        u[k] = (u[k] ^ u[(k + 1) & 7]) & (u[(k + 2) & 7] | 0x1234u);
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; k++) acc += x[k] + __uint_as_float(u[k]);
#pragma unroll
  for (int k = 0; k < 4; k++) acc += __uint_as_float((uint32_t)X[k]);
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// The per-2-element candidate sequence of the hot loop:
// FMUL2 (t = y*rho) -> F2FP pack -> F2FP unpack -> 2x FHFMA (d = y - q*s) -> FFMA2 (acc += d*d)
__global__ void __launch_bounds__(256) tput_seq(float* sink, float seed, long long* cycles) {
  float y[16];
#pragma unroll
  for (int k = 0; k < 16; k++) y[k] = seed + threadIdx.x * 1e-3f + k * 0.37f;
  unsigned long long acc = 0;
  float rho = 0.731f;
  uint16_t negs = 0xBC00;  // -1.0 in f16
  long long t0 = clock64();
  for (int it = 0; it < NITER / 8; it++) {
    unsigned long long R;
    asm volatile("mov.b64 %0, {%1,%1};" : "=l"(R) : "f"(rho));
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      unsigned long long Y, T, D;
      asm volatile("mov.b64 %0, {%1,%2};" : "=l"(Y) : "f"(y[k]), "f"(y[k + 1]));
      asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(T) : "l"(Y), "l"(R));
      float t0f, t1f;
      asm volatile("mov.b64 {%0,%1}, %2;" : "=f"(t0f), "=f"(t1f) : "l"(T));
      uint32_t h;
      asm volatile("{\n .reg .b8 b0;\n cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n cvt.rn.f16x2.e2m1x2 %0, b0;\n}" : "=r"(h) : "f"(t0f), "f"(t1f));
      float d0, d1;
      asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d0) : "h"((uint16_t)h), "h"(negs), "f"(y[k]));
      asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d1) : "h"((uint16_t)(h >> 16)), "h"(negs), "f"(y[k + 1]));
      asm volatile("mov.b64 %0, {%1,%2};" : "=l"(D) : "f"(d0), "f"(d1));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(D));
    }
    rho = rho * 1.0001f;
  }
  long long t1 = clock64();
  if (__uint_as_float((uint32_t)acc) == 1.2345f) sink[threadIdx.x] = 1.f;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

static void write_file(const std::string& path, const void* p, size_t n) {
  FILE* f = fopen(path.c_str(), "wb");
  if (!f) { perror(path.c_str()); exit(1); }
  fwrite(p, 1, n, f);
  fclose(f);
}

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : ".";
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("{\"device\": \"%s\", \"sm\": %d, \"cc\": \"%d.%d\", \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"regs_per_sm\": %d, \"clock_khz\": %d,\n",
         prop.name, prop.multiProcessorCount, prop.major, prop.minor, prop.l2CacheSize,
         prop.sharedMemPerMultiprocessor, prop.regsPerMultiprocessor, clk_khz);

  // (A) semantics
  uint32_t *d_out, *d_cnt;
  CK(cudaMalloc(&d_out, 8 * 4096));
  CK(cudaMalloc(&d_cnt, 4));
  const char* names[4] = {"e2m1_pos", "e2m1_neg", "e4m3_pos", "e4m3_neg"};
  for (int w = 0; w < 4; w++) {
    CK(cudaMemset(d_cnt, 0, 4));
    uint32_t base = (w & 1) ? 0x80000000u : 0u;
    if (w < 2) e2m1_transitions<<<148 * 16, 256>>>(base, 1ull << 31, d_out, d_cnt);
    else e4m3_transitions<<<148 * 16, 256>>>(base, 1ull << 31, d_out, d_cnt);
    CK(cudaDeviceSynchronize());
    uint32_t cnt;
    CK(cudaMemcpy(&cnt, d_cnt, 4, cudaMemcpyDeviceToHost));
    if (cnt > 4096) cnt = 4096;
    std::vector<uint32_t> h(2 * cnt);
    CK(cudaMemcpy(h.data(), d_out, 8 * cnt, cudaMemcpyDeviceToHost));
    write_file(dir + "/" + names[w] + "_transitions.u32", h.data(), 8 * cnt);
    printf("\"%s_transitions\": %u,\n", names[w], cnt);
  }
  e2m1_unpack_all<<<1, 256>>>(d_out);
  CK(cudaDeviceSynchronize());
  {
    std::vector<uint32_t> h(256);
    CK(cudaMemcpy(h.data(), d_out, 1024, cudaMemcpyDeviceToHost));
    write_file(dir + "/e2m1_unpack.u32", h.data(), 1024);
  }
  e2m1_pair_order<<<1, 1>>>(d_out);
  CK(cudaDeviceSynchronize());
  {
    uint32_t h[2];
    CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
    printf("\"pair_order_e2m1\": %u, \"pair_order_e4m3\": %u,\n", h[0], h[1]);
  }
  {
    const int n = 1 << 20;
    std::vector<uint16_t> a(n), b(n);
    std::vector<float> c(n), d(n);
    const uint16_t qs[8] = {0x0000, 0x3800, 0x3C00, 0x3E00, 0x4000, 0x4200, 0x4400, 0x4600};  // 0,.5,1,1.5,2,3,4,6
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < n; i++) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      a[i] = qs[s & 7] | ((s >> 3) & 1 ? 0x8000 : 0);
      int code = 1 + (int)((s >> 4) % 126);            // E4M3 code -> f16 bits (exact)
      int e = code >> 3, m = code & 7;
      float sv = e == 0 ? m * (1.0f / 512.0f) : (1.0f + m / 8.0f) * ldexpf(1.0f, e - 7);
      __half hs = __float2half_rn(-sv);
      b[i] = *reinterpret_cast<uint16_t*>(&hs);
      uint32_t yb = (uint32_t)(s >> 20);
      float y = ldexpf(1.0f + (yb & 0xFFFFFF) / 16777216.0f, (int)((s >> 44) % 24) - 12);
      c[i] = (s >> 63) ? -y : y;
    }
    uint16_t *da, *db; float *dc, *dd;
    CK(cudaMalloc(&da, 2 * n)); CK(cudaMalloc(&db, 2 * n)); CK(cudaMalloc(&dc, 4 * n)); CK(cudaMalloc(&dd, 4 * n));
    CK(cudaMemcpy(da, a.data(), 2 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), 2 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc, c.data(), 4 * n, cudaMemcpyHostToDevice));
    fhfma_check<<<n / 256, 256>>>(da, db, dc, dd, n);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(d.data(), dd, 4 * n, cudaMemcpyDeviceToHost));
    write_file(dir + "/fhfma_a.u16", a.data(), 2 * n);
    write_file(dir + "/fhfma_b.u16", b.data(), 2 * n);
    write_file(dir + "/fhfma_c.f32", c.data(), 4 * n);
    write_file(dir + "/fhfma_d.f32", d.data(), 4 * n);
  }

  // (B) throughput
  float* sink; long long* cyc;
  const int block = 256;
  int occs[9];
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[0], tput<0>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[1], tput<1>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[2], tput<2>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[3], tput<3>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[4], tput<4>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[5], tput<5>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[6], tput<6>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[7], tput<7>, block, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[8], tput_seq, block, 0));
  CK(cudaMalloc(&sink, 4 * 1024));
  CK(cudaMalloc(&cyc, 8 * prop.multiProcessorCount * 32));
  std::vector<long long> hc(prop.multiProcessorCount * 32);
  const char* opn[9] = {"FFMA", "FFMA2", "FMUL2", "F2FP_E2M1_PACK", "F2FP_E2M1_UNPACK", "FHFMA", "FMUL", "LOP3", "SEQ_per_2elem"};
  printf("\"throughput_warp_inst_per_clk_per_sm\": {");
  for (int op = 0; op < 9; op++) {
    const int grid = prop.multiProcessorCount * occs[op];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      switch (op) {
        case 0: tput<0><<<grid, block>>>(sink, 1.f, cyc); break;
        case 1: tput<1><<<grid, block>>>(sink, 1.f, cyc); break;
        case 2: tput<2><<<grid, block>>>(sink, 1.f, cyc); break;
        case 3: tput<3><<<grid, block>>>(sink, 1.f, cyc); break;
        case 4: tput<4><<<grid, block>>>(sink, 1.f, cyc); break;
        case 5: tput<5><<<grid, block>>>(sink, 1.f, cyc); break;
        case 6: tput<6><<<grid, block>>>(sink, 1.f, cyc); break;
        case 7: tput<7><<<grid, block>>>(sink, 1.f, cyc); break;
        case 8: tput_seq<<<grid, block>>>(sink, 1.f, cyc); break;
      }
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hc.data(), cyc, 8 * grid, cudaMemcpyDeviceToHost));
    double avg = 0; for (int q = 0; q < grid; q++) avg += hc[q]; avg /= grid;
    // per CTA: 8 warps; instructions per warp = NITER * (8 or 4) ; 8 CTAs per SM resident
    double per_warp = (op == 1 || op == 2) ? NITER * 4.0 : (op == 8 ? (NITER / 8) * 8.0 : NITER * 8.0);
    double insts_per_sm = per_warp * 8 /*warps*/ * occs[op] /*co-resident ctas per sm*/;
    double sm_clk_hz = avg / (ms * 1e-3) ;   // cycles per CTA over wall time ~ clock (approx)
    double ipc = insts_per_sm / avg;         // all 8 CTAs co-resident for the whole run
    printf("%s\"%s\": {\"ipc_sm\": %.3f, \"ms\": %.4f, \"cyc_per_cta\": %.0f, \"approx_clk_mhz\": %.0f, \"occ\": %d}",
           op ? ", " : "", opn[op], ipc, ms, avg, sm_clk_hz / 1e6, occs[op]);
  }
  printf("}}\n");
  return 0;
}
