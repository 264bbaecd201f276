// ss_api.cu — host side of libss.so: the C ABI declared in include/ss.h.
//
// Argument validation, per-(device, stream) workspace, kernel-variant
// dispatch by candidate count, the end-to-end host-buffer pipeline, and
// status reporting.  No CPU compute path exists: every entry point either
// launches sm_100a kernels or returns an error.
#include "ss.h"
#include "ss_kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

namespace {

using ss::Cand;
using ss::QuantParams;

struct Workspace {
  uint32_t* amax = nullptr;     // SS_GLOBAL_TENSOR slot
  uint32_t* flags = nullptr;    // sticky status flags
  uint32_t* ticket = nullptr;   // last-CTA reduction counter (self re-arming)
  double2* partials = nullptr;  // per-CTA error partial sums
  int partial_cap = 0;
};

std::mutex g_mu;
std::map<std::pair<int, void*>, Workspace> g_ws;

struct DeviceInfo {
  bool ok = false;
  int sms = 0;
};
DeviceInfo g_dev[64];
bool g_dev_init[64] = {false};

ss_status device_check(int* dev_out, DeviceInfo* info_out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return SS_ERR_UNSUPPORTED_DEVICE;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_dev_init[dev]) {
    int major = 0, sms = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    g_dev[dev].ok = (major == 10);
    g_dev[dev].sms = sms;
    g_dev_init[dev] = true;
  }
  if (!g_dev[dev].ok) return SS_ERR_UNSUPPORTED_DEVICE;
  *dev_out = dev;
  *info_out = g_dev[dev];
  return SS_OK;
}

ss_status get_ws(int dev, void* stream, int need_partials, Workspace** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  Workspace& w = g_ws[std::make_pair(dev, stream)];
  if (!w.amax) {
    void* p = nullptr;
    if (cudaMalloc(&p, 64) != cudaSuccess) return SS_ERR_CUDA;
    if (cudaMemset(p, 0, 64) != cudaSuccess) return SS_ERR_CUDA;
    w.amax = reinterpret_cast<uint32_t*>(p);
    w.flags = w.amax + 1;
    w.ticket = w.amax + 2;
  }
  if (need_partials > w.partial_cap) {
    if (w.partials) cudaFree(w.partials);
    void* p = nullptr;
    int cap = std::max(need_partials, 4096);
    if (cudaMalloc(&p, sizeof(double2) * cap) != cudaSuccess) return SS_ERR_CUDA;
    w.partials = reinterpret_cast<double2*>(p);
    w.partial_cap = cap;
  }
  *out = &w;
  return SS_OK;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

ss_status launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

ss_status amax_launch(const void* in, int64_t n, uint32_t* d_amax, bool accumulate,
                      cudaStream_t st, int sms) {
  if (!accumulate && cudaMemsetAsync(d_amax, 0, 4, st) != cudaSuccess) return SS_ERR_CUDA;
  if (n == 0) return SS_OK;
  const int64_t n16 = n / 8;
  const int n_tail = (int)(n % 8);
  const uint16_t* tail = reinterpret_cast<const uint16_t*>(in) + n16 * 8;
  int64_t want = (n16 + 255) / 256;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
  ss::amax_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(in), n16, tail, n_tail,
                                        d_amax);
  return launch_status();
}

// ---- quantize kernel variants ----------------------------------------------
typedef void (*QuantKernel)(QuantParams);

template <int NC>
QuantKernel kernel_for() { return ss::quant_kernel<NC>; }

QuantKernel pick_kernel(int nc) {
  switch (nc) {
#define SS_CASE(N) case N: return kernel_for<N>();
    SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8)
    SS_CASE(9) SS_CASE(10) SS_CASE(11) SS_CASE(12) SS_CASE(13) SS_CASE(14) SS_CASE(15)
    SS_CASE(16) SS_CASE(17) SS_CASE(25) SS_CASE(33)
#undef SS_CASE
    default: return kernel_for<0>();
  }
}

int occupancy(QuantKernel k) {
  static std::mutex mu;
  static std::map<QuantKernel, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(k);
  if (it != cache.end()) return it->second;
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, ss::kThreads, 0) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  occ = std::max(occ, 1);
  cache[k] = occ;
  return occ;
}

ss_status quantize_impl(const ss_quant_args* a) {
  if (!a) return SS_ERR_INVALID_ARG;
  if (a->rows < 0 || a->cols < 0 || (a->cols % 16) != 0) return SS_ERR_INVALID_ARG;
  if (a->f_min > 0 || a->f_max < 0) return SS_ERR_INVALID_ARG;
  if (a->global_scale_mode < 0 || a->global_scale_mode > 2) return SS_ERR_INVALID_ARG;
  if (a->global_scale_mode == SS_GLOBAL_DEVICE_AMAX && !a->d_amax_bits) return SS_ERR_INVALID_ARG;
  const int64_t n = a->rows * a->cols, nb = n / 16;
  if (nb > 0 && (!a->in_bf16 || !a->out_codes || !a->out_scales)) return SS_ERR_INVALID_ARG;
  if (!aligned(a->in_bf16, 16) || !aligned(a->out_codes, 8) || !aligned(a->out_err, 8))
    return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  ss_status st = device_check(&dev, &info);
  if (st) return st;
  const int fmin = std::max(a->f_min, -126), fmax = std::min(a->f_max, 126);
  const int nc = fmax - fmin + 1;
  QuantKernel k = pick_kernel(nc);
  const int occ = occupancy(k);
  int64_t want = (nb + ss::kThreads - 1) / ss::kThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)info.sms * occ));

  Workspace* ws = nullptr;
  st = get_ws(dev, a->stream, a->d_err_sums ? grid : 0, &ws);
  if (st) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(a->stream);

  const uint32_t* amax = a->d_amax_bits;
  if (a->global_scale_mode == SS_GLOBAL_TENSOR) {
    st = amax_launch(a->in_bf16, n, ws->amax, false, cs, info.sms);
    if (st) return st;
    amax = ws->amax;
  }
  if (nb == 0) {
    if (a->d_err_sums && cudaMemsetAsync(a->d_err_sums, 0, 16, cs) != cudaSuccess) return SS_ERR_CUDA;
    return SS_OK;
  }
  QuantParams p;
  p.in = reinterpret_cast<const uint4*>(a->in_bf16);
  p.nb = nb;
  p.fmin = fmin;
  p.fmax = fmax;
  p.gmode = a->global_scale_mode == SS_GLOBAL_NONE ? 0 : 1;
  p.amax_bits = amax ? amax : ws->amax;
  p.codes = reinterpret_cast<uint2*>(a->out_codes);
  p.scales = a->out_scales;
  p.offsets = a->out_offset;
  p.err = reinterpret_cast<float2*>(a->out_err);
  p.partials = a->d_err_sums ? ws->partials : nullptr;
  p.sums = a->d_err_sums;
  p.ticket = ws->ticket;
  p.g_out = a->d_global_scale;
  p.flags = ws->flags;
  k<<<grid, ss::kThreads, 0, cs>>>(p);
  return launch_status();
}

// ---- end-to-end host pipeline -----------------------------------------------
struct HostPipe {
  void* d_in = nullptr;
  void* d_codes = nullptr;
  void* d_scales = nullptr;
  void* d_err = nullptr;
  size_t cap_in = 0, cap_codes = 0, cap_scales = 0, cap_err = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  uint32_t* d_amax = nullptr;
};
std::mutex g_pipe_mu;
std::map<int, HostPipe> g_pipes;

ss_status grow(void** p, size_t* cap, size_t need) {
  if (need <= *cap) return SS_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  if (cudaMalloc(p, need) != cudaSuccess) return SS_ERR_CUDA;
  *cap = need;
  return SS_OK;
}

}  // namespace

extern "C" {

const char* ss_status_string(int s) {
  switch (s) {
    case SS_OK: return "ok";
    case SS_ERR_INVALID_ARG: return "invalid argument";
    case SS_ERR_ALIGNMENT: return "misaligned pointer";
    case SS_ERR_CUDA: return "CUDA error";
    case SS_ERR_NONFINITE: return "non-finite input";
    case SS_ERR_RANGE: return "global scale out of range";
    case SS_ERR_UNSUPPORTED_DEVICE: return "unsupported device (need compute capability 10.x)";
    default: return "unknown status";
  }
}

int ss_version(void) { return 100; }

ss_status ss_tensor_amax(const void* in_bf16, int64_t n, uint32_t* d_amax_bits, int accumulate,
                         void* stream) {
  if (n < 0 || !d_amax_bits || (n > 0 && !in_bf16)) return SS_ERR_INVALID_ARG;
  if (!aligned(in_bf16, 16)) return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  ss_status st = device_check(&dev, &info);
  if (st) return st;
  return amax_launch(in_bf16, n, d_amax_bits, accumulate != 0,
                     reinterpret_cast<cudaStream_t>(stream), info.sms);
}

ss_status ss_quantize_nvfp4(const void* in_bf16, int64_t rows, int64_t cols, int radius,
                            int global_scale_mode, uint8_t* out_codes, uint8_t* out_scales,
                            float* out_err, void* stream) {
  if (radius < 0) return SS_ERR_INVALID_ARG;
  if (global_scale_mode == SS_GLOBAL_DEVICE_AMAX) return SS_ERR_INVALID_ARG;
  ss_quant_args a;
  std::memset(&a, 0, sizeof(a));
  a.in_bf16 = in_bf16;
  a.rows = rows;
  a.cols = cols;
  a.f_min = -std::min(radius, 126);
  a.f_max = std::min(radius, 126);
  a.global_scale_mode = global_scale_mode;
  a.out_codes = out_codes;
  a.out_scales = out_scales;
  a.out_err = out_err;
  a.stream = stream;
  return quantize_impl(&a);
}

ss_status ss_quantize_nvfp4_ex(const ss_quant_args* args) { return quantize_impl(args); }

ss_status ss_dequantize_nvfp4(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                              int64_t cols, const float* d_global_scale, void* out_bf16,
                              void* stream) {
  if (rows < 0 || cols < 0 || cols % 16 != 0) return SS_ERR_INVALID_ARG;
  const int64_t nb = rows * cols / 16;
  if (nb > 0 && (!codes || !scales || !out_bf16)) return SS_ERR_INVALID_ARG;
  if (!aligned(codes, 8) || !aligned(out_bf16, 16)) return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  ss_status st = device_check(&dev, &info);
  if (st) return st;
  if (nb == 0) return SS_OK;
  int64_t want = (nb + 255) / 256;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)info.sms * 8));
  ss::dequant_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint2*>(codes), scales, nb, d_global_scale,
      reinterpret_cast<uint4*>(out_bf16));
  return launch_status();
}

ss_status ss_get_device_status(int* flags, void* stream) {
  if (!flags) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  ss_status st = device_check(&dev, &info);
  if (st) return st;
  Workspace* ws = nullptr;
  st = get_ws(dev, stream, 0, &ws);
  if (st) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  uint32_t h = 0;
  if (cudaMemcpyAsync(&h, ws->flags, 4, cudaMemcpyDeviceToHost, cs) != cudaSuccess) return SS_ERR_CUDA;
  if (cudaMemsetAsync(ws->flags, 0, 4, cs) != cudaSuccess) return SS_ERR_CUDA;
  if (cudaStreamSynchronize(cs) != cudaSuccess) return SS_ERR_CUDA;
  *flags = (int)h;
  return SS_OK;
}

ss_status ss_quantize_nvfp4_host(const void* h_in, int64_t rows, int64_t cols, int f_min,
                                 int f_max, int global_scale_mode, uint8_t* h_codes,
                                 uint8_t* h_scales, float* h_err) {
  if (rows < 0 || cols < 0 || cols % 16 != 0 || f_min > 0 || f_max < 0) return SS_ERR_INVALID_ARG;
  if (global_scale_mode != SS_GLOBAL_NONE && global_scale_mode != SS_GLOBAL_TENSOR)
    return SS_ERR_INVALID_ARG;
  const int64_t n = rows * cols, nb = n / 16;
  if (nb > 0 && (!h_in || !h_codes || !h_scales)) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  ss_status st = device_check(&dev, &info);
  if (st) return st;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostPipe& hp = g_pipes[dev];
  if (!hp.s_h2d) {
    if (cudaStreamCreateWithFlags(&hp.s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hp.s_comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hp.s_d2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&hp.d_amax, 64) != cudaSuccess)
      return SS_ERR_CUDA;
  }
  if (nb == 0) return SS_OK;
  if ((st = grow(&hp.d_in, &hp.cap_in, (size_t)n * 2)) ||
      (st = grow(&hp.d_codes, &hp.cap_codes, (size_t)nb * 8)) ||
      (st = grow(&hp.d_scales, &hp.cap_scales, (size_t)nb)) ||
      (h_err && (st = grow(&hp.d_err, &hp.cap_err, (size_t)nb * 8))))
    return st;
  // chunks of whole rows, ~32 Mi elements (64 MB of bf16) each
  const int64_t chunk_rows = std::max<int64_t>(1, (int64_t(32) << 20) / std::max<int64_t>(cols, 1));
  const int64_t nchunks = (rows + chunk_rows - 1) / chunk_rows;
  const char* hin = reinterpret_cast<const char*>(h_in);
  char* din = reinterpret_cast<char*>(hp.d_in);
  const bool tensor = global_scale_mode == SS_GLOBAL_TENSOR;
  cudaEvent_t ev_in[2], ev_out[2];
  for (int i = 0; i < 2; i++) {
    cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
  }
  auto fail = [&](ss_status s) {
    for (int i = 0; i < 2; i++) {
      cudaEventDestroy(ev_in[i]);
      cudaEventDestroy(ev_out[i]);
    }
    return s;
  };
  if (tensor && cudaMemsetAsync(hp.d_amax, 0, 4, hp.s_comp) != cudaSuccess) return fail(SS_ERR_CUDA);
  // phase 1: H2D every chunk; in TENSOR mode the amax of each chunk follows its copy
  for (int64_t k = 0; k < nchunks; k++) {
    const int64_t r0 = k * chunk_rows, r1 = std::min(rows, r0 + chunk_rows);
    const size_t off = (size_t)r0 * cols * 2, bytes = (size_t)(r1 - r0) * cols * 2;
    if (cudaMemcpyAsync(din + off, hin + off, bytes, cudaMemcpyHostToDevice, hp.s_h2d) != cudaSuccess)
      return fail(SS_ERR_CUDA);
    cudaEventRecord(ev_in[k & 1], hp.s_h2d);
    cudaStreamWaitEvent(hp.s_comp, ev_in[k & 1], 0);
    if (tensor) {
      if ((st = amax_launch(din + off, (r1 - r0) * cols, hp.d_amax, true, hp.s_comp, info.sms)))
        return fail(st);
    } else {
      // NONE mode: quantize and copy back chunk by chunk as the input lands
      ss_quant_args a;
      std::memset(&a, 0, sizeof(a));
      a.in_bf16 = din + off;
      a.rows = r1 - r0;
      a.cols = cols;
      a.f_min = f_min;
      a.f_max = f_max;
      a.global_scale_mode = SS_GLOBAL_NONE;
      a.out_codes = reinterpret_cast<uint8_t*>(hp.d_codes) + (size_t)r0 * cols / 2;
      a.out_scales = reinterpret_cast<uint8_t*>(hp.d_scales) + (size_t)r0 * cols / 16;
      a.out_err = h_err ? reinterpret_cast<float*>(hp.d_err) + (size_t)r0 * cols / 8 : nullptr;
      a.stream = hp.s_comp;
      if ((st = quantize_impl(&a))) return fail(st);
      cudaEventRecord(ev_out[k & 1], hp.s_comp);
      cudaStreamWaitEvent(hp.s_d2h, ev_out[k & 1], 0);
      cudaMemcpyAsync(h_codes + (size_t)r0 * cols / 2, a.out_codes, (size_t)(r1 - r0) * cols / 2,
                      cudaMemcpyDeviceToHost, hp.s_d2h);
      cudaMemcpyAsync(h_scales + (size_t)r0 * cols / 16, a.out_scales,
                      (size_t)(r1 - r0) * cols / 16, cudaMemcpyDeviceToHost, hp.s_d2h);
      if (h_err)
        cudaMemcpyAsync(h_err + (size_t)r0 * cols / 8, a.out_err, (size_t)(r1 - r0) * cols / 2,
                        cudaMemcpyDeviceToHost, hp.s_d2h);
    }
  }
  if (tensor) {
    // phase 2: quantize chunk by chunk with the final amax, copying results back
    for (int64_t k = 0; k < nchunks; k++) {
      const int64_t r0 = k * chunk_rows, r1 = std::min(rows, r0 + chunk_rows);
      ss_quant_args a;
      std::memset(&a, 0, sizeof(a));
      a.in_bf16 = din + (size_t)r0 * cols * 2;
      a.rows = r1 - r0;
      a.cols = cols;
      a.f_min = f_min;
      a.f_max = f_max;
      a.global_scale_mode = SS_GLOBAL_DEVICE_AMAX;
      a.d_amax_bits = hp.d_amax;
      a.out_codes = reinterpret_cast<uint8_t*>(hp.d_codes) + (size_t)r0 * cols / 2;
      a.out_scales = reinterpret_cast<uint8_t*>(hp.d_scales) + (size_t)r0 * cols / 16;
      a.out_err = h_err ? reinterpret_cast<float*>(hp.d_err) + (size_t)r0 * cols / 8 : nullptr;
      a.stream = hp.s_comp;
      if ((st = quantize_impl(&a))) return fail(st);
      cudaEventRecord(ev_out[k & 1], hp.s_comp);
      cudaStreamWaitEvent(hp.s_d2h, ev_out[k & 1], 0);
      cudaMemcpyAsync(h_codes + (size_t)r0 * cols / 2, a.out_codes, (size_t)(r1 - r0) * cols / 2,
                      cudaMemcpyDeviceToHost, hp.s_d2h);
      cudaMemcpyAsync(h_scales + (size_t)r0 * cols / 16, a.out_scales,
                      (size_t)(r1 - r0) * cols / 16, cudaMemcpyDeviceToHost, hp.s_d2h);
      if (h_err)
        cudaMemcpyAsync(h_err + (size_t)r0 * cols / 8, a.out_err, (size_t)(r1 - r0) * cols / 2,
                        cudaMemcpyDeviceToHost, hp.s_d2h);
    }
  }
  cudaError_t e1 = cudaStreamSynchronize(hp.s_comp);
  cudaError_t e2 = cudaStreamSynchronize(hp.s_d2h);
  cudaError_t e3 = cudaStreamSynchronize(hp.s_h2d);
  return fail((e1 || e2 || e3) ? SS_ERR_CUDA : SS_OK);
}

}  // extern "C"
