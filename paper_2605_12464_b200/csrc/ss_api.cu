// ss_api.cu — host side of libss.so: the C ABI declared in include/ss.h.
//
// Argument validation, per-(device, stream) workspace, batching of tensors
// into launches, kernel-variant dispatch by search window, the end-to-end
// host-buffer pipeline, and status reporting.  No CPU compute path exists:
// every entry point either launches sm_100a kernels or returns an error.
#include "ss.h"
#include "ss_kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

namespace {

using ss::AmaxBatch;
using ss::ATensor;
using ss::QTensor;
using ss::QuantBatch;

// ---- per-(device, stream) workspace -----------------------------------------
struct Workspace {
  uint32_t* flags = nullptr;     // sticky status flags (1 word)
  uint32_t* tick = nullptr;      // [kMaxTensors] per-tensor tickets (zero, self re-arming)
  uint32_t* ctr = nullptr;       // [kCounters + 1] scheduler counters (zero, self re-arming)
  uint32_t* done = nullptr;      // [kMaxTensors + 1] fused-amax completion counts + unit counter (zero, self re-arming)
  uint32_t* amax = nullptr;      // SS_GLOBAL_TENSOR slots
  int64_t amax_cap = 0;
  double2* part1 = nullptr;      // per-task partial sums
  int64_t part1_cap = 0;
  double2* part2 = nullptr;      // per-segment partial sums
  int64_t part2_cap = 0;
  // Held while a call grows and uses this workspace and enqueues its
  // launches.  Calls on distinct streams use distinct workspaces and never
  // wait for each other; a grow synchronizes only this workspace's stream.
  std::mutex mu;
};

std::mutex g_mu;      // the workspace map (lookup / insertion only)
std::mutex g_dev_mu;  // one-time device queries
#if defined(SS_COUNT_EVALS) || defined(SS_AF_TRACE)
unsigned long long* g_evals = nullptr;  // tools-only counting / tracing builds
#endif

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
  std::lock_guard<std::mutex> lk(g_dev_mu);
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

// Grow a device array; a buffer that may still be in use by queued kernels is
// released only after the stream drains.  `zero` clears the new buffer (on the
// stream, before any later kernel).
template <typename T>
ss_status grow_dev(T** p, int64_t* cap, int64_t need, bool zero, cudaStream_t st) {
  if (need <= *cap) return SS_OK;
  const int64_t n = std::max<int64_t>(need, std::max<int64_t>(2 * *cap, 1024));
  if (*p) {
    if (cudaStreamSynchronize(st) != cudaSuccess) return SS_ERR_CUDA;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
  }
  void* q = nullptr;
  if (cudaMalloc(&q, sizeof(T) * n) != cudaSuccess) return SS_ERR_CUDA;
  if (zero && cudaMemsetAsync(q, 0, sizeof(T) * n, st) != cudaSuccess) return SS_ERR_CUDA;
  *p = reinterpret_cast<T*>(q);
  *cap = n;
  return SS_OK;
}

// Workspace of (dev, stream), created on first use.  std::map nodes never
// move, so the pointer stays valid after g_mu is released.
ss_status get_ws(int dev, void* stream, Workspace** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  Workspace& w = g_ws[std::make_pair(dev, stream)];
  if (!w.flags) {
    void* p = nullptr;
    const size_t bytes = sizeof(uint32_t) * (1 + ss::kMaxTensors + ss::kCounters + 1 + ss::kMaxTensors + 2);
    if (cudaMalloc(&p, bytes) != cudaSuccess) return SS_ERR_CUDA;
    if (cudaMemset(p, 0, bytes) != cudaSuccess) return SS_ERR_CUDA;
    w.flags = reinterpret_cast<uint32_t*>(p);
    w.tick = w.flags + 1;
    w.ctr = w.tick + ss::kMaxTensors;
    w.done = w.ctr + ss::kCounters + 1;
  }
  *out = &w;
  return SS_OK;
}

struct FmtInfo {
  int vf, sf, bs;
};
bool fmt_info(int format, FmtInfo* f) {
  switch (format) {
    case SS_FMT_NVFP4: *f = {0, 0, 16}; return true;
    case SS_FMT_MXFP4: *f = {0, 1, 32}; return true;
    case SS_FMT_MXFP6_E2M3: *f = {1, 1, 32}; return true;
    case SS_FMT_NVFP6_E2M3: *f = {1, 0, 16}; return true;
    case SS_FMT_NVFP4_B32: *f = {0, 0, 32}; return true;
    case SS_FMT_NVFP4_B64: *f = {0, 0, 64}; return true;
    case SS_FMT_NVFP4_B128: *f = {0, 0, 128}; return true;
    case SS_FMT_NVFP4_B256: *f = {0, 0, 256}; return true;
    default: return false;
  }
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

ss_status launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

// Launch with programmatic stream serialization (PDL): the grid may start
// while the previous kernel in the stream is finishing; the kernel itself
// calls griddepcontrol.wait before touching anything the predecessor
// produces (quant_kernel, sums_kernel).
template <typename Arg>
ss_status launch_pdl(void (*k)(Arg), int grid, int block, cudaStream_t st, const Arg& arg) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k, arg) != cudaSuccess) {
    cudaGetLastError();
    return SS_ERR_CUDA;
  }
  return SS_OK;
}

// ---- amax --------------------------------------------------------------------
int amax_grid(int sms) {
  static const int occ = [] {  // thread-safe one-time query
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ss::amax_kernel, ss::kThreads, 0) != cudaSuccess) {
      cudaGetLastError();
      o = 4;
    }
    return std::max(o, 1);
  }();
  return sms * occ;
}

// Launch the batched amax over `count` tensors into the device slots out[0..count).
ss_status amax_launch(const void* const* in, const int64_t* n, uint32_t* out, int count,
                      bool accumulate, cudaStream_t st, int sms) {
  if (!accumulate && count > 0 && cudaMemsetAsync(out, 0, 4 * (size_t)count, st) != cudaSuccess)
    return SS_ERR_CUDA;
  int i = 0;
  while (i < count) {
    AmaxBatch b;
    std::memset(&b, 0, sizeof(b));
    int64_t chunks = 0;
    for (; i < count && b.n < ss::kMaxTensors; i++) {
      if (n[i] == 0) continue;
      ATensor& t = b.t[b.n++];
      t.in = reinterpret_cast<const uint4*>(in[i]);
      t.nvec = n[i] / 8;
      t.ntail = (int)(n[i] % 8);
      t.chunk0 = chunks;
      t.out = out + i;
      const int64_t full = t.nvec / ss::kAmaxChunk;
      chunks += full + ((t.nvec % ss::kAmaxChunk) || t.ntail ? 1 : 0);
    }
    if (b.n == 0) break;
    b.nchunks = chunks;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, amax_grid(sms)));
    ss::amax_kernel<<<grid, ss::kThreads, 0, st>>>(b);
    if (ss_status s = launch_status()) return s;
  }
  return SS_OK;
}

// ---- quantize kernel variants --------------------------------------------------
typedef void (*QuantKernel)(QuantBatch);

// ri: 0 plain, 1 per-block row index, 2 row-fused tensors (UE4M3 formats only:
// UE8M0 formats take no global scale)
template <int NEG, int POS, int FMT = ss::kFmtNVFP4>
QuantKernel qk(int ri, bool af = false) {
  if constexpr (FMT == ss::kFmtNVFP4) {
    if (af) return ss::quant_kernel<NEG, POS, 0, FMT, true>;
  }
  if constexpr (ss::Fmt<FMT>::SF == 0) {
    if (ri == 2) return ss::quant_kernel<NEG, POS, 2, FMT>;
  }
  return ri ? ss::quant_kernel<NEG, POS, 1, FMT> : ss::quant_kernel<NEG, POS, 0, FMT>;
}

// Other formats: fixed symmetric windows of radius 0..2 (MX formats use two
// offsets in practice), the runtime-window kernel otherwise.
template <int FMT>
QuantKernel qk_small(int fmin, int fmax, int ri) {
  if (fmin == -fmax) {
    switch (fmax) {
      case 0: return qk<0, 0, FMT>(ri);
      case 1: return qk<1, 1, FMT>(ri);
      case 2: return qk<2, 2, FMT>(ri);
      default: break;
    }
  }
  return qk<-1, -1, FMT>(ri);
}

QuantKernel pick_kernel(int fmin, int fmax, int ri, int format, bool af = false) {
  switch (format) {
    case SS_FMT_MXFP4: return qk_small<ss::kFmtMXFP4>(fmin, fmax, ri);
    case SS_FMT_MXFP6_E2M3: return qk_small<ss::kFmtMXFP6E2M3>(fmin, fmax, ri);
    case SS_FMT_NVFP6_E2M3: return qk_small<ss::kFmtNVFP6E2M3>(fmin, fmax, ri);
    case SS_FMT_NVFP4_B32: return qk<-1, -1, ss::kFmtNVFP4B32>(ri);
    case SS_FMT_NVFP4_B64: return qk<-1, -1, ss::kFmtNVFP4B64>(ri);
    case SS_FMT_NVFP4_B128: return qk<-1, -1, ss::kFmtNVFP4B128>(ri);
    case SS_FMT_NVFP4_B256: return qk<-1, -1, ss::kFmtNVFP4B256>(ri);
    default: break;
  }
  if (fmin == -fmax) {
    switch (fmax) {
#define SS_SYM(R) case R: return qk<R, R>(ri, af);
      SS_SYM(0) SS_SYM(1) SS_SYM(2) SS_SYM(3) SS_SYM(4) SS_SYM(5) SS_SYM(6) SS_SYM(7) SS_SYM(8)
      SS_SYM(9) SS_SYM(10) SS_SYM(11) SS_SYM(12) SS_SYM(13) SS_SYM(14) SS_SYM(15) SS_SYM(16)
#undef SS_SYM
      default: break;
    }
  }
  if (fmin == -2 && fmax == 6) return qk<2, 6>(ri, af);  // the paper's production window
  return qk<-1, -1>(ri, af);
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

inline int64_t tasks_of(int64_t nb) { return (nb + ss::kTaskBlocks - 1) / ss::kTaskBlocks; }

int sums_grid(int sms) {
  static const int occ = [] {  // thread-safe one-time query
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ss::sums_kernel, ss::kThreads, 0) != cudaSuccess) {
      cudaGetLastError();
      o = 4;
    }
    return std::max(o, 1);
  }();
  return sms * occ;
}

// The kernels index a tensor's 16-element half-blocks with 32 bits.  Larger
// tensors run as row pieces of at most kPieceMax half-blocks (quantize_core);
// -DSS_MAX_PIECE_BLOCKS (tools / test builds) shrinks the limit so the piece
// path can be checked against the oracle at small sizes.
#ifndef SS_MAX_PIECE_BLOCKS
#define SS_MAX_PIECE_BLOCKS ((1LL << 31) - (1LL << 16))
#endif
constexpr int64_t kPieceMax = SS_MAX_PIECE_BLOCKS;

// Rows per piece of a tensor (0: the tensor cannot be split this way).
int64_t piece_rows(const ss_tensor_io& t) {
  const int64_t hpr = t.cols / 16;
  if (hpr <= 0) return t.rows;
  if (t.rows * hpr <= kPieceMax) return t.rows;
  int64_t r = kPieceMax / hpr;
  if (t.scale_layout == SS_SCALE_SWIZZLED) r -= r % 128;  // pieces start on a 128-row tile band
  return r;
}

ss_status validate_io(const ss_tensor_io& t, int gmode, const FmtInfo& f) {
  if (t.rows < 0 || t.cols < 0 || (t.cols % f.bs) != 0) return SS_ERR_INVALID_ARG;
  const int64_t nb = t.rows * t.cols / 16;
  if (nb > 0 && (!t.in_bf16 || !t.out_codes || !t.out_scales)) return SS_ERR_INVALID_ARG;
  if (gmode == SS_GLOBAL_DEVICE_AMAX && !t.d_amax_bits) return SS_ERR_INVALID_ARG;
  if (gmode == SS_GLOBAL_ROW && nb > 0 && !t.d_global_scale) return SS_ERR_INVALID_ARG;
  if (t.scale_layout != SS_SCALE_LINEAR && t.scale_layout != SS_SCALE_SWIZZLED)
    return SS_ERR_INVALID_ARG;
  if (nb > 0 && piece_rows(t) <= 0) return SS_ERR_INVALID_ARG;  // a row (or 128-row band) over the piece limit
  // E2M1 codes are stored as one 8-B word per 16-element part, E2M3 codes
  // (one byte each) as one 16-B vector
  if (!aligned(t.in_bf16, 16) || !aligned(t.out_codes, f.vf ? 16 : 8) || !aligned(t.out_err, 8) ||
      !aligned(t.d_err_sums, 8) || !aligned(t.d_amax_bits, 4) || !aligned(t.d_global_scale, 4))
    return SS_ERR_ALIGNMENT;
  return SS_OK;
}

int64_t scale_bytes(int64_t rows, int64_t cols, int layout, int bs = 16) {
  const int64_t nbr = cols / bs;
  if (layout == SS_SCALE_SWIZZLED) return ((rows + 127) / 128) * ((nbr + 3) / 4) * 512;
  return rows * nbr;
}

void row_geometry(int64_t cols, uint32_t* nbr, uint32_t* magic, uint32_t* nkt, int bs = 16) {
  *nbr = (uint32_t)std::max<int64_t>(1, cols / bs);
  *magic = (uint32_t)(0xFFFFFFFFu / *nbr);
  *nkt = (*nbr + 3) / 4;
}

int rows_grid(int sms) {
  static const int occ = [] {  // thread-safe one-time query
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ss::rowscale_kernel, ss::kThreads, 0) != cudaSuccess) {
      cudaGetLastError();
      o = 4;
    }
    return std::max(o, 1);
  }();
  return sms * occ;
}

// Per-row global scales of every tensor into its d_global_scale (SS_GLOBAL_ROW).
ss_status rowscale_launch(const ss_tensor_io* io, int count, const std::vector<char>& fused,
                          uint32_t* flags, float numer, cudaStream_t st, int sms) {
  int i = 0;
  while (i < count) {
    ss::RowBatch b;
    std::memset(&b, 0, sizeof(b));
    b.flags = flags;
    b.g_numer = numer;
    int64_t tasks = 0;
    for (; i < count && b.n < ss::kMaxTensors; i++) {
      if (io[i].rows * io[i].cols == 0 || fused[i]) continue;
      ss::RTensor& t = b.t[b.n++];
      t.in = reinterpret_cast<const uint4*>(io[i].in_bf16);
      t.g_row = io[i].d_global_scale;
      t.rows = io[i].rows;
      t.rowvec = (int32_t)(io[i].cols / 8);
      int lpr = 1;
      while (lpr * 2 <= std::min(32, t.rowvec)) lpr *= 2;
      t.lpr = lpr;
      t.task0 = tasks;
      tasks += (t.rows + (32 / lpr) - 1) / (32 / lpr);
    }
    if (b.n == 0) break;
    b.ntasks = tasks;
    const int64_t want = (tasks + ss::kWarps - 1) / ss::kWarps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, rows_grid(sms)));
    ss::rowscale_kernel<<<grid, ss::kThreads, 0, st>>>(b);
    if (ss_status s = launch_status()) return s;
  }
  return SS_OK;
}

// SS_GLOBAL_ROW with the row amax fused into the quantize pass: rows of
// 64..512 half-blocks (1024..8192 elements), where a row is a few work items
// and the rows a whole grid has in flight fit in L2 (<= 4736 warps x 16 KB),
// so the quantize reads after the warp's own amax pass hit L2.  Shorter rows
// would leave lanes idle, longer ones would re-read HBM: those use the
// separate rowscale pass.  Tools-only builds compile -DSS_ROW_FUSION=0 for
// the A/B measurement; the library takes no environment input.
#ifndef SS_ROW_FUSION
#define SS_ROW_FUSION 1
#endif
// SS_GLOBAL_TENSOR, NVFP4, plain layout: the amax pass runs inside the quantize
// launch (quant_kernel<..., AF>); -DSS_AMAX_FUSION=0 (tools-only builds)
// restores the separate amax launch.
#ifndef SS_AMAX_FUSION
#define SS_AMAX_FUSION 1
#endif
// Row-fused scheduling units per row (0 = automatic, ~6 units per warp)
#ifndef SS_ROW_UPR
#define SS_ROW_UPR 0
#endif
inline int64_t amax_units(int64_t nb) { return (2 * nb + ss::kAmaxUnitVecs - 1) / ss::kAmaxUnitVecs; }

// `wide`: the window has >= 4 offsets.  For narrower windows the two-pass path
// (row-scale grid, then the quantize grid launched with PDL) is faster: C3
// r = 0 1792 vs 1719 GB/s, r = 1 1462 vs 1427 (profiles/r01/rowbench_v10.jsonl).
inline bool row_fused(const ss_tensor_io& t, int gmode, bool wide) {
  const int64_t hpr = t.cols / 16;
  return gmode == SS_GLOBAL_ROW && wide && t.rows > 0 && hpr >= ss::kTaskBlocks &&
         hpr <= 8 * ss::kTaskBlocks && SS_ROW_FUSION;
}
// Plain tensors: work items per scheduling unit (one ticket and one error-sum
// partial per unit).  Units of several items amortise the per-unit work
// (ticket, tensor lookup, the FP64 warp sums) when every warp gets many;
// -DSS_IPU_MAX (tools-only builds) caps it.
#ifndef SS_IPU_MAX
#define SS_IPU_MAX 4
#endif
inline int items_per_unit(const ss_tensor_io* io, int count, int sms) {
  int64_t items = 0;
  for (int i = 0; i < count; i++) items += tasks_of(io[i].rows * io[i].cols / 16);
  const int64_t warps = (int64_t)sms * 4 * ss::kWarps;  // ~ the persistent grid's warps
  return (int)std::max<int64_t>(1, std::min<int64_t>(SS_IPU_MAX, items / (warps * 8)));
}
inline int64_t parts_of(const ss_tensor_io& t, int gmode, bool wide, int ipu) {
  const int64_t nb = t.rows * t.cols / 16;
  if (!row_fused(t, gmode, wide)) return (tasks_of(nb) + ipu - 1) / ipu;
  return t.rows * ((t.cols / 16 + ss::kTaskBlocks - 1) / ss::kTaskBlocks);
}
inline int64_t psegs_of(int64_t parts) { return (parts + ss::kSegTasks - 1) / ss::kSegTasks; }

// ---- small single tensors ------------------------------------------------------
// Up to SS_SMALL_MAX_BLOCKS NVFP4 blocks in one tensor go to quant_small_kernel:
// one thread per block over every resident thread, no candidate table
// (DESIGN.md §4.8).  2^19 blocks = 8.4 M elements (C1 = 2^20 blocks: the
// persistent kernel wins at r = 8).
#ifndef SS_SMALL_MAX_BLOCKS
#define SS_SMALL_MAX_BLOCKS (1 << 19)
#endif
constexpr int64_t kSmallMaxBlocks = SS_SMALL_MAX_BLOCKS;
// Trailing amax (§4.2c) for per-tensor-G calls of at least this many elements
// (smaller calls keep the single fused launch); 0 disables it (tools-only A/B)
#ifndef SS_TRAIL_MIN_ELEMS
#define SS_TRAIL_MIN_ELEMS (int64_t(1) << 26)
#endif
constexpr int64_t kTrailMinElems = SS_TRAIL_MIN_ELEMS;

typedef void (*SmallKernel)(ss::SmallParams);
SmallKernel pick_small(int fmin, int fmax) {
  if (fmin == -8 && fmax == 8) return ss::quant_small_kernel<8, 8>;
  if (fmin == -2 && fmax == 6) return ss::quant_small_kernel<2, 6>;
  if (fmin == -1 && fmax == 1) return ss::quant_small_kernel<1, 1>;
  if (fmin == 0 && fmax == 0) return ss::quant_small_kernel<0, 0>;
  return ss::quant_small_kernel<-1, -1>;
}

ss_status small_launch(const ss_tensor_io& t, int fmin, int fmax, int gmode, const uint32_t* amax, float numer,
                       Workspace* ws, cudaStream_t cs, int sms) {
  const int64_t nb = t.rows * t.cols / 16;
  const int64_t chunks = (nb + 255) / 256;
  SmallKernel k = pick_small(fmin, fmax);
  static std::mutex mu;
  static std::map<SmallKernel, int> occ_cache;
  int occ;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ_cache.find(k);
    if (it == occ_cache.end()) {
      int o = 1;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 256, 0) != cudaSuccess) {
        cudaGetLastError();
        o = 1;
      }
      it = occ_cache.emplace(k, std::max(o, 1)).first;
    }
    occ = it->second;
  }
  ss::SmallParams p;
  std::memset(&p, 0, sizeof(p));
  p.in = reinterpret_cast<const uint4*>(t.in_bf16);
  p.nb = nb;
  p.fmin = fmin;
  p.fmax = fmax;
  p.gmode = gmode;
  p.amax = amax;
  p.g_numer = numer;
  p.codes = reinterpret_cast<uint2*>(t.out_codes);
  p.scales = t.out_scales;
  p.err = reinterpret_cast<float2*>(t.out_err);
  p.offsets = t.out_offset;
  p.g_out = t.d_global_scale;
  p.part1 = t.d_err_sums ? ws->part1 : nullptr;
  p.flags = ws->flags;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)sms * occ));
  if (ss_status s = launch_pdl(k, grid, 256, cs, p)) return s;
  if (t.d_err_sums) {  // reduce the per-chunk partials (fixed order) into the tensor's sums
    QuantBatch b;
    std::memset(&b, 0, sizeof(b));
    b.n = 1;
    b.part1 = ws->part1;
    b.part2 = ws->part2;
    b.tick = ws->tick;
    b.t[0].sums = t.d_err_sums;
    b.t[0].part0 = 0;
    b.t[0].npart = (int32_t)chunks;
    b.t[0].seg0 = 0;
    b.nsegs = (chunks + ss::kSegTasks - 1) / ss::kSegTasks;
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(b.nsegs, sums_grid(sms)));
    if (ss_status s = launch_pdl(ss::sums_kernel, g2, ss::kThreads, cs, b)) return s;
  }
  return SS_OK;
}

// The one quantization path behind every entry point.
// The next group's tensors whose local amaxes a sharded step wants while this
// call searches (ss_quantize_nvfp4_batched_next_amax).
// Peer-memory amax exchange of a sharded step.
struct XIn {                  // consumer: G from every rank's slot of this group
  const uint32_t* slots;      // own buffer: the group's first slot (stride kMaxPeers)
  const uint32_t* flags;      // own buffer: the group's flag words [world]
  int world;
  uint32_t epoch;
};
struct XOut {                 // producer: the next group's local amaxes to every rank
  uint32_t* slots[ss::kMaxPeers];  // rank p's buffer: the next group's first slot + this rank
  uint32_t* flags[ss::kMaxPeers];  // rank p's flag word [next group][this rank]
  int world;
  uint32_t epoch;
};

struct NextAmax {
  const void* const* in;
  const int64_t* n;
  int count;
  uint32_t* out;
  const XOut* xo = nullptr;   // also publish them (exchange)
};

ss_status publish_launch(const NextAmax* next, cudaStream_t cs) {
  ss::XPub x;
  std::memset(&x, 0, sizeof(x));
  x.local = next->out;
  x.count = next->count;
  x.world = next->xo->world;
  x.epoch = next->xo->epoch;
  for (int r = 0; r < x.world; r++) {
    x.slots[r] = next->xo->slots[r];
    x.flags[r] = next->xo->flags[r];
  }
  ss::exchange_publish_kernel<<<1, 32, 0, cs>>>(x);
  return launch_status();
}

// Launch decisions of one call (shared by quantize_core and ss_quantize_plan).
struct Plan {
  bool wide;       // >= 4 offsets: the search is ALU-bound (HBM crossover ~3 candidates)
  int ri;          // per-block row index level of the quantize kernel (quant_kernel RI)
  bool af_self;    // SS_GLOBAL_TENSOR: the amax pass inside the quantize launch (§4.2a)
  bool af_next;    // next-group amaxes inside the first quantize launch (§5)
  int small;       // index of the one small tensor for quant_small_kernel (§4.8), or -1
  int n_rowfused;  // tensors whose per-row amax runs inside the quantize pass (§4.4)
};

Plan make_plan(const ss_tensor_io* io, int count, int fmin, int fmax, int gmode, int format,
               const NextAmax* next) {
  Plan p;
  p.wide = fmax - fmin >= 3;
  p.ri = gmode == SS_GLOBAL_ROW ? 1 : 0;
  p.n_rowfused = 0;
  for (int i = 0; i < count; i++) {
    if (io[i].scale_layout == SS_SCALE_SWIZZLED) p.ri = std::max(p.ri, 1);
    if (row_fused(io[i], gmode, p.wide)) {
      p.ri = 2;
      p.n_rowfused++;
    }
  }
  // fused only where the search is ALU-bound and where most of the amax can
  // overlap a search: the first tensor's amax is exposed, so not when it holds
  // most of the elements (a single tensor: the dedicated amax kernel is faster)
  int64_t n_all = 0, n_first = -1;
  int live = -1, nlive = 0;
  for (int i = 0; i < count; i++) {
    const int64_t n = io[i].rows * io[i].cols;
    if (n > 0 && n_first < 0) n_first = n;
    if (n > 0) {
      live = i;
      nlive++;
    }
    n_all += n;
  }
  p.af_self = gmode == SS_GLOBAL_TENSOR && p.ri == 0 && format == SS_FMT_NVFP4 && p.wide &&
              2 * n_first <= n_all && SS_AMAX_FUSION;
  p.af_next = next && next->count > 0 && n_all > 0 && gmode == SS_GLOBAL_DEVICE_AMAX && p.ri == 0 &&
              format == SS_FMT_NVFP4 && SS_AMAX_FUSION;
  p.small = (!p.af_next && nlive == 1 && format == SS_FMT_NVFP4 && p.ri == 0 && !p.af_self &&
             io[live].rows * io[live].cols / 16 <= kSmallMaxBlocks)
                ? live
                : -1;
  return p;
}

// Launch batches of a trailing-amax call (§4.2c): exclusive tensor end index
// per launch, and whether the batch computes its own amax (the amax warps of
// §4.2a, with per-tensor waits) instead of having it folded by the previous
// launch.  Batch 0 holds about 1/64 of the elements and computes its own;
// each later batch at most doubles its predecessor's elements (its amax is
// folded by the predecessor's search warps at up to 4 KiB per 2 KiB work
// item), except that a batch whose first tensor alone is larger (small
// tensors, then a huge one) computes its own too: too few warps would fold
// it.  At most kMaxTensors / 2 tensors per batch, so a launch's own and
// next-batch amax tasks fit QuantBatch::am.  Fewer than two batches (empty
// result) means no trailing amax.
struct TrailPlan {
  std::vector<int> end;
  std::vector<char> self;
};
TrailPlan trail_batches(const ss_tensor_io* io, int count) {
  int64_t n_all = 0;
  for (int i = 0; i < count; i++) n_all += io[i].rows * io[i].cols;
  TrailPlan tp;
  if (count < 2 || kTrailMinElems <= 0 || n_all < kTrailMinElems) return tp;
  int64_t lim = std::max<int64_t>(n_all / 64, 1);
  int i = 0;
  while (i < count) {
    int64_t el = 0;
    int nt = 0;
    bool self = tp.end.empty();
    while (i < count && nt < ss::kMaxTensors / 2) {
      const int64_t n = io[i].rows * io[i].cols;
      if (nt > 0 && (el + n > lim || el + n > (int64_t(1) << 36))) break;  // 32-bit unit indices
      if (nt == 0 && n > lim) self = true;
      el += n;
      nt += n > 0;
      i++;
    }
    tp.end.push_back(i);
    tp.self.push_back(self);
    lim = 2 * std::max<int64_t>(el, 1);
  }
  if (tp.end.size() < 2) tp = TrailPlan();
  return tp;
}

ss_status quantize_core(const ss_tensor_io* io, int count, int f_min, int f_max, int gmode,
                        void* stream, int format = SS_FMT_NVFP4, const NextAmax* next = nullptr,
                        const XIn* xi = nullptr) {
  FmtInfo fi;
  if (!fmt_info(format, &fi)) return SS_ERR_INVALID_ARG;
  if (count < 0 || (count > 0 && !io)) return SS_ERR_INVALID_ARG;
  if (f_min > 0 || f_max < 0) return SS_ERR_INVALID_ARG;
  if (gmode < SS_GLOBAL_NONE || gmode > SS_GLOBAL_ROW) return SS_ERR_INVALID_ARG;
  if (fi.sf == 1 && gmode != SS_GLOBAL_NONE) return SS_ERR_INVALID_ARG;  // UE8M0: no global scale
  if (xi && (gmode != SS_GLOBAL_DEVICE_AMAX || format != SS_FMT_NVFP4)) return SS_ERR_INVALID_ARG;
  for (int i = 0; i < count; i++)  // exchange: G comes from the buffer, no d_amax_bits needed
    if (ss_status s = validate_io(io[i], xi ? SS_GLOBAL_NONE : gmode, fi)) return s;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  if (count == 0 && !(next && next->count > 0)) return SS_OK;
  const int lim = fi.sf ? 254 : 126;
  const int fmin = std::max(f_min, -lim), fmax = std::min(f_max, lim);
  const float numer = ss::global_numer(fi.vf);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);

  Workspace* ws = nullptr;
  if (ss_status s = get_ws(dev, stream, &ws)) return s;
  std::lock_guard<std::mutex> wlk(ws->mu);

  // Row pieces of tensors over the 32-bit half-block index (kPieceMax): each
  // piece is a tensor of its own for the launches, with its tensor's amax
  // slot, G output and window; the first piece also reduces every later
  // piece's error-sum partials (prole 1), the others only write theirs
  // (prole 2).  All pieces of a tensor go into one launch.
  const ss_tensor_io* io0 = io;
  const int count0 = count;
  std::vector<ss_tensor_io> pio;
  std::vector<int> psrc, prole, pnum;
  bool split = false;
  for (int i = 0; i < count0; i++) split |= io0[i].rows * io0[i].cols / 16 > kPieceMax;
  if (split) {
    for (int i = 0; i < count0; i++) {
      const ss_tensor_io& t = io0[i];
      const int64_t pr = piece_rows(t);
      const int np = t.rows * t.cols / 16 > kPieceMax ? (int)((t.rows + pr - 1) / pr) : 1;
      const int64_t nbr = t.cols / fi.bs;
      for (int k = 0; k < np; k++) {
        ss_tensor_io q = t;
        const int64_t r0 = k * pr;
        q.rows = std::min(pr, t.rows - r0);
        if (np > 1) {
          q.in_bf16 = static_cast<const uint8_t*>(t.in_bf16) + r0 * t.cols * 2;
          q.out_codes = t.out_codes + r0 * t.cols / (fi.vf ? 1 : 2);
          q.out_scales = t.out_scales + (t.scale_layout == SS_SCALE_SWIZZLED
                                             ? (r0 / 128) * ((nbr + 3) / 4) * 512 : r0 * nbr);
          if (t.out_err) q.out_err = t.out_err + 2 * r0 * nbr;
          if (t.out_offset) q.out_offset = t.out_offset + r0 * nbr;
          if (gmode == SS_GLOBAL_ROW && t.d_global_scale) q.d_global_scale = t.d_global_scale + r0;
        }
        pio.push_back(q);
        psrc.push_back(i);
        prole.push_back(np == 1 ? 0 : (k == 0 ? 1 : 2));
        pnum.push_back(k == 0 ? np : 0);
      }
    }
    io = pio.data();
    count = (int)pio.size();
  }

  Plan pl = make_plan(io, count, fmin, fmax, gmode, format, next);
  if (xi) pl.small = -1;  // the exchange reads G from the buffer: persistent kernel only
  const bool wide = pl.wide, af_self = pl.af_self && !split, af_next = pl.af_next && !split;
  const int ri = pl.ri;
  if (next && next->count > 0) {
    if (af_next) {
      if (cudaMemsetAsync(next->out, 0, 4 * (size_t)next->count, reinterpret_cast<cudaStream_t>(stream)) !=
          cudaSuccess)
        return SS_ERR_CUDA;
    } else {  // not fusable here: a plain amax launch first (and its publication)
      if (ss_status s = amax_launch(next->in, next->n, next->out, next->count, false,
                                    reinterpret_cast<cudaStream_t>(stream), info.sms))
        return s;
      if (next->xo)
        if (ss_status s = publish_launch(next, reinterpret_cast<cudaStream_t>(stream))) return s;
    }
  }
  const bool af = af_self || af_next;

  const int ipu = items_per_unit(io, count, info.sms);
  // sizes of the largest launch (workspace grown once, before any launch)
  int64_t max_tasks = 0, max_segs = 0;
  bool any_sums = false;
  {
    int64_t tk = 0, gr = 0;
    int in_batch = 0;
    for (int i = 0; i < count; i++) {
      const int64_t nb = io[i].rows * io[i].cols / 16;
      if (nb == 0) continue;
      if (in_batch == ss::kMaxTensors && !split) {  // split: launches keep pieces together, size for all
        max_tasks = std::max(max_tasks, tk);
        max_segs = std::max(max_segs, gr);
        tk = gr = 0;
        in_batch = 0;
      }
      tk += parts_of(io[i], gmode, wide, ipu);
      gr += psegs_of(parts_of(io[i], gmode, wide, ipu));
      in_batch++;
      any_sums |= io[i].d_err_sums != nullptr;
    }
    max_tasks = std::max(max_tasks, tk);
    max_segs = std::max(max_segs, gr);
  }
  if (any_sums) {
    if (ss_status s = grow_dev(&ws->part1, &ws->part1_cap, max_tasks, false, cs)) return s;
    if (ss_status s = grow_dev(&ws->part2, &ws->part2_cap, max_segs, false, cs)) return s;
  }

  // SS_GLOBAL_TENSOR: the amax pass of every tensor first (a2)
  std::vector<const uint32_t*> amax(count, nullptr);
  if (gmode == SS_GLOBAL_TENSOR) {
    if (ss_status s = grow_dev(&ws->amax, &ws->amax_cap, std::max(count, count0), false, cs)) return s;
    std::vector<const void*> ins(count0);
    std::vector<int64_t> ns(count0);
    for (int i = 0; i < count0; i++) {  // the whole tensors (a piece uses its tensor's slot)
      ins[i] = io0[i].in_bf16;
      ns[i] = io0[i].rows * io0[i].cols;
    }
    for (int i = 0; i < count; i++) amax[i] = ws->amax + (split ? psrc[i] : i);
    if (af) {  // the quantize launches fold their amax units into zeroed slots
      if (cudaMemsetAsync(ws->amax, 0, 4 * (size_t)count, cs) != cudaSuccess) return SS_ERR_CUDA;
    } else if (ss_status s = amax_launch(ins.data(), ns.data(), ws->amax, count0, false, cs, info.sms)) {
      return s;
    }
  } else if (gmode == SS_GLOBAL_DEVICE_AMAX) {
    for (int i = 0; i < count; i++) amax[i] = io[i].d_amax_bits;
  } else if (gmode == SS_GLOBAL_ROW) {
    std::vector<char> fused(count);
    for (int i = 0; i < count; i++) fused[i] = row_fused(io[i], gmode, wide);
    if (ss_status s = rowscale_launch(io, count, fused, ws->flags, numer, cs, info.sms)) return s;
  }
  // swizzled scales: zero the padding of partial 128x4 tiles first
  for (int i = 0; i < count; i++) {
    const ss_tensor_io& t = io[i];
    if (t.scale_layout == SS_SCALE_SWIZZLED && t.rows * t.cols > 0 &&
        (t.rows % 128 != 0 || (t.cols / fi.bs) % 4 != 0) &&
        cudaMemsetAsync(t.out_scales, 0, (size_t)scale_bytes(t.rows, t.cols, t.scale_layout, fi.bs), cs) !=
            cudaSuccess)
      return SS_ERR_CUDA;
  }

  // one small NVFP4 tensor: one thread per block (quant_small_kernel)
  if (pl.small >= 0) {
    const int live = pl.small;
    for (int i = 0; i < count; i++)
      if (i != live && io[i].d_err_sums && cudaMemsetAsync(io[i].d_err_sums, 0, 16, cs) != cudaSuccess)
        return SS_ERR_CUDA;
    return small_launch(io[live], fmin, fmax, gmode == SS_GLOBAL_NONE ? 0 : 1, amax[live], numer, ws, cs,
                        info.sms);
  }

  QuantKernel k = pick_kernel(fmin, fmax, ri, format, af);
  const int64_t slots = (int64_t)info.sms * occupancy(k);
  const QuantKernel k_plain = af_next ? pick_kernel(fmin, fmax, ri, format, false) : k;
  // Trailing amax (§4.2c): a per-tensor-G call of several tensors runs as a
  // chain of launches whose batches grow geometrically; launch 0 computes its
  // own (small) batch's amax with the amax warps, and every launch's search
  // warps also fold the NEXT batch's amax after each scheduling unit, so no
  // later launch waits for an amax and the amax reads spread over the search.
  const TrailPlan tplan = af_self && !xi ? trail_batches(io, count) : TrailPlan();
  const std::vector<int>& bend = tplan.end;
  const bool trail = bend.size() > 1;
  size_t launch_idx = 0;
  bool next_done = false;
  int i = 0;
  while (i < count) {
    QuantBatch b;
    std::memset(&b, 0, sizeof(b));
    b.fmin = fmin;
    b.fmax = fmax;
    b.gmode = xi ? 3 : (gmode == SS_GLOBAL_NONE ? 0 : (gmode == SS_GLOBAL_ROW ? 2 : 1));
    if (xi) {
      b.xw = xi->world;
      b.xin = xi->slots;
      b.xin_flag = xi->flags;
      b.xepoch_in = xi->epoch;
    }
    b.g_numer = numer;
    b.ipu = ipu;
    b.part1 = ws->part1;
    b.part2 = ws->part2;
    b.tick = ws->tick;
    b.ctr = ws->ctr;
#if defined(SS_COUNT_EVALS) || defined(SS_AF_TRACE)
    {
      std::lock_guard<std::mutex> lk(g_mu);
      if (!g_evals && cudaMalloc(&g_evals, 32) == cudaSuccess) cudaMemset(g_evals, 0, 32);
    }
    b.evals = g_evals;
#endif
    b.flags = ws->flags;
    b.done = ws->done;
    bool sums = false;
    int64_t tk = 0, gr = 0, pk = 0;
    const bool self_amax = af_self && (!trail || tplan.self[launch_idx]);
    for (; i < count && b.n < ss::kMaxTensors && (!trail || i < bend[launch_idx]); i++) {
      const ss_tensor_io& t = io[i];
      const int64_t nb = t.rows * t.cols / 16;
      if (nb == 0) {
        if (t.d_err_sums && cudaMemsetAsync(t.d_err_sums, 0, 16, cs) != cudaSuccess) return SS_ERR_CUDA;
        continue;
      }
      const bool rf = row_fused(t, gmode, wide);
      int hpr = 0, cpr = 0, upr = 0, cpu = 0;
      int64_t units = (tasks_of(nb) + ipu - 1) / ipu;
      if (rf) {
        // units of `cpu` chunks: enough units for ~6 per warp of the grid, so
        // the dynamic schedule balances; each unit re-reads its row from L2
        // for the row amax
        hpr = (int)(t.cols / 16);
        cpr = (hpr + ss::kTaskBlocks - 1) / ss::kTaskBlocks;
        const int64_t want = (6 * slots * ss::kWarps + t.rows - 1) / t.rows;
        upr = (int)std::min<int64_t>(cpr, std::max<int64_t>(1, want));
        if (SS_ROW_UPR > 0) upr = std::max(1, std::min(cpr, (int)SS_ROW_UPR));
        cpu = (cpr + upr - 1) / upr;
        upr = (cpr + cpu - 1) / cpu;
        units = t.rows * upr;
      }
      const int64_t parts = parts_of(t, gmode, wide, ipu);
      // a split tensor's pieces: all in this launch, the first reduces all partials
      const int role = split ? prole[i] : 0;
      int64_t all_units = units, all_parts = parts;
      if (role == 1) {
        all_units = all_parts = 0;
        for (int k = 0; k < pnum[i]; k++) {
          all_units += (tasks_of(io[i + k].rows * io[i + k].cols / 16) + ipu - 1) / ipu;
          all_parts += parts_of(io[i + k], gmode, wide, ipu);
        }
      }
      // the kernel indexes units, partials and amax units with 32 bits: close the batch before overflow
      const int64_t au = self_amax ? amax_units(nb) : 0;
      if (role != 2 && b.n > 0 &&
          (tk + all_units > (int64_t)INT32_MAX - ss::kCounters || pk + all_parts > (int64_t)INT32_MAX ||
           b.namax + au > (int64_t)INT32_MAX - ss::kWarps * 65536 ||
           (role == 1 && b.n + pnum[i] > ss::kMaxTensors)))
        break;
      QTensor& q = b.t[b.n++];
      q.in = reinterpret_cast<const uint8_t*>(t.in_bf16);
      q.codes = reinterpret_cast<uint2*>(t.out_codes);
      q.scales = t.out_scales;
      q.err = reinterpret_cast<float2*>(t.out_err);
      q.offsets = t.out_offset;
      q.sums = t.d_err_sums;
      q.g_out = t.d_global_scale;
      q.amax = amax[i];
      q.g_row = (gmode == SS_GLOBAL_ROW && !rf) ? t.d_global_scale : nullptr;
      if (gmode == SS_GLOBAL_ROW && !rf) q.g_out = nullptr;  // rowscale_kernel wrote G_r
      row_geometry(t.cols, &q.nbr, &q.nbr_magic, &q.nkt, fi.bs);
      q.swz = t.scale_layout == SS_SCALE_SWIZZLED;
      q.nb = nb;
      q.hpr = (int16_t)hpr;
      q.cpr = (int16_t)cpr;
      q.upr = (int16_t)upr;
      q.cpu = (int16_t)cpu;
      q.task0 = tk;
      q.part0 = (int32_t)pk;
      q.npart = (int32_t)(role == 0 ? parts : (role == 1 ? all_parts : 0));
      q.seg0 = gr;
      if (self_amax) {  // this tensor's own amax, counted into done[b.n - 1]
        ss::AmaxTask& a = b.am[b.nam++];
        a.in = reinterpret_cast<const uint4*>(t.in_bf16);
        a.nvec = 2 * nb;
        a.slot = const_cast<uint32_t*>(amax[i]);
        a.a0 = b.namax;
        a.done = b.n - 1;
      }
      q.na = (int32_t)au;
      q.xslot = split ? psrc[i] : i;
      b.namax += (int32_t)au;
      tk += units;
      pk += parts;
      gr += psegs_of(q.npart);
      sums |= t.d_err_sums != nullptr;
    }
    if (b.n == 0) break;
    bool publish_after = false;
    if (af_next && !next_done) {  // the next group's shards: local amaxes, nobody waits
      const int32_t a_first = b.namax;
      for (int j = 0; j < next->count; j++) {
        const int64_t nv = next->n[j] / 8;
        if (nv == 0) continue;
        ss::AmaxTask& a = b.am[b.nam++];
        a.in = reinterpret_cast<const uint4*>(next->in[j]);
        a.nvec = nv;
        a.slot = next->out + j;
        a.a0 = b.namax;
        a.done = -1;
        b.namax += (int32_t)((nv + ss::kAmaxUnitVecs - 1) / ss::kAmaxUnitVecs);
      }
      if (next->xo) {  // exchange: the warp finishing the last next-group unit publishes
        b.xunits_out = b.namax - a_first;
        b.xcount_out = next->count;
        b.xlocal = next->out;
        b.xw = next->xo->world;
        b.xepoch_out = next->xo->epoch;
        for (int r = 0; r < next->xo->world; r++) {
          b.xout[r] = next->xo->slots[r];
          b.xout_flag[r] = next->xo->flags[r];
        }
        publish_after = b.xunits_out == 0;  // no local next-group elements: publish the zeros after
      }
      next_done = true;
    }
    if (trail && launch_idx + 1 < bend.size() && !tplan.self[launch_idx + 1]) {  // the next batch's amax, folded here
      b.tr0 = b.nam;
      for (int j = bend[launch_idx]; j < bend[launch_idx + 1]; j++) {
        const int64_t nv = 2 * (io[j].rows * io[j].cols / 16);
        if (nv == 0) continue;
        ss::AmaxTask& a = b.am[b.nam++];
        a.in = reinterpret_cast<const uint4*>(io[j].in_bf16);
        a.nvec = nv;
        a.slot = const_cast<uint32_t*>(amax[j]);
        a.a0 = b.ntrail;
        a.done = -1;
        b.ntrail += (int32_t)((nv + ss::kTrailVecs - 1) / ss::kTrailVecs);
      }
      b.tpu = (int32_t)((b.ntrail + tk - 1) / tk);
    }
    launch_idx++;
    b.ntasks = tk;
    b.nsegs = gr;
    const int64_t want = (tk + ss::kWarps - 1) / ss::kWarps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, slots));
    // later launches of a next-amax call carry no amax tasks: the plain kernel
    if (ss_status s = launch_pdl(b.nam ? k : (af_self ? k : k_plain), grid, ss::kThreads, cs, b)) return s;
    if (publish_after)
      if (ss_status s = publish_launch(next, cs)) return s;
    if (sums) {
      const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(gr, sums_grid(info.sms)));
      if (ss_status s = launch_pdl(ss::sums_kernel, g2, ss::kThreads, cs, b)) return s;
    }
  }
  return SS_OK;
}

ss_tensor_io io_from_args(const ss_quant_args* a) {
  ss_tensor_io t;
  std::memset(&t, 0, sizeof(t));
  t.in_bf16 = a->in_bf16;
  t.rows = a->rows;
  t.cols = a->cols;
  t.d_amax_bits = a->d_amax_bits;
  t.out_codes = a->out_codes;
  t.out_scales = a->out_scales;
  t.out_err = a->out_err;
  t.out_offset = a->out_offset;
  t.d_err_sums = a->d_err_sums;
  t.d_global_scale = a->d_global_scale;
  t.scale_layout = a->scale_layout;
  return t;
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

// Ring of whole-tensor device slots for the batched host pipeline.
struct HostRing {
  static constexpr int kSlots = 3;
  void* mem = nullptr;
  size_t slot_bytes = 0;
  uint32_t* amax = nullptr;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t in_ready[kSlots], out_ready[kSlots], slot_free[kSlots];
};
std::mutex g_ring_mu;
std::map<int, HostRing> g_rings;

// ---- generic ExMy block formats ----------------------
bool gen_fmt(const ss_gen_format* g, ss::GenFmt* f) {
  if (!g) return false;
  const int ve = g->value_e, vm = g->value_m, se = g->scale_e, sm = g->scale_m;
  if (ve < 1 || vm < 0 || ve + vm > 7 || se < 1 || sm < 0 || se + sm > 8 || (sm > 0 && se > 7))
    return false;
  if (g->block != 16 && g->block != 32) return false;
  f->ve = ve;
  f->vm = vm;
  f->se = se;
  f->sm = sm;
  const int vbias = (1 << (ve - 1)) - 1;
  f->vemin = 1 - vbias;
  f->vmax = (float)std::ldexp((double)((2 << vm) - 1), (1 << ve) - 1 - vbias - vm);
  f->kinv = 1.0f / f->vmax;  // RN(1/vmax), binary32 division (R8)
  f->sbias = (1 << (se - 1)) - 1;
  f->semin = 1 - f->sbias;
  f->smaxc = (1 << (se + sm)) - 2;
  if (sm == 0) {
    f->smax = (float)std::ldexp(1.0, f->smaxc - f->sbias);
  } else {
    const int E = f->smaxc >> sm, M = f->smaxc & ((1 << sm) - 1);
    f->smax = (float)std::ldexp((double)((1 << sm) + M), E - f->sbias - sm);
  }
  return true;
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

int ss_version(void) { return 500; }

int64_t ss_scale_bytes(int64_t rows, int64_t cols, int scale_layout) {
  if (rows < 0 || cols < 0 || cols % 16 != 0) return -1;
  if (scale_layout != SS_SCALE_LINEAR && scale_layout != SS_SCALE_SWIZZLED) return -1;
  return scale_bytes(rows, cols, scale_layout);
}

ss_status ss_tensor_amax(const void* in_bf16, int64_t n, uint32_t* d_amax_bits, int accumulate,
                         void* stream) {
  return ss_tensor_amax_batched(&in_bf16, &n, 1, d_amax_bits, accumulate, stream);
}

ss_status ss_tensor_amax_batched(const void* const* in_bf16, const int64_t* n, int count,
                                 uint32_t* d_amax_bits, int accumulate, void* stream) {
  if (count < 0 || (count > 0 && (!in_bf16 || !n || !d_amax_bits))) return SS_ERR_INVALID_ARG;
  for (int i = 0; i < count; i++) {
    if (n[i] < 0 || (n[i] > 0 && !in_bf16[i])) return SS_ERR_INVALID_ARG;
    if (!aligned(in_bf16[i], 16)) return SS_ERR_ALIGNMENT;
  }
  if (!aligned(d_amax_bits, 4)) return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  return amax_launch(in_bf16, n, d_amax_bits, count, accumulate != 0,
                     reinterpret_cast<cudaStream_t>(stream), info.sms);
}

ss_status ss_quantize_nvfp4(const void* in_bf16, int64_t rows, int64_t cols, int radius,
                            int global_scale_mode, uint8_t* out_codes, uint8_t* out_scales,
                            float* out_err, void* stream) {
  if (radius < 0) return SS_ERR_INVALID_ARG;
  if (global_scale_mode != SS_GLOBAL_NONE && global_scale_mode != SS_GLOBAL_TENSOR)
    return SS_ERR_INVALID_ARG;
  ss_tensor_io t;
  std::memset(&t, 0, sizeof(t));
  t.in_bf16 = in_bf16;
  t.rows = rows;
  t.cols = cols;
  t.out_codes = out_codes;
  t.out_scales = out_scales;
  t.out_err = out_err;
  const int r = std::min(radius, 126);
  return quantize_core(&t, 1, -r, r, global_scale_mode, stream);
}

ss_status ss_quantize_nvfp4_ex(const ss_quant_args* a) {
  if (!a) return SS_ERR_INVALID_ARG;
  ss_tensor_io t = io_from_args(a);
  return quantize_core(&t, 1, a->f_min, a->f_max, a->global_scale_mode, a->stream, a->format);
}

ss_status ss_quantize_batched_fmt(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                                  int global_scale_mode, int format, void* stream) {
  return quantize_core(tensors, count, f_min, f_max, global_scale_mode, stream, format);
}

int64_t ss_scale_bytes_fmt(int64_t rows, int64_t cols, int scale_layout, int format) {
  FmtInfo f;
  if (!fmt_info(format, &f) || rows < 0 || cols < 0 || cols % f.bs != 0) return -1;
  if (scale_layout != SS_SCALE_LINEAR && scale_layout != SS_SCALE_SWIZZLED) return -1;
  return scale_bytes(rows, cols, scale_layout, f.bs);
}

int64_t ss_code_bytes(int64_t rows, int64_t cols, int format) {
  FmtInfo f;
  if (!fmt_info(format, &f) || rows < 0 || cols < 0 || cols % f.bs != 0) return -1;
  return f.vf ? rows * cols : rows * cols / 2;
}

ss_status ss_quantize_nvfp4_batched(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                                    int global_scale_mode, void* stream) {
  return quantize_core(tensors, count, f_min, f_max, global_scale_mode, stream);
}

ss_status ss_quantize_nvfp4_batched_next_amax(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                                              const void* const* next_in, const int64_t* next_n,
                                              int next_count, uint32_t* next_amax_bits, void* stream) {
  if (next_count < 0 || next_count > ss::kMaxTensors ||
      (next_count > 0 && (!next_in || !next_n || !next_amax_bits)))
    return SS_ERR_INVALID_ARG;
  for (int j = 0; j < next_count; j++) {
    if (next_n[j] < 0 || next_n[j] % 16 != 0 || (next_n[j] > 0 && !next_in[j])) return SS_ERR_INVALID_ARG;
    if (!aligned(next_in[j], 16)) return SS_ERR_ALIGNMENT;
  }
  if (!aligned(next_amax_bits, 4)) return SS_ERR_ALIGNMENT;
  NextAmax nx{next_in, next_n, next_count, next_amax_bits};
  return quantize_core(tensors, count, f_min, f_max, SS_GLOBAL_DEVICE_AMAX, stream, SS_FMT_NVFP4, &nx);
}

int64_t ss_exchange_bytes(int max_tensors, int max_groups) {
  if (max_tensors < 1 || max_groups < 1) return 0;
  return 4 * (2 * (int64_t)max_tensors * ss::kMaxPeers + (int64_t)max_groups * ss::kMaxPeers);
}

ss_status ss_exchange_init(void* d_buf, int max_tensors, int max_groups, void* stream) {
  const int64_t bytes = ss_exchange_bytes(max_tensors, max_groups);
  if (!d_buf || bytes <= 0 || !aligned(d_buf, 4)) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  return cudaMemsetAsync(d_buf, 0, (size_t)bytes, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SS_OK : SS_ERR_CUDA;
}

ss_status ss_exchange_alloc(int max_tensors, int max_groups, void** d_buf) {
  const int64_t bytes = ss_exchange_bytes(max_tensors, max_groups);
  if (!d_buf || bytes <= 0) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  *d_buf = nullptr;
  if (cudaMalloc(d_buf, (size_t)bytes) != cudaSuccess) return SS_ERR_CUDA;
  if (cudaMemset(*d_buf, 0, (size_t)bytes) != cudaSuccess) return SS_ERR_CUDA;  // synchronous: ready for peers
  return SS_OK;
}

ss_status ss_exchange_free(void* d_buf) {
  if (!d_buf) return SS_ERR_INVALID_ARG;
  return cudaFree(d_buf) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

ss_status ss_ipc_handle(const void* d_ptr, void* handle) {
  if (!d_ptr || !handle) return SS_ERR_INVALID_ARG;
  static_assert(sizeof(cudaIpcMemHandle_t) == SS_IPC_HANDLE_BYTES, "IPC handle size");
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)) != cudaSuccess) return SS_ERR_CUDA;
  std::memcpy(handle, &h, sizeof(h));
  return SS_OK;
}

ss_status ss_ipc_open(const void* handle, void** d_ptr) {
  if (!handle || !d_ptr) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return SS_ERR_CUDA;
  return SS_OK;
}

ss_status ss_ipc_close(void* d_ptr) {
  if (!d_ptr) return SS_ERR_INVALID_ARG;
  return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

}  // extern "C"

namespace {
// Buffer geometry (ss.h): words [2][max_tensors][kMaxPeers] of amax slots
// (step parity, group tensor, rank), then [max_groups][kMaxPeers] flags.
bool exchange_ok(const ss_exchange* x, const ss_exchange_group* g, int count) {
  if (!x || !g || x->world < 1 || x->world > ss::kMaxPeers || x->rank < 0 || x->rank >= x->world) return false;
  if (x->max_tensors < 1 || x->max_groups < 1 || g->epoch == 0) return false;
  if (g->group < 0 || g->group >= x->max_groups || g->slot0 < 0 || g->count != count ||
      g->slot0 + count > x->max_tensors)
    return false;
  for (int r = 0; r < x->world; r++)
    if (!x->buf[r] || !aligned(x->buf[r], 4)) return false;
  return true;
}
uint32_t* ex_slots(const ss_exchange* x, int r, const ss_exchange_group* g) {
  return x->buf[r] + ((int64_t)(g->epoch & 1u) * x->max_tensors + g->slot0) * ss::kMaxPeers;
}
uint32_t* ex_flags(const ss_exchange* x, int r, int group) {
  return x->buf[r] + 2 * (int64_t)x->max_tensors * ss::kMaxPeers + (int64_t)group * ss::kMaxPeers;
}
void make_xout(const ss_exchange* x, const ss_exchange_group* g, XOut* o) {
  std::memset(o, 0, sizeof(*o));
  o->world = x->world;
  o->epoch = g->epoch;
  for (int r = 0; r < x->world; r++) {
    o->slots[r] = ex_slots(x, r, g) + x->rank;
    o->flags[r] = ex_flags(x, r, g->group) + x->rank;
  }
}
}  // namespace

extern "C" {

ss_status ss_exchange_publish(const ss_exchange* x, const ss_exchange_group* g, const uint32_t* d_local_amax,
                              void* stream) {
  if (!x || !g || !exchange_ok(x, g, g->count) || (g->count > 0 && !d_local_amax)) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  XOut o;
  make_xout(x, g, &o);
  NextAmax nx{nullptr, nullptr, g->count, const_cast<uint32_t*>(d_local_amax), &o};
  return publish_launch(&nx, reinterpret_cast<cudaStream_t>(stream));
}

ss_status ss_quantize_nvfp4_exchange(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                                     const ss_exchange* x, const ss_exchange_group* g_in,
                                     const void* const* next_in, const int64_t* next_n, int next_count,
                                     uint32_t* next_local_amax, const ss_exchange_group* g_next,
                                     void* stream) {
  if (!exchange_ok(x, g_in, count)) return SS_ERR_INVALID_ARG;
  if (next_count < 0 || (next_count > 0 && (!next_in || !next_n || !next_local_amax || !g_next)) ||
      next_count > ss::kMaxTensors)
    return SS_ERR_INVALID_ARG;
  if (next_count > 0 && !exchange_ok(x, g_next, next_count)) return SS_ERR_INVALID_ARG;
  for (int j = 0; j < next_count; j++)
    if (next_n[j] < 0 || next_n[j] % 8 != 0 || (next_n[j] > 0 && !aligned(next_in[j], 16)))
      return SS_ERR_INVALID_ARG;
  XIn xi;
  xi.slots = ex_slots(x, x->rank, g_in);
  xi.flags = ex_flags(x, x->rank, g_in->group);
  xi.world = x->world;
  xi.epoch = g_in->epoch;
  XOut o;
  if (next_count > 0) make_xout(x, g_next, &o);
  NextAmax nx{next_in, next_n, next_count, next_local_amax, next_count > 0 ? &o : nullptr};
  return quantize_core(tensors, count, f_min, f_max, SS_GLOBAL_DEVICE_AMAX, stream, SS_FMT_NVFP4,
                       next_count > 0 ? &nx : nullptr, &xi);
}

ss_status ss_quantize_plan(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                          int global_scale_mode, int format, ss_plan* out) {
  FmtInfo fi;
  if (!out || !fmt_info(format, &fi)) return SS_ERR_INVALID_ARG;
  if (count < 0 || (count > 0 && !tensors)) return SS_ERR_INVALID_ARG;
  if (f_min > 0 || f_max < 0) return SS_ERR_INVALID_ARG;
  if (global_scale_mode < SS_GLOBAL_NONE || global_scale_mode > SS_GLOBAL_ROW) return SS_ERR_INVALID_ARG;
  if (fi.sf == 1 && global_scale_mode != SS_GLOBAL_NONE) return SS_ERR_INVALID_ARG;
  for (int i = 0; i < count; i++)
    if (ss_status s = validate_io(tensors[i], global_scale_mode, fi)) return s;
  const int lim = fi.sf ? 254 : 126;
  const int fmin = std::max(f_min, -lim), fmax = std::min(f_max, lim);
  const Plan pl = make_plan(tensors, count, fmin, fmax, global_scale_mode, format, nullptr);
  int live = 0, plain_rows = 0;
  for (int i = 0; i < count; i++) {
    if (tensors[i].rows * tensors[i].cols == 0) continue;
    live++;
    if (global_scale_mode == SS_GLOBAL_ROW && !row_fused(tensors[i], global_scale_mode, pl.wide)) plain_rows++;
  }
  const int per = ss::kMaxTensors;
  int launches = 0;
  if (global_scale_mode == SS_GLOBAL_TENSOR && !pl.af_self) launches += (live + per - 1) / per;  // amax_kernel
  if (global_scale_mode == SS_GLOBAL_ROW) launches += (plain_rows + per - 1) / per;              // rowscale_kernel
  bool split = false;  // tensors over the piece limit run as row pieces, never with the fused amax
  for (int i = 0; i < count; i++) split |= tensors[i].rows * tensors[i].cols / 16 > kPieceMax;
  const std::vector<int> bend = pl.af_self && !split ? trail_batches(tensors, count).end : std::vector<int>();
  if (pl.small >= 0) {
    launches += 1 + (tensors[pl.small].d_err_sums ? 1 : 0);  // quant_small_kernel (+ sums_kernel)
  } else if (bend.size() > 1) {  // trailing amax: one quantize launch (+ sums_kernel) per batch
    int i0 = 0;
    for (const int e : bend) {
      bool live_b = false, sums = false;
      for (int i = i0; i < e; i++) {
        live_b |= tensors[i].rows * tensors[i].cols > 0;
        sums |= tensors[i].rows * tensors[i].cols > 0 && tensors[i].d_err_sums != nullptr;
      }
      if (live_b) launches += 1 + (sums ? 1 : 0);
      i0 = e;
    }
  } else {
    int k = 0;
    bool sums = false;
    for (int i = 0; i < count; i++) {  // batches of 128 live tensors: quant_kernel (+ sums_kernel)
      if (tensors[i].rows * tensors[i].cols == 0) continue;
      sums |= tensors[i].d_err_sums != nullptr;
      if (++k == per) {
        launches += 1 + (sums ? 1 : 0);
        k = 0;
        sums = false;
      }
    }
    if (k) launches += 1 + (sums ? 1 : 0);
  }
  out->amax_fused = pl.af_self && !split ? 1 : 0;
  out->trail_batches = bend.size() > 1 ? (int)bend.size() : 0;
  out->small_path = pl.small >= 0 ? 1 : 0;
  out->row_fused = pl.n_rowfused;
  out->launches = launches;
  return SS_OK;
}

ss_status ss_dequantize_nvfp4_ex(const ss_dequant_args* a) {
  if (!a) return SS_ERR_INVALID_ARG;
  FmtInfo fi;
  if (!fmt_info(a->format, &fi)) return SS_ERR_INVALID_ARG;
  if (a->rows < 0 || a->cols < 0 || a->cols % fi.bs != 0) return SS_ERR_INVALID_ARG;
  if (a->scale_layout != SS_SCALE_LINEAR && a->scale_layout != SS_SCALE_SWIZZLED)
    return SS_ERR_INVALID_ARG;
  const int64_t nb = a->rows * a->cols / 16;
  if (nb > 0 && (!a->codes || !a->scales || !a->out_bf16)) return SS_ERR_INVALID_ARG;
  if (a->g_per_row && nb > 0 && !a->d_global_scale) return SS_ERR_INVALID_ARG;
  ss_tensor_io shape;
  std::memset(&shape, 0, sizeof(shape));
  shape.rows = a->rows;
  shape.cols = a->cols;
  shape.scale_layout = a->scale_layout;
  const int64_t pr = piece_rows(shape);  // row pieces over the 32-bit half-block index
  if (nb > 0 && pr <= 0) return SS_ERR_INVALID_ARG;
  if (!aligned(a->codes, fi.vf ? 16 : 8) || !aligned(a->out_bf16, 16)) return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  if (nb == 0) return SS_OK;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(a->stream);
  const int64_t nbr = a->cols / fi.bs;
  for (int64_t r0 = 0; r0 < a->rows; r0 += pr) {
    const int64_t rows = std::min(pr, a->rows - r0);
    ss::DequantParams p;
    p.codes = a->codes + r0 * a->cols / (fi.vf ? 1 : 2);
    p.scales = a->scales + (a->scale_layout == SS_SCALE_SWIZZLED ? (r0 / 128) * ((nbr + 3) / 4) * 512 : r0 * nbr);
    p.nb = rows * a->cols / 16;
    p.g = a->d_global_scale && a->g_per_row ? a->d_global_scale + r0 : a->d_global_scale;
    p.g_per_row = a->g_per_row;
    row_geometry(a->cols, &p.nbr, &p.nbr_magic, &p.nkt, fi.bs);
    p.swz = a->scale_layout == SS_SCALE_SWIZZLED;
    p.out = reinterpret_cast<uint4*>(static_cast<uint8_t*>(a->out_bf16) + r0 * a->cols * 2);
    const int64_t want = (p.nb + 255) / 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)info.sms * 8));
    switch (a->format) {
      case SS_FMT_MXFP4: ss::dequant_kernel<ss::kFmtMXFP4><<<grid, 256, 0, cs>>>(p); break;
      case SS_FMT_MXFP6_E2M3: ss::dequant_kernel<ss::kFmtMXFP6E2M3><<<grid, 256, 0, cs>>>(p); break;
      case SS_FMT_NVFP6_E2M3: ss::dequant_kernel<ss::kFmtNVFP6E2M3><<<grid, 256, 0, cs>>>(p); break;
      case SS_FMT_NVFP4_B32: ss::dequant_kernel<ss::kFmtNVFP4B32><<<grid, 256, 0, cs>>>(p); break;
      case SS_FMT_NVFP4_B64: ss::dequant_kernel<ss::kFmtNVFP4B64><<<grid, 256, 0, cs>>>(p); break;
      case SS_FMT_NVFP4_B128: ss::dequant_kernel<ss::kFmtNVFP4B128><<<grid, 256, 0, cs>>>(p); break;
      case SS_FMT_NVFP4_B256: ss::dequant_kernel<ss::kFmtNVFP4B256><<<grid, 256, 0, cs>>>(p); break;
      default: ss::dequant_kernel<ss::kFmtNVFP4><<<grid, 256, 0, cs>>>(p); break;
    }
    if (ss_status s = launch_status()) return s;
  }
  return SS_OK;
}

ss_status ss_quantize_nvfp4_f32(const float* in, int64_t rows, int64_t cols, int f_min, int f_max,
                                const float* d_global_scale, uint8_t* out_codes, uint8_t* out_scales,
                                float* out_err, int8_t* out_offset, void* stream) {
  if (rows < 0 || cols < 0 || cols % 16 != 0 || f_min > 0 || f_max < 0) return SS_ERR_INVALID_ARG;
  const int64_t nb = rows * cols / 16;
  if (nb > 0 && (!in || !out_codes || !out_scales)) return SS_ERR_INVALID_ARG;
  if (!aligned(in, 16) || !aligned(out_codes, 8) || !aligned(out_err, 8) || !aligned(d_global_scale, 4))
    return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  if (nb == 0) return SS_OK;
  Workspace* ws = nullptr;
  if (ss_status s = get_ws(dev, stream, &ws)) return s;
  ss::F32Params p;
  p.in = reinterpret_cast<const float4*>(in);
  p.nb = nb;
  p.fmin = std::max(f_min, -126);
  p.fmax = std::min(f_max, 126);
  p.g = d_global_scale;
  p.codes = reinterpret_cast<uint2*>(out_codes);
  p.scales = out_scales;
  p.err = reinterpret_cast<float2*>(out_err);
  p.offsets = out_offset;
  p.flags = ws->flags;
  void (*k)(ss::F32Params) = ss::quant_f32_kernel<-1, -1>;
  if (p.fmin == -8 && p.fmax == 8) k = ss::quant_f32_kernel<8, 8>;
  else if (p.fmin == -2 && p.fmax == 6) k = ss::quant_f32_kernel<2, 6>;
  else if (p.fmin == -1 && p.fmax == 1) k = ss::quant_f32_kernel<1, 1>;
  else if (p.fmin == 0 && p.fmax == 0) k = ss::quant_f32_kernel<0, 0>;
  const int64_t want = (nb + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)info.sms * 8));
  k<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  return launch_status();
}

ss_status ss_dequantize_nvfp4(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                              int64_t cols, const float* d_global_scale, void* out_bf16,
                              void* stream) {
  ss_dequant_args a;
  std::memset(&a, 0, sizeof(a));
  a.codes = codes;
  a.scales = scales;
  a.rows = rows;
  a.cols = cols;
  a.d_global_scale = d_global_scale;
  a.out_bf16 = out_bf16;
  a.stream = stream;
  return ss_dequantize_nvfp4_ex(&a);
}

ss_status ss_get_device_status(int* flags, void* stream) {
  if (!flags) return SS_ERR_INVALID_ARG;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  Workspace* ws = nullptr;
  if (ss_status s = get_ws(dev, stream, &ws)) return s;
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
  if (ss_status s = device_check(&dev, &info)) return s;
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
  ss_status st;
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
  std::vector<cudaEvent_t> ev(2 * nchunks);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  auto done = [&](ss_status s) {
    for (auto& e : ev) cudaEventDestroy(e);
    return s;
  };
  auto quant_chunk = [&](int64_t k) -> ss_status {
    const int64_t r0 = k * chunk_rows, r1 = std::min(rows, r0 + chunk_rows);
    ss_tensor_io t;
    std::memset(&t, 0, sizeof(t));
    t.in_bf16 = din + (size_t)r0 * cols * 2;
    t.rows = r1 - r0;
    t.cols = cols;
    t.d_amax_bits = hp.d_amax;
    t.out_codes = reinterpret_cast<uint8_t*>(hp.d_codes) + (size_t)r0 * cols / 2;
    t.out_scales = reinterpret_cast<uint8_t*>(hp.d_scales) + (size_t)r0 * cols / 16;
    t.out_err = h_err ? reinterpret_cast<float*>(hp.d_err) + (size_t)r0 * cols / 8 : nullptr;
    ss_status s = quantize_core(&t, 1, f_min, f_max,
                                tensor ? SS_GLOBAL_DEVICE_AMAX : SS_GLOBAL_NONE, hp.s_comp);
    if (s) return s;
    cudaEventRecord(ev[nchunks + k], hp.s_comp);
    cudaStreamWaitEvent(hp.s_d2h, ev[nchunks + k], 0);
    cudaMemcpyAsync(h_codes + (size_t)r0 * cols / 2, t.out_codes, (size_t)(r1 - r0) * cols / 2,
                    cudaMemcpyDeviceToHost, hp.s_d2h);
    cudaMemcpyAsync(h_scales + (size_t)r0 * cols / 16, t.out_scales, (size_t)(r1 - r0) * cols / 16,
                    cudaMemcpyDeviceToHost, hp.s_d2h);
    if (h_err)
      cudaMemcpyAsync(h_err + (size_t)r0 * cols / 8, t.out_err, (size_t)(r1 - r0) * cols / 2,
                      cudaMemcpyDeviceToHost, hp.s_d2h);
    return SS_OK;
  };
  if (tensor && cudaMemsetAsync(hp.d_amax, 0, 4, hp.s_comp) != cudaSuccess) return done(SS_ERR_CUDA);
  // phase 1: H2D every chunk; in TENSOR mode the amax of each chunk follows its copy,
  // in NONE mode the chunk is quantized and copied back as soon as it lands
  for (int64_t k = 0; k < nchunks; k++) {
    const int64_t r0 = k * chunk_rows, r1 = std::min(rows, r0 + chunk_rows);
    const size_t off = (size_t)r0 * cols * 2, bytes = (size_t)(r1 - r0) * cols * 2;
    if (cudaMemcpyAsync(din + off, hin + off, bytes, cudaMemcpyHostToDevice, hp.s_h2d) != cudaSuccess)
      return done(SS_ERR_CUDA);
    cudaEventRecord(ev[k], hp.s_h2d);
    cudaStreamWaitEvent(hp.s_comp, ev[k], 0);
    if (tensor) {
      const void* p = din + off;
      const int64_t cnt = (r1 - r0) * cols;
      if ((st = amax_launch(&p, &cnt, hp.d_amax, 1, true, hp.s_comp, info.sms))) return done(st);
    } else if ((st = quant_chunk(k))) {
      return done(st);
    }
  }
  // phase 2 (TENSOR): quantize chunk by chunk with the final amax, copying results back
  if (tensor)
    for (int64_t k = 0; k < nchunks; k++)
      if ((st = quant_chunk(k))) return done(st);
  cudaError_t e1 = cudaStreamSynchronize(hp.s_comp);
  cudaError_t e2 = cudaStreamSynchronize(hp.s_d2h);
  cudaError_t e3 = cudaStreamSynchronize(hp.s_h2d);
  return done((e1 || e2 || e3) ? SS_ERR_CUDA : SS_OK);
}

ss_status ss_quantize_nvfp4_host_batched(const ss_host_tensor_io* t, int count, int f_min,
                                         int f_max, int global_scale_mode) {
  if (count < 0 || (count > 0 && !t) || f_min > 0 || f_max < 0) return SS_ERR_INVALID_ARG;
  if (global_scale_mode != SS_GLOBAL_NONE && global_scale_mode != SS_GLOBAL_TENSOR)
    return SS_ERR_INVALID_ARG;
  int64_t max_n = 0;
  bool any_err = false;
  for (int i = 0; i < count; i++) {
    if (t[i].rows < 0 || t[i].cols < 0 || t[i].cols % 16 != 0) return SS_ERR_INVALID_ARG;
    const int64_t n = t[i].rows * t[i].cols;
    if (n > 0 && (!t[i].h_in_bf16 || !t[i].h_codes || !t[i].h_scales)) return SS_ERR_INVALID_ARG;
    max_n = std::max(max_n, n);
    any_err |= t[i].h_err != nullptr;
  }
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  if (count == 0 || max_n == 0) return SS_OK;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  HostRing& R = g_rings[dev];
  if (!R.s_h2d) {
    if (cudaStreamCreateWithFlags(&R.s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&R.s_comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&R.s_d2h, cudaStreamNonBlocking) != cudaSuccess)
      return SS_ERR_CUDA;
    for (int k = 0; k < HostRing::kSlots; k++)
      if (cudaEventCreateWithFlags(&R.in_ready[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&R.out_ready[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&R.slot_free[k], cudaEventDisableTiming) != cudaSuccess)
        return SS_ERR_CUDA;
  }
  // every sub-buffer of a slot (and every slot) starts on a 256-B boundary:
  // the kernels load the input and store E2M1 codes / errors as 16-B and 8-B
  // vectors
  auto up256 = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t per_slot = up256((size_t)max_n * 2) + up256((size_t)max_n / 2) + up256((size_t)max_n / 16) +
                          (any_err ? up256((size_t)max_n / 2) : 0);
  if (per_slot > R.slot_bytes) {
    cudaStreamSynchronize(R.s_h2d);
    cudaStreamSynchronize(R.s_comp);
    cudaStreamSynchronize(R.s_d2h);
    if (R.mem) cudaFree(R.mem);
    R.mem = nullptr;
    R.slot_bytes = 0;
    if (cudaMalloc(&R.mem, per_slot * HostRing::kSlots) != cudaSuccess) return SS_ERR_CUDA;
    R.slot_bytes = per_slot;
  }
  if (!R.amax && cudaMalloc(&R.amax, 4 * HostRing::kSlots) != cudaSuccess) return SS_ERR_CUDA;
  const bool tensor = global_scale_mode == SS_GLOBAL_TENSOR;
  for (int i = 0; i < count; i++) {
    const int64_t n = t[i].rows * t[i].cols, nb = n / 16;
    if (n == 0) continue;
    const int k = i % HostRing::kSlots;
    char* base = reinterpret_cast<char*>(R.mem) + (size_t)k * R.slot_bytes;
    void* d_in = base;
    uint8_t* d_codes = reinterpret_cast<uint8_t*>(base + up256((size_t)n * 2));
    uint8_t* d_scales = d_codes + up256((size_t)nb * 8);
    float* d_err = t[i].h_err ? reinterpret_cast<float*>(d_scales + up256((size_t)nb)) : nullptr;
    // the slot's previous tensor must be fully copied out before reuse
    if (cudaStreamWaitEvent(R.s_h2d, R.slot_free[k], 0) != cudaSuccess) return SS_ERR_CUDA;
    if (cudaMemcpyAsync(d_in, t[i].h_in_bf16, (size_t)n * 2, cudaMemcpyHostToDevice, R.s_h2d) !=
        cudaSuccess)
      return SS_ERR_CUDA;
    cudaEventRecord(R.in_ready[k], R.s_h2d);
    cudaStreamWaitEvent(R.s_comp, R.in_ready[k], 0);
    ss_tensor_io io;
    std::memset(&io, 0, sizeof(io));
    io.in_bf16 = d_in;
    io.rows = t[i].rows;
    io.cols = t[i].cols;
    io.d_amax_bits = R.amax + k;
    io.out_codes = d_codes;
    io.out_scales = d_scales;
    io.out_err = d_err;
    if (tensor) {
      const void* p = d_in;
      if (ss_status s = amax_launch(&p, &n, R.amax + k, 1, false, R.s_comp, info.sms)) return s;
    }
    if (ss_status s = quantize_core(&io, 1, f_min, f_max,
                                    tensor ? SS_GLOBAL_DEVICE_AMAX : SS_GLOBAL_NONE, R.s_comp))
      return s;
    cudaEventRecord(R.out_ready[k], R.s_comp);
    cudaStreamWaitEvent(R.s_d2h, R.out_ready[k], 0);
    cudaMemcpyAsync(t[i].h_codes, d_codes, (size_t)nb * 8, cudaMemcpyDeviceToHost, R.s_d2h);
    cudaMemcpyAsync(t[i].h_scales, d_scales, (size_t)nb, cudaMemcpyDeviceToHost, R.s_d2h);
    if (d_err)
      cudaMemcpyAsync(t[i].h_err, d_err, (size_t)nb * 8, cudaMemcpyDeviceToHost, R.s_d2h);
    if (cudaEventRecord(R.slot_free[k], R.s_d2h) != cudaSuccess) return SS_ERR_CUDA;
  }
  cudaError_t e1 = cudaStreamSynchronize(R.s_h2d);
  cudaError_t e2 = cudaStreamSynchronize(R.s_comp);
  cudaError_t e3 = cudaStreamSynchronize(R.s_d2h);
  return (e1 || e2 || e3) ? SS_ERR_CUDA : SS_OK;
}

// ---- generic ExMy block formats ----------------------
ss_status ss_quantize_gen(const ss_tensor_io* t, int f_min, int f_max, int global_scale_mode,
                          const ss_gen_format* fmt, void* stream) {
  ss::GenFmt f;
  if (!t || !gen_fmt(fmt, &f)) return SS_ERR_INVALID_ARG;
  const int bs = fmt->block;
  if (t->rows < 0 || t->cols < 0 || t->cols % bs != 0 || f_min > 0 || f_max < 0) return SS_ERR_INVALID_ARG;
  if (global_scale_mode != SS_GLOBAL_NONE && global_scale_mode != SS_GLOBAL_TENSOR &&
      global_scale_mode != SS_GLOBAL_DEVICE_AMAX)
    return SS_ERR_INVALID_ARG;
  const int64_t nb = t->rows * t->cols / bs;
  if (nb > 0 && (!t->in_bf16 || !t->out_codes || !t->out_scales)) return SS_ERR_INVALID_ARG;
  if (global_scale_mode == SS_GLOBAL_DEVICE_AMAX && !t->d_amax_bits) return SS_ERR_INVALID_ARG;
  // a global scale needs a finite numerator vmax * smax (not UE8M0, whose range needs none)
  if (global_scale_mode != SS_GLOBAL_NONE && !std::isfinite(f.vmax * f.smax)) return SS_ERR_INVALID_ARG;
  if (!aligned(t->in_bf16, 16) || !aligned(t->out_codes, 16) || !aligned(t->out_err, 8) ||
      !aligned(t->d_err_sums, 8) || !aligned(t->d_amax_bits, 4) || !aligned(t->d_global_scale, 4))
    return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (nb == 0) {
    if (t->d_err_sums && cudaMemsetAsync(t->d_err_sums, 0, 16, cs) != cudaSuccess) return SS_ERR_CUDA;
    return SS_OK;
  }
  Workspace* ws = nullptr;
  if (ss_status s = get_ws(dev, stream, &ws)) return s;
  std::lock_guard<std::mutex> wlk(ws->mu);
  const int64_t chunks = (nb + 255) / 256;
  if (t->d_err_sums) {
    if (ss_status s = grow_dev(&ws->part1, &ws->part1_cap, chunks, false, cs)) return s;
    if (ss_status s = grow_dev(&ws->part2, &ws->part2_cap, (chunks + ss::kSegTasks - 1) / ss::kSegTasks,
                               false, cs))
      return s;
  }
  const uint32_t* amax = nullptr;
  if (global_scale_mode == SS_GLOBAL_TENSOR) {
    if (ss_status s = grow_dev(&ws->amax, &ws->amax_cap, 1, false, cs)) return s;
    const void* in = t->in_bf16;
    const int64_t n = t->rows * t->cols;
    if (ss_status s = amax_launch(&in, &n, ws->amax, 1, false, cs, info.sms)) return s;
    amax = ws->amax;
  } else if (global_scale_mode == SS_GLOBAL_DEVICE_AMAX) {
    amax = t->d_amax_bits;
  }
  ss::GenParams p;
  std::memset(&p, 0, sizeof(p));
  p.in = reinterpret_cast<const uint4*>(t->in_bf16);
  p.nb = nb;
  p.fmin = std::max(f_min, -f.smaxc);
  p.fmax = std::min(f_max, f.smaxc);
  p.gmode = amax ? 1 : 0;
  p.amax = amax;
  p.g_numer = f.vmax * f.smax;  // exact: both have few significant bits
  p.codes = reinterpret_cast<uint4*>(t->out_codes);
  p.scales = t->out_scales;
  p.err = reinterpret_cast<float2*>(t->out_err);
  p.offsets = t->out_offset;
  p.g_out = t->d_global_scale;
  p.part1 = t->d_err_sums ? ws->part1 : nullptr;
  p.flags = ws->flags;
  p.f = f;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)info.sms * 8));
  ss_status st = bs == 16 ? launch_pdl(ss::quant_gen_kernel<16>, grid, 256, cs, p)
                          : launch_pdl(ss::quant_gen_kernel<32>, grid, 256, cs, p);
  if (st) return st;
  if (t->d_err_sums) {  // reduce the per-chunk partials (fixed order) into the tensor's sums
    QuantBatch b;
    std::memset(&b, 0, sizeof(b));
    b.n = 1;
    b.part1 = ws->part1;
    b.part2 = ws->part2;
    b.tick = ws->tick;
    b.t[0].sums = t->d_err_sums;
    b.t[0].part0 = 0;
    b.t[0].npart = (int32_t)chunks;
    b.t[0].seg0 = 0;
    b.nsegs = (chunks + ss::kSegTasks - 1) / ss::kSegTasks;
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(b.nsegs, sums_grid(info.sms)));
    if (ss_status s = launch_pdl(ss::sums_kernel, g2, ss::kThreads, cs, b)) return s;
  }
  return SS_OK;
}

ss_status ss_dequantize_gen(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols,
                            const ss_gen_format* fmt, const float* d_global_scale, void* out_bf16,
                            void* stream) {
  ss::GenFmt f;
  if (!gen_fmt(fmt, &f)) return SS_ERR_INVALID_ARG;
  if (rows < 0 || cols < 0 || cols % fmt->block != 0) return SS_ERR_INVALID_ARG;
  const int64_t n = rows * cols;
  if (n > 0 && (!codes || !scales || !out_bf16)) return SS_ERR_INVALID_ARG;
  if (!aligned(out_bf16, 2) || !aligned(d_global_scale, 4)) return SS_ERR_ALIGNMENT;
  int dev;
  DeviceInfo info;
  if (ss_status s = device_check(&dev, &info)) return s;
  if (n == 0) return SS_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)info.sms * 8));
  ss::dequant_gen_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      codes, scales, n, fmt->block, d_global_scale, f, reinterpret_cast<__nv_bfloat16*>(out_bf16));
  return launch_status();
}

#ifdef SS_COUNT_EVALS
/* Tools-only (libss_count.so): block-candidate evaluations executed since the
 * last call (synchronizes the device). */
SS_API unsigned long long ss_debug_take_evals(void) {
  unsigned long long h = 0;
  if (!g_evals) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(&h, g_evals, 8, cudaMemcpyDeviceToHost);
  cudaMemset(g_evals, 0, 8);
  return h;
}
#endif
#ifdef SS_AF_TRACE
/* Tools-only (libss_trace.so): fused-amax trace of the launches since the last
 * call: {first CTA start, last amax-warp finish, summed search-warp wait,
 * last warp finish}, globaltimer ns (synchronizes the device). */
SS_API void ss_debug_take_aftrace(unsigned long long* out) {
  if (!g_evals) return;
  cudaDeviceSynchronize();
  cudaMemcpy(out, g_evals, 32, cudaMemcpyDeviceToHost);
  unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
  cudaMemcpy(g_evals, init, 32, cudaMemcpyHostToDevice);
}
#endif

}  // extern "C"
