/*
 * ss.h — C ABI of libss.so: ScaleSearch NVFP4 quantization on B200 (sm_100a).
 *
 * Method: arxiv 2605.12464, "Search Your Block Floating Point Scales!".
 * Citations "P:n" are lines of the paper's LaTeX source; "R<k>"
 * are the readings of the paper listed in DESIGN.md §3.
 *
 * Formats.  A bf16 tensor X[rows][cols] (row-major, cols % 16 == 0)
 * is cut into 16-element blocks along each row.  Each block is stored
 * as 16 E2M1 nibbles (values {0,±0.5,±1,±1.5,±2,±3,±4,±6}) and one
 * UE4M3 scale byte (OCP E4M3 code 0..126, bias 7; R1, R2).  A per-tensor FP32
 * global scale G = RN(2688 / max|X|) maps the tensor amax onto 6*448 first
 * (figVLLMnvf4; R9), so block b quantizes y = RN(x * G).
 *
 * ScaleSearch (Algorithm 1): per block, c0 = round_UE4M3(max|y| *
 * RN(1/6)) (R8); for each offset f in [f_min, f_max] (R6) with valid code
 * c = c0 + f (1 <= c <= 126; plus the zero scale when c0 == 0, f == 0; R2, R3)
 * the block is quantized with t_i = RN(y_i * RN(1/s_c)) (R7), q_i =
 * E2M1_RNE_satfinite(t_i) (R10), d_i = RN(y_i - q_i*s_c) and loss
 * L = RN(a + b) with a, b the FP32 FMA chains of d_i^2 over even / odd i (R12).
 * The winner is the lexicographic minimum of (L, c): ties keep the smaller
 * scale (Alg. 1 strict <; R4).  Outputs are bit-identical to the CPU
 * oracle (oracle/ss_oracle.c) under this contract.
 *
 * Layouts (R15): codes [rows][cols/2] u8, element 2j in the low nibble of byte
 * j, sign in bit 3 of each nibble (negative values that round to 0 keep the
 * sign, R11); scales [rows][cols/16] u8 E4M3 codes, linear row-major, or the
 * tensor-core swizzled layout (SS_SCALE_SWIZZLED, R15b).  Per-row global
 * scales (SS_GLOBAL_ROW, R9b) and other block formats (SS_FMT_*, R19, R20)
 * are opt-in through the _ex / _batched / _fmt entry points.
 *
 * Implementation notes (outputs are unaffected by all of them):
 *  - candidates that provably cannot win are skipped (exact branch and
 *    bound);
 *  - with SS_GLOBAL_TENSOR the amax pass of a multi-tensor batch runs inside
 *    the quantize launch (§4.2a); a call of >= 2^26 elements runs as a chain
 *    of launches whose search warps fold the next launch's amax (§4.2c);
 *  - a single small tensor (<= 2^19 blocks) takes a one-thread-per-block
 *    kernel built on the device routine of ss_device.cuh (§4.8);
 *  - FP32 input: ss_quantize_nvfp4_f32; sharded steps:
 *    ss_quantize_nvfp4_batched_next_amax (§5).
 *
 * Conventions for every entry point:
 *  - All array arguments are DEVICE pointers owned by the caller unless the
 *    name starts with h_ (host).  The library never keeps a pointer after the
 *    call returns; its only allocations are a per-(device, stream) workspace
 *    (status flags, scheduler counters, amax slots, error-sum partials) and,
 *    for the host-buffer entry points, a ring of device staging slots, all
 *    created on first use, grown monotonically and reused.  Growing one
 *    synchronizes its stream once; a CUDA graph may capture a call whose
 *    workspace is already warm (tests/test_parity_gpu.py).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call only enqueues work on `stream` and returns; none synchronizes
 *    except ss_get_device_status and the two _host entry points.
 *  - Argument errors are detected synchronously and returned without
 *    launching anything.  A failed launch returns SS_ERR_CUDA.
 *  - Non-finite input (NaN/Inf) cannot be reported synchronously: the amax
 *    pass sets a sticky device flag (read with ss_get_device_status), uses
 *    G = 1, and the outputs are defined but meaningless.
 *  - Reentrant; calls on distinct streams may run concurrently.
 *  - There is no CPU fallback: without an sm_100 device every call returns
 *    SS_ERR_UNSUPPORTED_DEVICE.
 *  - No environment input: every choice is an argument or compile-time
 *    (tools build their A/B variants as separate libss_<variant>.so files).
 *
 * Differences from the interface sketched in SURVEY.md §8(b) (itself mapped
 * from SPEC S:150-158):
 *  - every enqueueing call takes an explicit trailing `stream` argument (or
 *    an ss_quant_args.stream field) instead of a thread-local stream set by
 *    ss_set_stream(): a call's stream is visible at the call site, and
 *    calls from several threads need no per-thread state;
 *  - ss_tensor_amax takes an `accumulate` flag, so the amaxes of several
 *    chunks or row shards can be folded into one slot before the all-reduce;
 *  - ss_quantize_nvfp4 takes the north star's argument list plus `stream`;
 *    the optional outputs (f*, FP64 sums, G), explicit windows, formats and
 *    layouts are in ss_quantize_nvfp4_ex / the batched calls.
 */
#ifndef SS_H
#define SS_H

#include <stdint.h>

#if defined(__GNUC__)
#define SS_API __attribute__((visibility("default")))
#else
#define SS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SS_OK = 0,
  SS_ERR_INVALID_ARG = 1,        /* null pointer, bad size, cols % 16, f_min > 0 or f_max < 0 */
  SS_ERR_ALIGNMENT = 2,          /* in_bf16 / out_bf16 not 16-B aligned, E2M1 codes not 8-B   */
                                 /* aligned, E2M3 codes not 16-B aligned, err not 8-B aligned */
  SS_ERR_CUDA = 3,               /* a CUDA runtime call or launch failed                      */
  SS_ERR_NONFINITE = 4,          /* (device flag) NaN/Inf seen by an amax pass                */
  SS_ERR_RANGE = 5,              /* (device flag) 0 < amax < 2688/FLT_MAX: G overflows        */
  SS_ERR_UNSUPPORTED_DEVICE = 6  /* current device is not compute capability 10.x            */
} ss_status;

/* Global-scale modes (R9). */
enum {
  SS_GLOBAL_NONE = 0,        /* G = 1: y = x (the paper's §4.1 synthetic setting)      */
  SS_GLOBAL_TENSOR = 1,      /* G from the amax of THIS tensor (one extra HBM read pass)      */
  SS_GLOBAL_DEVICE_AMAX = 2, /* G from *d_amax_bits supplied by the caller, e.g. the NCCL max  */
                             /* over all row shards of a tensor                */
  SS_GLOBAL_ROW = 3          /* per-row G_r = RN(2688 / max|x_r|) ("after per-row scaling",  */
                             /* P:313): d_global_scale is REQUIRED and        */
                             /* receives [rows] f32; each row is its own tensor of mode 1    */
};

/* Scale-factor layouts (R15, R15b). */
enum {
  SS_SCALE_LINEAR = 0,       /* [rows][cols/16] u8 row-major                                   */
  SS_SCALE_SWIZZLED = 1      /* the block-scaled tensor-core layout (cuBLAS/CUTLASS sm_100     */
                             /* "128x4" scale-factor atom): 512-B tiles of 128 rows x 4 scale  */
                             /* columns, tiles row-band-major, inside a tile byte             */
                             /* (r%32)*16 + ((r/32)%4)*4 + j%4; rows padded to 128 and scale  */
                             /* columns to 4 with zero bytes.  Size: ss_scale_bytes()         */
};

/* Block formats (readings R19, R20).
 * Codes: E2M1 values two per byte (low nibble = even element), E2M3 values
 * one 6-bit code per byte (sign bit 5).  Scales: UE4M3 codes 0..126, or UE8M0
 * codes 0..254 = 2^(c-127) rounded UP from x_max / vmax (R19; no global scale:
 * UE8M0 formats take SS_GLOBAL_NONE only).  32-element blocks need
 * cols % block == 0; their loss is the tree sum of the 16-element parts' R12 losses. */
enum {
  SS_FMT_NVFP4 = 0,          /* E2M1 values, UE4M3 scales, 16-blocks (the north star)         */
  SS_FMT_MXFP4 = 1,          /* E2M1 values, UE8M0 scales, 32-blocks                          */
  SS_FMT_MXFP6_E2M3 = 2,     /* E2M3 values, UE8M0 scales, 32-blocks                          */
  SS_FMT_NVFP6_E2M3 = 3,     /* E2M3 values, UE4M3 scales, 16-blocks (the value-format sweep) */
  SS_FMT_NVFP4_B32 = 4,      /* NVFP4 values and scales on 32-, 64-, 128-, 256-element       */
  SS_FMT_NVFP4_B64 = 5,      /* blocks: the block-size study (fig:block_size);    */
  SS_FMT_NVFP4_B128 = 6,     /* a block's loss is the pairwise tree sum of its 16-element    */
  SS_FMT_NVFP4_B256 = 7      /* parts' R12 losses (R20)                                       */
};

/* Bytes of the scale buffer of a [rows][cols] tensor in `scale_layout`
 * (NVFP4 blocks). */
SS_API int64_t ss_scale_bytes(int64_t rows, int64_t cols, int scale_layout);
/* Same for any format, and the bytes of its code buffer.  -1 on bad input. */
SS_API int64_t ss_scale_bytes_fmt(int64_t rows, int64_t cols, int scale_layout, int format);
SS_API int64_t ss_code_bytes(int64_t rows, int64_t cols, int format);

/* Human-readable name of a status code (static string). */
SS_API const char* ss_status_string(int status);

/* ABI version (major * 100 + minor). */
SS_API int ss_version(void);

/*
 * Global amax (step a2; "dividing by the global scale from ... tensor
 * scaling").  Reduces max|x| over n bf16 values at in_bf16 into
 * *d_amax_bits as the FP32 bit pattern of the maximum (bf16 -> f32 is exact,
 * so this is exact and independent of order).  The reduction is an unsigned
 * integer max on |x| bit patterns, so NaN > Inf > any finite value: a result
 * >= 0x7F800000 means the input was not finite.
 *   accumulate = 0: *d_amax_bits is overwritten with the max of this call.
 *   accumulate = 1: *d_amax_bits = max(*d_amax_bits, max of this call)
 *                   (several chunks or row shards into one slot).
 * in_bf16 must be 16-B aligned; n >= 0 (n == 0 leaves / sets 0).
 */
SS_API ss_status ss_tensor_amax(const void* in_bf16, int64_t n, uint32_t* d_amax_bits,
                         int accumulate, void* stream);

/*
 * Batched global amax: d_amax_bits[i] = max|x| of tensor i (same semantics as
 * ss_tensor_amax), for `count` tensors in ONE launch (per launch at most 128
 * tensors; more are split into several launches).  in_bf16[i] / n[i] are HOST
 * arrays of device pointers / element counts; d_amax_bits is a device array
 * of `count` u32.  This is the per-shard half of the multi-GPU exchange step:
 * the slots can go straight into one NCCL max all-reduce.
 */
SS_API ss_status ss_tensor_amax_batched(const void* const* in_bf16, const int64_t* n, int count,
                                 uint32_t* d_amax_bits, int accumulate, void* stream);

/*
 * ScaleSearch quantization with a symmetric window f in [-radius, radius]
 * (north star; radius > 126 is clamped to 126 = exhaustive search).
 *   in_bf16     [rows][cols] bf16, 16-B aligned, cols % 16 == 0, rows >= 0
 *   global_scale_mode  SS_GLOBAL_NONE or SS_GLOBAL_TENSOR (this call runs the
 *               amax pass itself; a row shard of a larger tensor must use
 *               ss_quantize_nvfp4_ex with SS_GLOBAL_DEVICE_AMAX instead)
 *   out_codes   [rows][cols/2] u8, 8-B aligned
 *   out_scales  [rows][cols/16] u8
 *   out_err     nullable; [rows*cols/16][2] f32 {err_best, err_base}, the
 *               y-domain squared error of the winner and of the max-abs
 *               scale (f = 0), 8-B aligned
 */
SS_API ss_status ss_quantize_nvfp4(const void* in_bf16, int64_t rows, int64_t cols, int radius,
                            int global_scale_mode, uint8_t* out_codes, uint8_t* out_scales,
                            float* out_err, void* stream);

/* Full argument set.  Unused nullable outputs cost nothing. */
typedef struct {
  const void* in_bf16;          /* [rows][cols] bf16, 16-B aligned                         */
  int64_t rows, cols;           /* rows >= 0, cols % (block size of `format`) == 0         */
  int f_min, f_max;             /* inclusive window, f_min <= 0 <= f_max (R6); clamped to   */
                                /* [-126, 126] (UE4M3) / [-254, 254] (UE8M0); e.g. the      */
                                /* paper's production [-2, 6]                        */
  int global_scale_mode;        /* SS_GLOBAL_*                                              */
  const uint32_t* d_amax_bits;  /* SS_GLOBAL_DEVICE_AMAX: device u32 FP32 bits of the amax  */
  uint8_t* out_codes;           /* ss_code_bytes(): [rows][cols/2] u8 for E2M1, 8-B aligned;*/
                                /* [rows][cols] u8 for E2M3, 16-B aligned                   */
  uint8_t* out_scales;          /* ss_scale_bytes_fmt(): [rows][cols/bs] u8 or swizzled     */
  float* out_err;               /* nullable: [nb][2] f32 {err_best, err_base}, 8-B aligned; */
                                /* nb = rows * cols / block size                            */
  int8_t* out_offset;           /* nullable: [nb] f* = c* - c0 (R5)                          */
  double* d_err_sums;           /* nullable: device f64[2] = {sum err_best, sum err_base},  */
                                /* overwritten; fixed-order reduction of per-warp-task      */
                                /* partials (sums_kernel): deterministic for any grid       */
  float* d_global_scale;        /* nullable: device f32 receives G (for dequantization);    */
                                /* SS_GLOBAL_ROW: required, [rows] f32                     */
  void* stream;
  int scale_layout;             /* SS_SCALE_* (0 = linear)                                  */
  int format;                   /* SS_FMT_* (0 = NVFP4)                                      */
} ss_quant_args;

SS_API ss_status ss_quantize_nvfp4_ex(const ss_quant_args* args);

/* One tensor of a batched call; fields as in ss_quant_args. */
typedef struct {
  const void* in_bf16;          /* [rows][cols] bf16, 16-B aligned                         */
  int64_t rows, cols;           /* rows >= 0, cols % 16 == 0                                */
  const uint32_t* d_amax_bits;  /* SS_GLOBAL_DEVICE_AMAX: device u32 amax bits of THIS tensor */
  uint8_t* out_codes;           /* [rows][cols/2] u8, 8-B aligned (E2M3 formats:             */
                                /* [rows][cols] u8, 16-B aligned)                           */
  uint8_t* out_scales;          /* [rows][cols/16] u8                                       */
  float* out_err;               /* nullable: [nb][2] f32 {err_best, err_base}, 8-B aligned  */
  int8_t* out_offset;           /* nullable: [nb] f* = c* - c0                               */
  double* d_err_sums;           /* nullable: device f64[2] of THIS tensor, overwritten      */
  float* d_global_scale;        /* nullable: device f32 receives this tensor's G;           */
                                /* SS_GLOBAL_ROW: required, [rows] f32                     */
  int scale_layout;             /* SS_SCALE_* (0 = linear)                                  */
} ss_tensor_io;

/*
 * Batched ScaleSearch quantization: every tensor of `tensors[0..count)` (a
 * HOST array) with one window and one global-scale mode, in as few launches
 * as possible (one persistent grid per 128 tensors, so a step over many
 * small tensors has no per-tensor tail).  SS_GLOBAL_TENSOR computes each
 * tensor's amax inside the quantize launch when the format is NVFP4,
 * the scales are linear, the window has >= 4 offsets and the first tensor
 * holds at most half of the elements (amax warps run ahead of the search;
 * DESIGN.md §4.2a), else in one batched amax launch first.  A call of
 * >= 2^26 elements then runs as a chain of launches (first batch ~1/64 of the
 * elements, each later one at most twice its predecessor, <= 64 tensors),
 * each folding the next batch's amax after its scheduling units (§4.2c).
 * Results are bit-identical every way and to per-tensor calls;
 * ss_quantize_plan reports which was chosen.
 */
SS_API ss_status ss_quantize_nvfp4_batched(const ss_tensor_io* tensors, int count, int f_min,
                                    int f_max, int global_scale_mode, void* stream);

/*
 * One group of a sharded step: quantize `tensors` with
 * SS_GLOBAL_DEVICE_AMAX (each d_amax_bits already all-reduced) and, inside
 * the same launch, compute the LOCAL amax (FP32 bits of max|x|) of the
 * next group's shards into next_amax_bits[0..next_count) — overwritten —
 * ready for that group's all-reduce.  The amax pass of the next group thus
 * runs under this group's search (the amax warps of §4.2a), so a pipelined
 * step exposes only the first group's amax.
 *   next_in[j]   DEVICE bf16, 16-B aligned, next_n[j] elements (multiple of 16)
 *   next_count   <= 128
 * NVFP4, linear scales; any other case computes the next amaxes with a
 * separate launch first.  Results are bit-identical to
 * ss_tensor_amax_batched + ss_quantize_nvfp4_batched.
 */
SS_API ss_status ss_quantize_nvfp4_batched_next_amax(const ss_tensor_io* tensors, int count, int f_min,
                                                     int f_max, const void* const* next_in,
                                                     const int64_t* next_n, int next_count,
                                                     uint32_t* next_amax_bits, void* stream);

/*
 * Peer-memory amax exchange for row-sharded steps (the one
 * exchange of the method: G needs the whole tensor's amax).  Instead
 * of a host-issued NCCL all-reduce between the amax and quantize launches,
 * every rank owns an exchange buffer that every other rank maps (CUDA IPC,
 * over NVLink/NVSwitch).  The quantize launch of tensor group g reads the
 * ranks' shard amaxes of g from its own buffer once each rank's flag word
 * for g carries the step's epoch; the same launch computes the LOCAL amaxes
 * of group g+1 (the fused amax warps) and the warp that finishes the last of
 * them stores them into every rank's buffer and releases its flags there.
 * No host round trip and no collective kernel sit on the step's critical path.
 *
 * Buffer (ss_exchange_bytes): u32 words [2][max_tensors][8] amax slots (step
 * parity, tensor slot, rank) + [max_groups][8] flag words, zeroed once by
 * ss_exchange_init.  Epochs: the caller numbers steps 1, 2, ... identically
 * on every rank.  A consumer accepts a flag >= its epoch (a rank may run one
 * step ahead: it needs nothing from a peer's consumption to publish the next
 * step), and slots alternate by epoch parity, so that rank never overwrites
 * values a peer still reads (two steps ahead it would need the peer's next
 * publication, which is stream-ordered after the peer's reads).  A rank that never publishes
 * trips a ~10 s watchdog (SS_FLAG_EXCHANGE_TIMEOUT, G = 1) instead of a hang.
 */
#define SS_FLAG_EXCHANGE_TIMEOUT 8
#define SS_MAX_PEERS 8
#define SS_IPC_HANDLE_BYTES 64
typedef struct {
  int world;                    /* ranks, 1..8                                              */
  int rank;                     /* this rank                                                */
  uint32_t* buf[SS_MAX_PEERS];  /* DEVICE: every rank's exchange buffer as mapped in this   */
                                /* process (buf[rank] = own, the others via ss_ipc_open)    */
  int max_tensors;              /* geometry, identical on every rank                        */
  int max_groups;
} ss_exchange;
typedef struct {
  int slot0;                    /* first tensor slot of the group within a step             */
  int count;                    /* tensors of the group (= the call's count)                */
  int group;                    /* flag word index, < max_groups                            */
  uint32_t epoch;               /* step number >= 1, the same on every rank                 */
} ss_exchange_group;

SS_API int64_t ss_exchange_bytes(int max_tensors, int max_groups);
/* Zero a (new) exchange buffer of ss_exchange_bytes bytes on `stream`. */
SS_API ss_status ss_exchange_init(void* d_buf, int max_tensors, int max_groups, void* stream);
/* A zeroed exchange buffer in its own cudaMalloc allocation (so that
 * ss_ipc_handle exports exactly it; a sub-allocation of a caching allocator
 * would export its whole segment), and its release. */
SS_API ss_status ss_exchange_alloc(int max_tensors, int max_groups, void** d_buf);
SS_API ss_status ss_exchange_free(void* d_buf);
/* CUDA IPC: export a device allocation (SS_IPC_HANDLE_BYTES written to
 * `handle`), map a peer's (LAZY peer access), unmap.  Plain host calls. */
SS_API ss_status ss_ipc_handle(const void* d_ptr, void* handle);
SS_API ss_status ss_ipc_open(const void* handle, void** d_ptr);
SS_API ss_status ss_ipc_close(void* d_ptr);
/* Publish `g->count` local amaxes (DEVICE u32, FP32 bits) of a group to every
 * rank (one warp; used for the first group of a step, after
 * ss_tensor_amax_batched). */
SS_API ss_status ss_exchange_publish(const ss_exchange* x, const ss_exchange_group* g,
                                     const uint32_t* d_local_amax, void* stream);
/* Quantize group g_in (NVFP4, linear scales; per-tensor G from the ranks'
 * amaxes in the exchange, d_amax_bits ignored) and, in the same launch, the
 * local amaxes of the next group's shards (next_in / next_n as in
 * ss_quantize_nvfp4_batched_next_amax, into next_local_amax, overwritten),
 * published to every rank as group g_next.  next_count = 0: consume only.
 * Bit-identical to ss_tensor_amax_batched + all-reduce(max) +
 * ss_quantize_nvfp4_batched in SS_GLOBAL_DEVICE_AMAX mode. */
SS_API ss_status ss_quantize_nvfp4_exchange(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                                            const ss_exchange* x, const ss_exchange_group* g_in,
                                            const void* const* next_in, const int64_t* next_n,
                                            int next_count, uint32_t* next_local_amax,
                                            const ss_exchange_group* g_next, void* stream);

/*
 * The launch plan of a batched call, without enqueueing anything (no device
 * needed; pointers are validated for null / alignment but never read):
 * which kernels ss_quantize_batched_fmt / ss_quantize_nvfp4_batched would
 * launch for these arguments.  bench.py reads it for its gpu_launches count
 * and its traffic model (a fused amax reads the input twice).
 */
typedef struct {
  int amax_fused;   /* 1: SS_GLOBAL_TENSOR amax inside the quantize launch   */
  int small_path;   /* 1: one small tensor through the one-thread-per-block kernel (§4.8)      */
  int row_fused;    /* tensors whose per-row amax runs inside the quantize pass (§4.4)         */
  int launches;     /* kernels the call enqueues (amax, row-scale, quantize, error-sum)        */
  int trail_batches; /* > 1: a fused-amax call run as this many quantize launches, each
                        folding the next one's amax (trailing amax); else 0  */
} ss_plan;
SS_API ss_status ss_quantize_plan(const ss_tensor_io* tensors, int count, int f_min, int f_max,
                                  int global_scale_mode, int format, ss_plan* out);

/* The same for any block format (SS_FMT_*); windows are clamped to +-126
 * (UE4M3) or +-254 (UE8M0) code steps. */
SS_API ss_status ss_quantize_batched_fmt(const ss_tensor_io* tensors, int count, int f_min,
                                  int f_max, int global_scale_mode, int format, void* stream);

/*
 * Generic ExMy block formats: the format sweeps of the paper's §4.1
 * (fig:nvfp-scale: scale formats at E2M1 values; fig:nvfp-val: value formats
 * at UE4M3 scales; fig:mxfp: value formats at UE8M0 scales; P:237-260,
 * P:301-303 "hypothetical block quantization formats").  Reading R21
 * (DESIGN.md §3):
 *   value format ExMy   1 <= value_e, value_e + value_m <= 7; a sign bit above
 *                       the magnitude bits; bias 2^(e-1)-1, subnormals at
 *                       E = 0, every code finite (the OCP FP4/FP6 rule);
 *                       rounding RNE, saturating, sign kept (R10, R11)
 *   scale format UExMy  1 <= scale_e, scale_e + scale_m <= 8 (scale_e <= 7
 *                       when scale_m > 0); the all-ones code is NaN and never
 *                       used.  scale_m >= 1: subnormals, code 0 is the zero
 *                       scale (R3), c0 = nearest code ties-to-even satfinite
 *                       (Alg. 1 line 2); scale_m = 0: powers of two
 *                       2^(c - bias), c0 = the smallest >= x_max/vmax (R19)
 *   block               16 or 32 (a 32-block's loss: RN(low + high), R20)
 * Everything else is the NVFP4 contract: t = RN(y * RN(1/s)) (R7), R12 loss,
 * ascending strict-< scan (R4), f* = c* - c0, y = RN(x * G) with
 * G = RN(vmax * smax / A) (SS_GLOBAL_TENSOR / SS_GLOBAL_DEVICE_AMAX) or 1.
 * UE4M3 / E2M1 / 16 reproduces SS_FMT_NVFP4 bit for bit.
 */
typedef struct {
  int value_e, value_m;         /* value format ExMy                                         */
  int scale_e, scale_m;         /* scale format UExMy                                        */
  int block;                    /* 16 or 32                                                  */
} ss_gen_format;

/*
 * ScaleSearch over a generic format, one tensor (t->scale_layout must be
 * linear; t->d_amax_bits is read in SS_GLOBAL_DEVICE_AMAX mode):
 *   out_codes   DEVICE [rows][cols] u8, ONE value code per byte, 16-B aligned
 *   out_scales  DEVICE [rows][cols/block] u8 scale codes
 *   out_err     nullable float2 [nb] {err_best, err_base}; out_offset nullable
 *               int8 [nb] f* clamped to [-128, 127]; d_err_sums nullable
 *               double[2]; d_global_scale nullable float (G used)
 *   f_min, f_max  window, clamped to +-(2^(scale_e+scale_m) - 2)
 * Errors: SS_ERR_INVALID_ARG for a format outside the ranges above, cols %
 * block != 0, an inverted window, or a global-scale mode whose numerator
 * vmax * smax is not finite in binary32 (UE8M0 scales: use SS_GLOBAL_NONE); SS_ERR_ALIGNMENT as ss_quantize_nvfp4_ex.
 * A study kernel (software rounding, one thread per block).
 * Enqueued on `stream`, no host sync.
 */
SS_API ss_status ss_quantize_gen(const ss_tensor_io* t, int f_min, int f_max, int global_scale_mode,
                                 const ss_gen_format* fmt, void* stream);

/* a8 for a generic format: xhat = RNE_bf16(RN((q * s) / G)), codes and scales
 * as written by ss_quantize_gen; d_global_scale nullable (G = 1). */
SS_API ss_status ss_dequantize_gen(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                                   int64_t cols, const ss_gen_format* fmt, const float* d_global_scale,
                                   void* out_bf16, void* stream);

/*
 * FP32-input ScaleSearch NVFP4 through the one-thread block routine of
 * include/ss_device.cuh (the search a fused producer, e.g. attention's P
 * tile, runs in registers).  One thread per block.
 *   in              DEVICE float [rows][cols], 16-B aligned, cols % 16 == 0
 *   f_min, f_max    window as in ss_quantize_nvfp4_ex (clamped to +-126)
 *   d_global_scale  DEVICE float G (y = RN(x * G), R9), nullable => G = 1;
 *                   e.g. 2688 / amax, or a fixed scale for bounded data
 *   out_codes       [rows][cols/2] u8; out_scales [rows][cols/16] u8 (linear)
 *   out_err         nullable float2 [nb] {err_best, err_base}; out_offset
 *                   nullable int8 [nb] f*
 * Same contract as the bf16 path: for bf16-representable inputs and the
 * same G, outputs are bit-identical to ss_quantize_nvfp4_ex.  A non-finite
 * input sets SS_FLAG_NONFINITE (poll ss_get_device_status).  Enqueued on
 * `stream`, no host sync.
 */
SS_API ss_status ss_quantize_nvfp4_f32(const float* in, int64_t rows, int64_t cols, int f_min,
                                       int f_max, const float* d_global_scale, uint8_t* out_codes,
                                       uint8_t* out_scales, float* out_err, int8_t* out_offset,
                                       void* stream);

/*
 * Dequantization (step a8): xhat = RNE_bf16(RN((q * s) / G)).
 *   codes [rows][cols/2] u8 (8-B aligned), scales [rows][cols/16] u8,
 *   d_global_scale nullable (NULL => G = 1), out_bf16 [rows][cols] (16-B aligned).
 */
SS_API ss_status ss_dequantize_nvfp4(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                              int64_t cols, const float* d_global_scale, void* out_bf16,
                              void* stream);

/*
 * End-to-end from HOST memory (the e2e leg of bench.py): copies h_in to the
 * device in chunks, runs the amax pass per chunk as it lands (SS_GLOBAL_TENSOR)
 * and the quantization per chunk, and copies codes / scales (and errors when
 * h_err != NULL) back to host memory, overlapping copies with kernels on two
 * internal streams.  Host buffers should be pinned (cudaHostAlloc /
 * torch pin_memory) for full PCIe bandwidth; pageable memory works but is
 * staged by the driver.  Synchronous: returns after the outputs are in host
 * memory.  Device buffers are library-owned, cached per device and grown on
 * demand (size of one tensor plus its outputs).
 */
SS_API ss_status ss_quantize_nvfp4_host(const void* h_in_bf16, int64_t rows, int64_t cols, int f_min,
                                 int f_max, int global_scale_mode, uint8_t* h_codes,
                                 uint8_t* h_scales, float* h_err);

/* One tensor of ss_quantize_nvfp4_host_batched: HOST buffers. */
typedef struct {
  const void* h_in_bf16;        /* [rows][cols] bf16                                        */
  int64_t rows, cols;           /* rows >= 0, cols % 16 == 0                                */
  uint8_t* h_codes;             /* [rows][cols/2] u8                                        */
  uint8_t* h_scales;            /* [rows][cols/16] u8                                       */
  float* h_err;                 /* nullable: [nb][2] f32 {err_best, err_base}               */
} ss_host_tensor_io;

/*
 * End to end from HOST memory for a list of tensors (the e2e leg of bench.py
 * at N = 1): tensor k is copied in, its amax (SS_GLOBAL_TENSOR: each tensor's
 * own G) and quantization run, and its outputs are copied out, while tensor
 * k+1 is already being copied in and tensor k-1 copied out: three internal
 * streams and a ring of library-owned device slots, each sized for the
 * largest tensor.  Host buffers should be pinned.  Synchronous.  Results are
 * bit-identical to ss_quantize_nvfp4_batched.
 */
SS_API ss_status ss_quantize_nvfp4_host_batched(const ss_host_tensor_io* tensors, int count,
                                         int f_min, int f_max, int global_scale_mode);

/* Dequantization with per-row global scales and / or the swizzled layout. */
typedef struct {
  const uint8_t* codes;         /* [rows][cols/2] u8, 8-B aligned (E2M3: [rows][cols], 16-B) */
  const uint8_t* scales;        /* layout per scale_layout                                  */
  int64_t rows, cols;
  const float* d_global_scale;  /* nullable (G = 1); [1] or, with g_per_row, [rows]         */
  int g_per_row;
  int scale_layout;             /* SS_SCALE_*                                               */
  void* out_bf16;               /* [rows][cols] bf16, 16-B aligned                          */
  void* stream;
  int format;                   /* SS_FMT_* (0 = NVFP4)                                      */
} ss_dequant_args;

SS_API ss_status ss_dequantize_nvfp4_ex(const ss_dequant_args* args);

/* Synchronizes `stream`, returns and clears the sticky device flags of this
 * (device, stream) workspace: bit 0 = non-finite input seen (SS_ERR_NONFINITE),
 * bit 1 = global scale out of range (SS_ERR_RANGE), bit 2 = a fused-amax
 * search warp gave up waiting for its tensor's amax after ~10 s (a
 * watchdog against a stalled GPU; that tensor's outputs are meaningless),
 * bit 3 = a peer-exchange wait gave up after ~10 s (a rank never published;
 * SS_FLAG_EXCHANGE_TIMEOUT, that group's outputs are meaningless). */
SS_API ss_status ss_get_device_status(int* flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SS_H */
