/*
 * ss_oracle.h — CPU oracle for ScaleSearch NVFP4 quantization.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2605_12464_b200/, include/ss.h, libss.so) never
 * links, imports or calls anything here, and this file shares no code,
 * header, table or constant with it.
 *
 * Citations: "P:n" is /root/reference/PAPER.md line n (arxiv 2605.12464,
 * LaTeX source).  Readings of the paper where it is silent, garbled or
 * inconsistent are numbered R1..R18 and listed in DESIGN.md §3; they are the
 * same readings as SURVEY.md §8(c).
 *
 * All status codes: 0 = ok, 1 = invalid argument, 4 = non-finite input,
 * 5 = global scale out of range (G not finite).
 */
#ifndef SS_ORACLE_H
#define SS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Number formats. */
double so_e2m1_value(int nibble);          /* nibble 0..15 -> value (sign bit 3)   */
int    so_e2m1_encode(float t);            /* RNE, saturating, sign kept (R10,R11) */
float  so_e4m3_value(int code);            /* code 0..126 -> value; 127 -> NaN (R2) */
int    so_e4m3_encode(float v);            /* v >= 0: RNE, satfinite -> 0..126      */
void   so_e2m1_encode_array(const float* t, int64_t n, uint8_t* nib);
void   so_e4m3_encode_array(const float* v, int64_t n, uint8_t* code);

/* Algorithm 1 on one 16-element block y (already multiplied by
 * the global scale), over offsets f in [fmin, fmax] (fmin <= 0 <= fmax).
 * Outputs: c0 (max-abs code), cstar (winner code), err_best, err_base, the
 * 16 winner nibbles (one per byte) and the number of candidates evaluated. */
typedef struct {
  int32_t c0, cstar, fstar, n_evaluated;
  float err_best, err_base;
  uint8_t nib[16];
} so_block_result;
int so_search_block(const float y[16], int fmin, int fmax, so_block_result* out);

/* Global amax over n bf16 values (exact): writes the FP32 bit pattern of
 * max|x|.  Returns 4 if any value is NaN/Inf. */
int so_tensor_amax(const uint16_t* x_bf16, int64_t n, uint32_t* amax_bits);

/* Global scale G from amax bits (figVLLMnvf4, R9):
 * gmode 0 (NONE): G = 1; otherwise G = RN(2688 / A), G = 1 when A == 0. */
int so_global_scale(int gmode, uint32_t amax_bits, float* G);

/* Whole-tensor quantization: x is [rows][cols] bf16 row-major, cols % 16 == 0.
 * gmode: 0 NONE, 1 TENSOR (amax of this tensor), 2 GIVEN (use *amax_bits_in,
 * e.g. the max over all row shards), 3 ROW (each row is its own tensor of
 * mode 1: G_r from the row amax; G_out then has `rows` entries).
 * Outputs (nullable except codes/scales):
 *   codes   [rows][cols/2]  u8, low nibble = even element (R15)
 *   scales  [rows][cols/16] u8 E4M3 code
 *   offsets [rows*cols/16]  i8 f* = c* - c0
 *   err     [rows*cols/16][2] f32 {err_best, err_base} (y-domain SSE)
 *   sums    [2] f64 {sum err_best, sum err_base} in block order
 *   n_eval  [1] i64 total candidates evaluated
 *   G_out   [1] f32 global scale used ([rows] in mode 3)
 * threads <= 0 means "all cores".  Blocks are independent; threads only split
 * rows and never change any arithmetic or summation order. */
int so_quantize(const uint16_t* x_bf16, int64_t rows, int64_t cols, int fmin,
                int fmax, int gmode, const uint32_t* amax_bits_in,
                uint8_t* codes, uint8_t* scales, int8_t* offsets, float* err,
                double* sums, int64_t* n_eval, float* G_out, int threads);

/* Other block formats: value format vfmt 0 E2M1 / 1 E2M3,
 * scale format sfmt 0 UE4M3 / 1 UE8M0 (R19), block size bs 16..256 (16 * 2^k;
 * loss = pairwise tree sum of the 16-element parts' R12 losses; R20). */
double so_e2m3_value(int code);            /* code 0..63 (sign bit 5) -> value      */
int    so_e2m3_encode(float t);            /* RNE, saturating at 7.5, sign kept     */
float  so_ue8m0_value(int code);           /* 2^(code-127), code 0..254             */
int    so_ue8m0_encode(float v);           /* smallest power of two >= v, sat. (R19)*/
typedef struct {
  int32_t c0, cstar, fstar, n_evaluated;
  float err_best, err_base;
  uint8_t code[256];                       /* value codes of the winner, one per byte */
} so_block_result_fmt;
int so_search_block_fmt(int vfmt, int sfmt, int bs, const float* y, int fmin, int fmax,
                        so_block_result_fmt* out);
int so_quantize_fmt(const uint16_t* x_bf16, int64_t rows, int64_t cols, int fmin, int fmax,
                    int gmode, const uint32_t* amax_bits_in, int vfmt, int sfmt, int bs,
                    uint8_t* codes, uint8_t* scales, int8_t* offsets, float* err,
                    double* sums, int64_t* n_eval, float* G_out, int threads);

int so_dequantize_fmt(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols,
                      int vfmt, int sfmt, int bs, const float* G, int per_row, uint16_t* out_bf16);

/* Generic ExMy formats (fig:nvfp-scale / fig:nvfp-val /
 * fig:mxfp P:237-260; reading R21): value ExMy (e >= 1, sign bit
 * above the e+m magnitude bits, every code finite), unsigned scale UExMy
 * (all-ones code NaN; m >= 1 with subnormals and a zero code, c0 by nearest
 * ties-to-even satfinite; m == 0 pure powers of two, c0 rounded up, R19).
 * Codes one per byte, scales one per block. */
double so_gen_value(int e, int m, int code);
int    so_gen_encode(int e, int m, float t);
double so_gen_scale_value(int e, int m, int code);   /* NaN for the all-ones code */
int    so_gen_scale_encode(int e, int m, float v);
float  so_gen_numer(int ve, int vm, int se, int sm); /* RN(vmax * smax) */
int so_search_block_gen(int ve, int vm, int se, int sm, int bs, const float* y, int fmin,
                        int fmax, so_block_result_fmt* out);
int so_quantize_gen(const uint16_t* x_bf16, int64_t rows, int64_t cols, int fmin, int fmax,
                    int gmode, const uint32_t* amax_bits_in, int ve, int vm, int se, int sm,
                    int bs, uint8_t* codes, uint8_t* scales, int8_t* offsets, float* err,
                    double* sums, int64_t* n_eval, float* G_out, int threads);
int so_dequantize_gen(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols,
                      int ve, int vm, int se, int sm, int bs, float G, uint16_t* out_bf16);

/* Dequantization: xhat = RNE_bf16(RN((q * s) / G)). */
int so_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                  int64_t cols, float G, uint16_t* out_bf16);

#ifdef __cplusplus
}
#endif
#endif
