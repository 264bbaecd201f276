/*
 * ss_oracle.c — plain, slow, obviously correct CPU oracle for ScaleSearch
 * NVFP4 quantization (arxiv 2605.12464, Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY (see ss_oracle.h).  It shares no code with the
 * CUDA path and is never linked into the product.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (x86-64 SSE: every float operation below is a single IEEE-754 binary32
 * operation rounded to nearest-even; FMAs appear only where fmaf() is
 * written, as the arithmetic contract in DESIGN.md §3 (R7, R8, R12) says).
 *
 * Style: scalar loops, rounding by enumerating the format's values and
 * taking the nearest (ties to the even code), no bit tricks, no tables
 * shared with anything else.  Each step cites the paper passage it follows.
 */
#include "ss_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------- */
/* E2M1: R_E2M1 = {0, +-0.5, +-1, +-1.5, +-2, +-3, +-4, +-6}.  */
/* Magnitude code k = (exponent bits << 1) | mantissa bit, sign in bit 3.  */
/* ---------------------------------------------------------------------- */
static const double E2M1_MAGNITUDE[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};

double so_e2m1_value(int nibble) {
  double v = E2M1_MAGNITUDE[nibble & 7];
  return (nibble & 8) ? -v : v;
}

/* round_E2M1 ("ordinary nearest-neighbor rounding"): the
 * magnitude nearest |t|, ties to the even code (R10); |t| above the largest
 * value saturates to 6 (satfinite, R10); the sign bit is copied from t, so a
 * negative t that rounds to 0 gives nibble 0x8 (R11). */
int so_e2m1_encode(float t) {
  int sign = signbit(t) ? 8 : 0;
  double a = fabs((double)t);
  if (a > 6.0) return sign | 7; /* nearest value of the set is 6 */
  /* For a <= 6 every difference below is exact in double precision. */
  int best = 0;
  double best_d = fabs(a - E2M1_MAGNITUDE[0]);
  for (int k = 1; k < 8; k++) {
    double d = fabs(a - E2M1_MAGNITUDE[k]);
    if (d < best_d || (d == best_d && (k % 2) == 0)) {
      best = k;
      best_d = d;
    }
  }
  return sign | best;
}

/* ---------------------------------------------------------------------- */
/* UE4M3 scale (R1): OCP E4M3 with bias 7, e = code>>3, m = code&7,  */
/* value = m * 2^-9 if e == 0 else (1 + m/8) * 2^(e-7); code 127 is NaN.    */
/* ---------------------------------------------------------------------- */
float so_e4m3_value(int code) {
  if (code < 0 || code > 126) return NAN;
  int e = code >> 3, m = code & 7;
  double v = (e == 0) ? ldexp((double)m, -9) : ldexp(1.0 + m / 8.0, e - 7);
  return (float)v; /* exact: at most 4 significant bits */
}

/* round_UE4M3 (Alg. 1 line 2): the finite code nearest v >= 0, ties
 * to the even code; v above the largest finite value 448 gives 448
 * (satfinite).  Codes 0..126 only (R2). */
int so_e4m3_encode(float v) {
  double a = (double)v;
  if (!(a >= 0.0)) return 0; /* negative or NaN never reach here */
  if (a >= 448.0) return 126;
  /* For a < 448 every difference below is exact in double precision. */
  int best = 0;
  double best_d = fabs(a - (double)so_e4m3_value(0));
  for (int c = 1; c <= 126; c++) {
    double d = fabs(a - (double)so_e4m3_value(c));
    if (d < best_d || (d == best_d && (c % 2) == 0)) {
      best = c;
      best_d = d;
    }
  }
  return best;
}

void so_e2m1_encode_array(const float* t, int64_t n, uint8_t* nib) {
  for (int64_t i = 0; i < n; i++) nib[i] = (uint8_t)so_e2m1_encode(t[i]);
}

void so_e4m3_encode_array(const float* v, int64_t n, uint8_t* code) {
  for (int64_t i = 0; i < n; i++) code[i] = (uint8_t)so_e4m3_encode(v[i]);
}

/* ---------------------------------------------------------------------- */
/* One candidate scale: quantize, dequantize, loss (Alg. 1 lines 7-9).     */
/* ---------------------------------------------------------------------- */
static float candidate_loss(const float y[16], float s, float rho, uint8_t nib[16]) {
  float d[16];
  for (int i = 0; i < 16; i++) {
    /* q_i = round_E2M1(x_i / s) (Alg. 1 line 7), with x_i / s computed as
     * x_i * RN(1/s) the way the vLLM kernel does (figVLLMnvf4; R7). */
    float t = y[i] * rho;
    nib[i] = (uint8_t)so_e2m1_encode(t);
    float q = (float)so_e2m1_value(nib[i]);
    /* xhat_i = q_i * s (line 8; exact: <= 6 significant bits) and the
     * residual x_i - xhat_i, rounded once. */
    d[i] = fmaf(-q, s, y[i]);
  }
  /* loss = sum_i (x_i - xhat_i)^2 (line 9) in the fixed order of R12:
   * two FMA chains, even indices and odd indices, then one add. */
  float a = d[0] * d[0];
  for (int i = 2; i < 16; i += 2) a = fmaf(d[i], d[i], a);
  float b = d[1] * d[1];
  for (int i = 3; i < 16; i += 2) b = fmaf(d[i], d[i], b);
  return a + b;
}

/* Algorithm 1, "NVFP4 Scale Search", with the readings R2-R5. */
int so_search_block(const float y[16], int fmin, int fmax, so_block_result* out) {
  if (fmin > 0 || fmax < 0) return 1;
  /* line 1: x_max = max_i |x_i| */
  float xmax = 0.0f;
  for (int i = 0; i < 16; i++)
    if (fabsf(y[i]) > xmax) xmax = fabsf(y[i]);
  /* line 2: s = round_UE4M3(x_max * (1.0/6.0)); 1/6 rounded once (R8) */
  const float one_sixth = 1.0f / 6.0f;
  float v = xmax * one_sixth;
  int c0 = so_e4m3_encode(v);
  /* line 3: s_int8 = reinterpret(s, int8) == c0.  line 4: l* = +inf. */
  int have = 0, cstar = -1, n_eval = 0;
  float best = INFINITY, base = NAN;
  uint8_t nib[16], best_nib[16] = {0};
  for (int f = fmin; f <= fmax; f++) { /* line 5 */
    int c = c0 + f;
    float s, rho;
    if (f == 0 && c0 == 0) {
      /* zero-scale candidate (R3): every value quantizes to 0. */
      s = 0.0f;
      rho = 0.0f;
    } else if (c < 1 || c > 126) {
      continue; /* line 6: scale out of range (127 is NaN, R2) */
    } else {
      s = so_e4m3_value(c); /* line 7: s^(f) = reinterpret(s_int8 + f) */
      rho = 1.0f / s;
    }
    float loss = candidate_loss(y, s, rho, nib);
    n_eval++;
    if (f == 0) base = loss;
    /* line 10: strict "<" while scanning f upward, so equal losses keep the
     * smaller scale (R4); the first valid candidate is always taken (R3). */
    if (!have || loss < best) {
      have = 1;
      best = loss;
      cstar = c;
      memcpy(best_nib, nib, 16);
    }
  }
  out->c0 = c0;
  out->cstar = cstar;
  out->fstar = cstar - c0; /* R5 */
  out->n_evaluated = n_eval;
  out->err_best = best;
  out->err_base = base;
  memcpy(out->nib, best_nib, 16);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Tensor level.                                                            */
/* ---------------------------------------------------------------------- */
static float bf16_to_float(uint16_t h) {
  /* bf16 is the top half of a binary32: the conversion is exact. */
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint32_t float_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}

static float bits_float(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* A = max |x| over the tensor ("dividing by the global scale from ...
 * tensor scaling"); non-finite input is an error (R14). */
int so_tensor_amax(const uint16_t* x, int64_t n, uint32_t* amax_bits) {
  float a = 0.0f;
  for (int64_t i = 0; i < n; i++) {
    float v = bf16_to_float(x[i]);
    if (!isfinite(v)) return 4;
    if (fabsf(v) > a) a = fabsf(v);
  }
  *amax_bits = float_bits(a);
  return 0;
}

/* G maps the tensor amax onto 6 * 448 = 2688, the largest NVFP4 magnitude
 * (figVLLMnvf4 P:126-129 SFScaleVal multiplies; R9). */
int so_global_scale(int gmode, uint32_t amax_bits, float* G) {
  if (gmode == 0) {
    *G = 1.0f;
    return 0;
  }
  float A = bits_float(amax_bits);
  if (!isfinite(A) || A < 0.0f) return 4;
  if (A == 0.0f) {
    *G = 1.0f;
    return 0;
  }
  float g = 2688.0f / A;
  if (!isfinite(g)) return 5;
  *G = g;
  return 0;
}

int so_quantize(const uint16_t* x, int64_t rows, int64_t cols, int fmin, int fmax,
                int gmode, const uint32_t* amax_bits_in, uint8_t* codes,
                uint8_t* scales, int8_t* offsets, float* err, double* sums,
                int64_t* n_eval, float* G_out, int threads) {
  if (rows < 0 || cols < 0 || cols % 16 != 0 || fmin > 0 || fmax < 0) return 1;
  if (gmode < 0 || gmode > 3 || (gmode == 2 && !amax_bits_in)) return 1;
  if (fmin < -126) fmin = -126;
  if (fmax > 126) fmax = 126;
  const int64_t nbr = cols / 16, nb = rows * nbr;
  /* Gr[r] = the global scale of row r.  Modes 0-2: one G for the tensor.
   * Mode 3 (ROW, "after per-row scaling"): every row is
   * its own tensor in the sense of mode 1, G_r = RN(2688 / max_k |x_rk|). */
  float* Gr = (float*)malloc(sizeof(float) * (rows > 0 ? rows : 1));
  float* e = (float*)malloc(sizeof(float) * 2 * (nb > 0 ? nb : 1));
  int32_t* ne = (int32_t*)malloc(sizeof(int32_t) * (nb > 0 ? nb : 1));
  if (!Gr || !e || !ne) {
    free(Gr);
    free(e);
    free(ne);
    return 1;
  }
  if (gmode == 3) {
    for (int64_t r = 0; r < rows; r++) {
      uint32_t ab = 0;
      int st = so_tensor_amax(x + r * cols, cols, &ab);
      if (!st) st = so_global_scale(1, ab, &Gr[r]);
      if (st) {
        free(Gr);
        free(e);
        free(ne);
        return st;
      }
    }
    if (G_out)
      for (int64_t r = 0; r < rows; r++) G_out[r] = Gr[r];
  } else {
    uint32_t amax_bits = 0;
    if (gmode == 1) {
      int st = so_tensor_amax(x, rows * cols, &amax_bits);
      if (st) {
        free(Gr);
        free(e);
        free(ne);
        return st;
      }
    } else if (gmode == 2) {
      amax_bits = *amax_bits_in;
    }
    float G;
    int st = so_global_scale(gmode, amax_bits, &G);
    if (st) {
      free(Gr);
      free(e);
      free(ne);
      return st;
    }
    if (G_out) *G_out = G;
    for (int64_t r = 0; r < rows; r++) Gr[r] = G;
  }
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_num_procs();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
#endif
  for (int64_t r = 0; r < rows; r++) {
    for (int64_t bj = 0; bj < nbr; bj++) {
      const int64_t blk = r * nbr + bj;
      float y[16];
      for (int i = 0; i < 16; i++) /* y = x * G (mode NONE: y = x exactly) */
        y[i] = (gmode == 0) ? bf16_to_float(x[r * cols + bj * 16 + i])
                            : bf16_to_float(x[r * cols + bj * 16 + i]) * Gr[r];
      so_block_result res;
      so_search_block(y, fmin, fmax, &res);
      for (int j = 0; j < 8; j++)
        codes[r * (cols / 2) + bj * 8 + j] =
            (uint8_t)(res.nib[2 * j] | (res.nib[2 * j + 1] << 4));
      scales[blk] = (uint8_t)res.cstar;
      if (offsets) offsets[blk] = (int8_t)res.fstar;
      e[2 * blk] = res.err_best;
      e[2 * blk + 1] = res.err_base;
      ne[blk] = res.n_evaluated;
    }
  }
  double sb = 0.0, s0 = 0.0;
  int64_t total = 0;
  for (int64_t b = 0; b < nb; b++) { /* FP64 sums in block order */
    sb += (double)e[2 * b];
    s0 += (double)e[2 * b + 1];
    total += ne[b];
  }
  if (err) memcpy(err, e, sizeof(float) * 2 * nb);
  if (sums) {
    sums[0] = sb;
    sums[1] = s0;
  }
  if (n_eval) *n_eval = total;
  free(Gr);
  free(e);
  free(ne);
  return 0;
}

/* Round a binary32 to the nearest bfloat16, ties to even: pick the nearer of
 * the two bf16 values that bracket v. */
static uint16_t float_to_bf16_rne(float v) {
  uint32_t u = float_bits(v);
  uint32_t lo = u & 0xFFFF0000u;           /* toward zero */
  uint32_t hi = lo + 0x00010000u;           /* next bf16 away from zero */
  double dv = (double)v;
  double dl = fabs(dv - (double)bits_float(lo));
  double dh = fabs((double)bits_float(hi) - dv);
  if ((u & 0xFFFFu) == 0) return (uint16_t)(lo >> 16);
  if (dl < dh) return (uint16_t)(lo >> 16);
  if (dh < dl) return (uint16_t)(hi >> 16);
  return ((lo >> 16) & 1) ? (uint16_t)(hi >> 16) : (uint16_t)(lo >> 16);
}

int so_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                  int64_t cols, float G, uint16_t* out) {
  if (rows < 0 || cols < 0 || cols % 16 != 0 || !(G > 0.0f)) return 1;
  const int64_t nbr = cols / 16;
  for (int64_t r = 0; r < rows; r++)
    for (int64_t k = 0; k < cols; k++) {
      uint8_t byte = codes[r * (cols / 2) + k / 2];
      int nib = (k % 2 == 0) ? (byte & 15) : (byte >> 4);
      float s = so_e4m3_value(scales[r * nbr + k / 16]);
      float q = (float)so_e2m1_value(nib);
      float xs = q * s; /* exact */
      out[r * cols + k] = float_to_bf16_rne(xs / G);
    }
  return 0;
}


/* ====================================================================== */
/* Other block formats ("the quantization and   */
/* dequantization algorithms are identical", P:301-308 format study).     */
/*   value formats: E2M1 (vmax 6) and E2M3 (MXFP6 values, vmax 7.5)        */
/*   scale formats: UE4M3 (codes 1..126, R2) and UE8M0 (2^(c-127),         */
/*                  codes 0..254; no zero, no NaN code 255)                */
/*   block size:    16 or 32                                               */
/* ====================================================================== */

/* E2M3 (1 sign, 2 exponent bits, bias 1, 3 mantissa bits): code = e<<3|m,
 * e = 0: m/8; else (1 + m/8) * 2^(e-1).  Largest 7.5. */
double so_e2m3_value(int code) {
  int mag = code & 31, e = mag >> 3, m = mag & 7;
  double v = (e == 0) ? m / 8.0 : ldexp(1.0 + m / 8.0, e - 1);
  return (code & 32) ? -v : v;
}

/* round_E2M3: nearest magnitude, ties to the even code, saturating at 7.5,
 * sign copied from t (as R10/R11 for E2M1). */
int so_e2m3_encode(float t) {
  int sign = signbit(t) ? 32 : 0;
  double a = fabs((double)t);
  if (a > 7.5) return sign | 31;
  int best = 0;
  double best_d = a;
  for (int k = 1; k < 32; k++) {
    double d = fabs(a - so_e2m3_value(k));
    if (d < best_d || (d == best_d && (k % 2) == 0)) {
      best = k;
      best_d = d;
    }
  }
  return sign | best;
}

/* UE8M0 scale value 2^(c - 127), c = 0..254. */
float so_ue8m0_value(int code) {
  if (code < 0 || code > 254) return NAN;
  return (float)ldexp(1.0, code - 127);
}

/* round_UE8M0 (R19): the smallest power of two >= v, saturating to
 * [2^-127, 2^127] (the format has no zero).  The paper only says the MXFP4
 * algorithm is "identical" with a UE8M0 scale; rounding the scale
 * up keeps x_max / s <= vmax (no clamping of the block maximum), is the
 * hardware conversion cvt.rp.satfinite.ue8m0x2.f32, and reproduces the
 * MXFP4 offset histogram of P:308 (two offsets, mostly 0). */
int so_ue8m0_encode(float v) {
  double a = (double)v;
  for (int c = 0; c <= 254; c++)
    if (ldexp(1.0, c - 127) >= a) return c;
  return 254;
}

static double fmt_value(int vfmt, int code) {
  return vfmt == 0 ? so_e2m1_value(code) : so_e2m3_value(code);
}
static int fmt_encode(int vfmt, float t) {
  return vfmt == 0 ? so_e2m1_encode(t) : so_e2m3_encode(t);
}
static float fmt_inv_vmax(int vfmt) {
  /* RN(1 / vmax) in binary32, the Alg. 1 line 2 form (R8) */
  return vfmt == 0 ? 1.0f / 6.0f : 1.0f / 7.5f;
}

/* One candidate of a `bs`-element block (bs = 16 * 2^k): quantize,
 * dequantize, loss.  The loss of each 16-element part is the R12 chain pair
 * (a over even, b over odd indices of the part, then a + b); the parts'
 * losses are added as a balanced pairwise tree: level 1 adds parts (0,1),
 * (2,3), ..., level 2 adds those sums pairwise, and so on (R20: for 32
 * elements simply low + high). */
static float fmt_candidate_loss(int vfmt, int bs, const float* y, float s, float rho,
                                uint8_t* code) {
  float part[16];
  const int np = bs / 16;
  for (int h = 0; h < np; h++) {
    float d[16];
    for (int i = 0; i < 16; i++) {
      float t = y[16 * h + i] * rho; /* R7 */
      code[16 * h + i] = (uint8_t)fmt_encode(vfmt, t);
      float q = (float)fmt_value(vfmt, code[16 * h + i]);
      d[i] = fmaf(-q, s, y[16 * h + i]);
    }
    float a = d[0] * d[0];
    for (int i = 2; i < 16; i += 2) a = fmaf(d[i], d[i], a);
    float b = d[1] * d[1];
    for (int i = 3; i < 16; i += 2) b = fmaf(d[i], d[i], b);
    part[h] = a + b;
  }
  for (int w = 1; w < np; w *= 2) /* pairwise tree */
    for (int h = 0; h < np; h += 2 * w) part[h] = part[h] + part[h + w];
  return part[0];
}

static int bs_ok(int bs) { return bs == 16 || bs == 32 || bs == 64 || bs == 128 || bs == 256; }

/* Algorithm 1 for one block of a format (vfmt, sfmt, bs): the NVFP4 rules
 * R2-R5 for UE4M3 scales; for UE8M0 every code 0..254 is a valid scale (there
 * is no zero-scale candidate) and c0 = round_UE8M0(x_max * RN(1/vmax)). */
int so_search_block_fmt(int vfmt, int sfmt, int bs, const float* y, int fmin, int fmax,
                        so_block_result_fmt* out) {
  if (fmin > 0 || fmax < 0 || !bs_ok(bs) || vfmt < 0 || vfmt > 1 || sfmt < 0 ||
      sfmt > 1)
    return 1;
  float xmax = 0.0f;
  for (int i = 0; i < bs; i++)
    if (fabsf(y[i]) > xmax) xmax = fabsf(y[i]);
  const float v = xmax * fmt_inv_vmax(vfmt);
  const int c0 = sfmt == 0 ? so_e4m3_encode(v) : so_ue8m0_encode(v);
  const int cmax = sfmt == 0 ? 126 : 254, cmin = sfmt == 0 ? 1 : 0;
  int have = 0, cstar = -1, n_eval = 0;
  float best = INFINITY, base = NAN;
  uint8_t code[256], best_code[256] = {0};
  for (int f = fmin; f <= fmax; f++) {
    int c = c0 + f;
    float s, rho;
    if (sfmt == 0 && f == 0 && c0 == 0) {
      s = 0.0f; /* R3 */
      rho = 0.0f;
    } else if (c < cmin || c > cmax) {
      continue;
    } else {
      s = sfmt == 0 ? so_e4m3_value(c) : so_ue8m0_value(c);
      rho = 1.0f / s;
    }
    float loss = fmt_candidate_loss(vfmt, bs, y, s, rho, code);
    n_eval++;
    if (f == 0) base = loss;
    if (!have || loss < best) { /* R4 */
      have = 1;
      best = loss;
      cstar = c;
      memcpy(best_code, code, (size_t)bs);
    }
  }
  out->c0 = c0;
  out->cstar = cstar;
  out->fstar = cstar - c0;
  out->n_evaluated = n_eval;
  out->err_best = best;
  out->err_base = base;
  memcpy(out->code, best_code, (size_t)bs);
  return 0;
}

/* Whole tensor in a format.  Codes: E2M1 packed two per byte (low nibble =
 * even element, R15) -> [rows][cols/2]; E2M3 one 6-bit code per byte (sign
 * bit 5) -> [rows][cols].  Scales [rows][cols/bs].  gmode: 0 NONE, 1 TENSOR,
 * 2 GIVEN, 3 ROW, as so_quantize, with G = RN(vmax * 448 / A) for UE4M3
 * scales; UE8M0 scales take gmode 0 only (their range needs no global scale). */
int so_quantize_fmt(const uint16_t* x, int64_t rows, int64_t cols, int fmin, int fmax,
                    int gmode, const uint32_t* amax_bits_in, int vfmt, int sfmt, int bs,
                    uint8_t* codes, uint8_t* scales, int8_t* offsets, float* err,
                    double* sums, int64_t* n_eval, float* G_out, int threads) {
  if (rows < 0 || cols < 0 || !bs_ok(bs) || cols % bs != 0 || fmin > 0 ||
      fmax < 0 || vfmt < 0 || vfmt > 1 || sfmt < 0 || sfmt > 1)
    return 1;
  if (gmode < 0 || gmode > 3 || (gmode == 2 && !amax_bits_in) || (sfmt == 1 && gmode != 0))
    return 1;
  const int lim = sfmt == 0 ? 126 : 254;
  if (fmin < -lim) fmin = -lim;
  if (fmax > lim) fmax = lim;
  const float numer = vfmt == 0 ? 2688.0f : 3360.0f; /* vmax * 448 */
  const int64_t nbr = cols / bs, nb = rows * nbr;
  float* Gr = (float*)malloc(sizeof(float) * (rows > 0 ? rows : 1));
  float* e = (float*)malloc(sizeof(float) * 2 * (nb > 0 ? nb : 1));
  int32_t* ne = (int32_t*)malloc(sizeof(int32_t) * (nb > 0 ? nb : 1));
  if (!Gr || !e || !ne) {
    free(Gr);
    free(e);
    free(ne);
    return 1;
  }
  int st = 0;
  for (int64_t r = 0; r < rows && !st; r++) Gr[r] = 1.0f;
  if (gmode == 3) {
    for (int64_t r = 0; r < rows && !st; r++) {
      uint32_t ab = 0;
      st = so_tensor_amax(x + r * cols, cols, &ab);
      float A;
      memcpy(&A, &ab, 4);
      if (!st && A > 0.0f) {
        Gr[r] = numer / A;
        if (!isfinite(Gr[r])) st = 5;
      }
    }
    if (!st && G_out)
      for (int64_t r = 0; r < rows; r++) G_out[r] = Gr[r];
  } else if (gmode == 1 || gmode == 2) {
    uint32_t ab = 0;
    if (gmode == 1)
      st = so_tensor_amax(x, rows * cols, &ab);
    else
      ab = *amax_bits_in;
    float A;
    memcpy(&A, &ab, 4);
    if (!st && !(A >= 0.0f && isfinite(A))) st = 4;
    float G = 1.0f;
    if (!st && A > 0.0f) {
      G = numer / A;
      if (!isfinite(G)) st = 5;
    }
    for (int64_t r = 0; r < rows; r++) Gr[r] = G;
    if (!st && G_out) *G_out = G;
  } else if (G_out) {
    *G_out = 1.0f;
  }
  if (st) {
    free(Gr);
    free(e);
    free(ne);
    return st;
  }
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_num_procs();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
#endif
  for (int64_t r = 0; r < rows; r++) {
    for (int64_t bj = 0; bj < nbr; bj++) {
      const int64_t blk = r * nbr + bj;
      float y[256];
      for (int i = 0; i < bs; i++) {
        float xv = bf16_to_float(x[r * cols + bj * bs + i]);
        y[i] = (gmode == 0) ? xv : xv * Gr[r];
      }
      so_block_result_fmt res;
      so_search_block_fmt(vfmt, sfmt, bs, y, fmin, fmax, &res);
      if (vfmt == 0) {
        for (int j = 0; j < bs / 2; j++)
          codes[r * (cols / 2) + bj * (bs / 2) + j] =
              (uint8_t)(res.code[2 * j] | (res.code[2 * j + 1] << 4));
      } else {
        for (int j = 0; j < bs; j++) codes[r * cols + bj * bs + j] = res.code[j];
      }
      scales[blk] = (uint8_t)res.cstar;
      if (offsets) offsets[blk] = (int8_t)res.fstar;
      e[2 * blk] = res.err_best;
      e[2 * blk + 1] = res.err_base;
      ne[blk] = res.n_evaluated;
    }
  }
  double sb = 0.0, s0 = 0.0;
  int64_t total = 0;
  for (int64_t b = 0; b < nb; b++) {
    sb += (double)e[2 * b];
    s0 += (double)e[2 * b + 1];
    total += ne[b];
  }
  if (err) memcpy(err, e, sizeof(float) * 2 * nb);
  if (sums) {
    sums[0] = sb;
    sums[1] = s0;
  }
  if (n_eval) *n_eval = total;
  free(Gr);
  free(e);
  free(ne);
  return 0;
}

/* Dequantization in a format: xhat = RNE_bf16(RN((q * s) / G_r)) with the
 * code layout of so_quantize_fmt; G has one entry, or `rows` when per_row. */
int so_dequantize_fmt(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols,
                      int vfmt, int sfmt, int bs, const float* G, int per_row, uint16_t* out) {
  if (rows < 0 || cols < 0 || !bs_ok(bs) || cols % bs != 0) return 1;
  const int64_t nbr = cols / bs;
  for (int64_t r = 0; r < rows; r++) {
    const float g = per_row ? G[r] : G[0];
    if (!(g > 0.0f)) return 1;
    for (int64_t k = 0; k < cols; k++) {
      int code;
      if (vfmt == 0) {
        uint8_t byte = codes[r * (cols / 2) + k / 2];
        code = (k % 2 == 0) ? (byte & 15) : (byte >> 4);
      } else {
        code = codes[r * cols + k] & 63;
      }
      const int sc = scales[r * nbr + k / bs];
      const float s = sfmt == 0 ? so_e4m3_value(sc) : so_ue8m0_value(sc);
      const float q = (float)(vfmt == 0 ? so_e2m1_value(code) : so_e2m3_value(code));
      out[r * cols + k] = float_to_bf16_rne((q * s) / g);
    }
  }
  return 0;
}


/* ====================================================================== */
/* Generic ExMy block formats (fig:nvfp-scale,            */
/* fig:nvfp-val, fig:mxfp P:237-260, "hypothetical block quantization     */
/* formats having different scale representation bits ... value           */
/* representation bits" P:301-303).  Reading R21:          */
/*  value format ExMy (e >= 1): sign bit above e+m magnitude bits, bias    */
/*    2^(e-1)-1, E = 0 subnormal M * 2^(1-bias-m), else                    */
/*    (2^m + M) * 2^(E-bias-m); every code finite (the OCP FP4/FP6 rule).   */
/*  scale format UExMy (unsigned): the all-ones code is NaN (as E4M3 0x7F, */
/*    E8M0 0xFF).  m >= 1: IEEE-like with subnormals, code 0 = the zero    */
/*    scale (R3); c0 = nearest code, ties to the even code, satfinite (the */
/*    UE4M3 rule, Alg. 1 line 2).  m = 0: pure powers of two 2^(c-bias),    */
/*    no zero; c0 = the smallest power of two >= v (R19, the UE8M0 rule).  */
/*  x_max -> v = RN(x_max * RN(1/vmax)) (R8); global scale numerator       */
/*    vmax * smax (2688 for NVFP4, R9).                                     */
/* Rounding is by enumerating the format's values (no bit tricks).         */
/* ====================================================================== */

/* magnitude of code c of an ExMy grid; m == 0 && pow2: 2^(c - bias) */
static double gen_mag(int e, int m, int c, int pow2) {
  const int bias = (1 << (e - 1)) - 1;
  if (pow2) return ldexp(1.0, c - bias);
  const int E = c >> m, M = c & ((1 << m) - 1);
  if (E == 0) return ldexp((double)M, 1 - bias - m);
  return ldexp((double)((1 << m) + M), E - bias - m);
}

static int gen_fmt_ok(int ve, int vm, int se, int sm) {
  /* values: sign + e + m <= 8 bits; scales: e + m <= 8 bits and every finite
   * scale, times vmax, inside binary32 */
  if (ve < 1 || vm < 0 || ve + vm > 7) return 0;
  if (se < 1 || sm < 0 || se + sm > 8) return 0;
  if (sm > 0 && se > 7) return 0;
  return 1;
}

double so_gen_value(int e, int m, int code) {
  const int nmag = 1 << (e + m);
  if (code < 0 || code >= 2 * nmag) return NAN;
  const double v = gen_mag(e, m, code & (nmag - 1), 0);
  return (code & nmag) ? -v : v;
}

/* nearest magnitude to |t| (ties to the even code), saturating at the
 * largest value; sign bit from t (R10, R11). */
int so_gen_encode(int e, int m, float t) {
  const int nmag = 1 << (e + m);
  const int sign = signbit(t) ? nmag : 0;
  const double a = fabs((double)t);
  const double vmax = gen_mag(e, m, nmag - 1, 0);
  if (a >= vmax) return sign | (nmag - 1); /* satfinite (and +-inf) */
  int best = 0;
  double best_d = a;
  for (int k = 1; k < nmag; k++) {
    const double d = fabs(a - gen_mag(e, m, k, 0));
    if (d < best_d || (d == best_d && (k % 2) == 0)) {
      best = k;
      best_d = d;
    }
  }
  return sign | best;
}

double so_gen_scale_value(int e, int m, int code) {
  const int ncode = 1 << (e + m);
  if (code < 0 || code >= ncode - 1) return NAN; /* all ones: NaN */
  return gen_mag(e, m, code, m == 0);
}

int so_gen_scale_encode(int e, int m, float v) {
  const int maxc = (1 << (e + m)) - 2;
  const double a = (double)v;
  if (m == 0) { /* R19: smallest power of two >= v, saturating */
    for (int c = 0; c <= maxc; c++)
      if (gen_mag(e, m, c, 1) >= a) return c;
    return maxc;
  }
  if (a >= gen_mag(e, m, maxc, 0)) return maxc; /* satfinite */
  int best = 0;
  double best_d = fabs(a);
  for (int c = 1; c <= maxc; c++) {
    const double d = fabs(a - gen_mag(e, m, c, 0));
    if (d < best_d || (d == best_d && (c % 2) == 0)) {
      best = c;
      best_d = d;
    }
  }
  return best;
}

/* RN(vmax * smax): the global-scale numerator of a format (R9, R21) */
float so_gen_numer(int ve, int vm, int se, int sm) {
  const float vmax = (float)gen_mag(ve, vm, (1 << (ve + vm)) - 1, 0);
  const float smax = (float)gen_mag(se, sm, (1 << (se + sm)) - 2, sm == 0);
  return vmax * smax;
}

/* One candidate (Alg. 1 lines 6-9) of a bs-element block in an ExMy value
 * format: t = RN(y * rho) (R7), q = round(t), d = RN(y - q*s) (q*s exact),
 * R12 chains per 16-element part, parts added as the R20 pairwise tree. */
static float gen_candidate_loss(int ve, int vm, int bs, const float* y, float s, float rho,
                                uint8_t* code) {
  float part[16];
  const int np = bs / 16;
  for (int h = 0; h < np; h++) {
    float d[16];
    for (int i = 0; i < 16; i++) {
      float t = y[16 * h + i] * rho;
      code[16 * h + i] = (uint8_t)so_gen_encode(ve, vm, t);
      float q = (float)so_gen_value(ve, vm, code[16 * h + i]);
      d[i] = fmaf(-q, s, y[16 * h + i]);
    }
    float a = d[0] * d[0];
    for (int i = 2; i < 16; i += 2) a = fmaf(d[i], d[i], a);
    float b = d[1] * d[1];
    for (int i = 3; i < 16; i += 2) b = fmaf(d[i], d[i], b);
    part[h] = a + b;
  }
  for (int w = 1; w < np; w *= 2)
    for (int h = 0; h < np; h += 2 * w) part[h] = part[h] + part[h + w];
  return part[0];
}

/* Algorithm 1 for one block of a generic format: scan f
 * ascending over valid codes (UExMy m >= 1: 1..maxc plus the zero scale at
 * c0 = 0, f = 0; m = 0: 0..maxc), strict "<" (ties keep the smaller code). */
int so_search_block_gen(int ve, int vm, int se, int sm, int bs, const float* y, int fmin,
                        int fmax, so_block_result_fmt* out) {
  if (fmin > 0 || fmax < 0 || !bs_ok(bs) || !gen_fmt_ok(ve, vm, se, sm)) return 1;
  const int maxc = (1 << (se + sm)) - 2, cmin = sm == 0 ? 0 : 1;
  const float vmax = (float)gen_mag(ve, vm, (1 << (ve + vm)) - 1, 0);
  const float kinv = 1.0f / vmax; /* RN(1/vmax), R8 */
  float xmax = 0.0f;
  for (int i = 0; i < bs; i++)
    if (fabsf(y[i]) > xmax) xmax = fabsf(y[i]);
  const int c0 = so_gen_scale_encode(se, sm, xmax * kinv);
  int have = 0, cstar = -1, n_eval = 0;
  float best = INFINITY, base = NAN;
  uint8_t code[256], best_code[256] = {0};
  for (int f = fmin; f <= fmax; f++) {
    const int c = c0 + f;
    float s, rho;
    if (sm > 0 && f == 0 && c0 == 0) {
      s = 0.0f; /* R3 */
      rho = 0.0f;
    } else if (c < cmin || c > maxc) {
      continue;
    } else {
      s = (float)so_gen_scale_value(se, sm, c);
      rho = 1.0f / s;
    }
    const float loss = gen_candidate_loss(ve, vm, bs, y, s, rho, code);
    n_eval++;
    if (f == 0) base = loss;
    if (!have || loss < best) {
      have = 1;
      best = loss;
      cstar = c;
      memcpy(best_code, code, (size_t)bs);
    }
  }
  out->c0 = c0;
  out->cstar = cstar;
  out->fstar = cstar - c0;
  out->n_evaluated = n_eval;
  out->err_best = best;
  out->err_base = base;
  memcpy(out->code, best_code, (size_t)bs);
  return 0;
}

/* Whole tensor in a generic format.  codes [rows][cols], one value code per
 * byte; scales [rows][cols/bs]; gmode 0 NONE, 1 TENSOR, 2 GIVEN (amax bits),
 * with G = RN(numer / A), numer = so_gen_numer. */
int so_quantize_gen(const uint16_t* x, int64_t rows, int64_t cols, int fmin, int fmax,
                    int gmode, const uint32_t* amax_bits_in, int ve, int vm, int se, int sm,
                    int bs, uint8_t* codes, uint8_t* scales, int8_t* offsets, float* err,
                    double* sums, int64_t* n_eval, float* G_out, int threads) {
  if (rows < 0 || cols < 0 || !bs_ok(bs) || cols % bs != 0 || fmin > 0 || fmax < 0 ||
      !gen_fmt_ok(ve, vm, se, sm) || gmode < 0 || gmode > 2 || (gmode == 2 && !amax_bits_in))
    return 1;
  const int lim = (1 << (se + sm)) - 2;
  if (fmin < -lim) fmin = -lim;
  if (fmax > lim) fmax = lim;
  const float numer = so_gen_numer(ve, vm, se, sm);
  if (gmode != 0 && !isfinite(numer)) return 1; /* vmax * smax beyond binary32 (e.g. UE8M0) */
  float G = 1.0f;
  if (gmode != 0) {
    uint32_t ab = 0;
    int st = 0;
    if (gmode == 1)
      st = so_tensor_amax(x, rows * cols, &ab);
    else
      ab = *amax_bits_in;
    if (st) return st;
    const float A = bits_float(ab);
    if (!(A >= 0.0f && isfinite(A))) return 4;
    if (A > 0.0f) {
      G = numer / A;
      if (!isfinite(G)) return 5;
    }
  }
  if (G_out) *G_out = G;
  const int64_t nbr = cols / bs, nb = rows * nbr;
  float* e = (float*)malloc(sizeof(float) * 2 * (nb > 0 ? nb : 1));
  int32_t* ne = (int32_t*)malloc(sizeof(int32_t) * (nb > 0 ? nb : 1));
  if (!e || !ne) {
    free(e);
    free(ne);
    return 1;
  }
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_num_procs();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
#endif
  for (int64_t r = 0; r < rows; r++) {
    for (int64_t bj = 0; bj < nbr; bj++) {
      const int64_t blk = r * nbr + bj;
      float y[256];
      for (int i = 0; i < bs; i++) {
        const float xv = bf16_to_float(x[r * cols + bj * bs + i]);
        y[i] = gmode == 0 ? xv : xv * G;
      }
      so_block_result_fmt res;
      so_search_block_gen(ve, vm, se, sm, bs, y, fmin, fmax, &res);
      for (int j = 0; j < bs; j++) codes[r * cols + bj * bs + j] = res.code[j];
      scales[blk] = (uint8_t)res.cstar;
      if (offsets) offsets[blk] = (int8_t)(res.fstar < -128 ? -128 : (res.fstar > 127 ? 127 : res.fstar));
      e[2 * blk] = res.err_best;
      e[2 * blk + 1] = res.err_base;
      ne[blk] = res.n_evaluated;
    }
  }
  double sb = 0.0, s0 = 0.0;
  int64_t total = 0;
  for (int64_t b = 0; b < nb; b++) {
    sb += (double)e[2 * b];
    s0 += (double)e[2 * b + 1];
    total += ne[b];
  }
  if (err) memcpy(err, e, sizeof(float) * 2 * nb);
  if (sums) {
    sums[0] = sb;
    sums[1] = s0;
  }
  if (n_eval) *n_eval = total;
  free(e);
  free(ne);
  return 0;
}

/* xhat = RNE_bf16(RN((q * s) / G)) for the code layout of so_quantize_gen. */
int so_dequantize_gen(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols,
                      int ve, int vm, int se, int sm, int bs, float G, uint16_t* out) {
  if (rows < 0 || cols < 0 || !bs_ok(bs) || cols % bs != 0 || !gen_fmt_ok(ve, vm, se, sm) ||
      !(G > 0.0f))
    return 1;
  const int64_t nbr = cols / bs;
  for (int64_t r = 0; r < rows; r++)
    for (int64_t k = 0; k < cols; k++) {
      const float q = (float)so_gen_value(ve, vm, codes[r * cols + k]);
      const int sc = scales[r * nbr + k / bs];
      const float s = (sm > 0 && sc == 0) ? 0.0f : (float)so_gen_scale_value(se, sm, sc);
      out[r * cols + k] = float_to_bf16_rne((q * s) / G);
    }
  return 0;
}
