/*
 * brute_nvfp4.c -- an independent exhaustive NVFP4 block search, used only by
 * tests/test_oracle_bruteforce.py to pin the oracle (oracle/ss_oracle.c).
 *
 * Written separately from the oracle on purpose: no shared code, header or
 * table, and a different technique at every step where one exists --
 *   - UE4M3 scale values are assembled from their bit fields (the oracle
 *     evaluates (1 + m/8) * 2^(e-7) with ldexp);
 *   - the max-abs scale code c0 is rounded by frexpf + nearbyintf on the
 *     scaled mantissa (the oracle enumerates all 127 codes);
 *   - E2M1 rounding compares |t| against the seven decision thresholds with
 *     the tie direction of each spelled out (the oracle enumerates the grid);
 *   - the search visits every code 0..126 of the window and keeps the
 *     lexicographic minimum of (loss, code) (the oracle scans f upward with
 *     a strict "<").
 * The arithmetic contract is the paper's Algorithm 1 with the
 * DESIGN.md readings: t = RN(y * RN(1/s)) (R7), d = RN(y - q*s) as one fmaf
 * (exact product), loss = RN(a + b) over the even / odd fmaf chains (R12),
 * c0 = RNE_satfinite(RN(m * RN(1/6))) (R8), the zero-scale candidate when
 * c0 == 0 (R3), codes 1..126 (R2).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float from_bits(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* UE4M3 code 1..126 -> value: normal codes (exponent field >= 1) are the
 * binary32 with exponent field + 120 and the 3 mantissa bits on top;
 * subnormal codes 1..7 are c * 2^-9. */
static float scale_value(int c) {
  if (c >= 8) return from_bits((uint32_t)(((c >> 3) + 120) << 23) | ((uint32_t)(c & 7) << 20));
  return ldexpf((float)c, -9);
}

/* round-to-nearest-even into UE4M3 codes 0..126, satfinite */
static int scale_code(float v) {
  if (!(v > 0.0f)) return 0;
  int e;
  float m = frexpf(v, &e); /* v = m * 2^e, m in [0.5, 1) */
  e -= 1;                   /* v = (2m) * 2^e, 2m in [1, 2) */
  int code;
  if (e < -6) {
    code = (int)nearbyintf(v * 512.0f); /* subnormal quantum 2^-9: exact scaling */
  } else {
    int q = (int)nearbyintf(2.0f * m * 8.0f); /* 8..16, ties to even */
    code = ((e + 7) << 3) + (q - 8);          /* q == 16 carries into the next binade */
  }
  return code > 126 ? 126 : code;
}

/* E2M1 round-to-nearest-even, saturating, sign kept (R10, R11): returns the
 * signed value and the nibble. */
static float e2m1(float t, int* nib) {
  float a = fabsf(t);
  int k;            /* magnitude code: 0..7 = 0, .5, 1, 1.5, 2, 3, 4, 6 */
  if (a <= 0.25f) k = 0;        /* tie .25 -> 0 (even) */
  else if (a < 0.75f) k = 1;    /* tie .75 -> 1.0 (even) */
  else if (a <= 1.25f) k = 2;   /* tie 1.25 -> 1.0 */
  else if (a < 1.75f) k = 3;    /* tie 1.75 -> 2.0 */
  else if (a <= 2.5f) k = 4;    /* tie 2.5 -> 2.0 */
  else if (a < 3.5f) k = 5;     /* tie 3.5 -> 4.0 */
  else if (a <= 5.0f) k = 6;    /* tie 5 -> 4.0 */
  else k = 7;                   /* above 5, incl. > 6: saturate to 6 */
  static const float mag[8] = {0.0f, 0.5f, 1.0f, 1.5f, 2.0f, 3.0f, 4.0f, 6.0f};
  int neg = signbit(t) != 0;
  *nib = (neg << 3) | k;
  return neg ? -mag[k] : mag[k];
}

static float loss_of(const float* y, float s, float rho, uint8_t* nib) {
  float d[16];
  for (int i = 0; i < 16; i++) {
    int n;
    float q = e2m1(y[i] * rho, &n);
    nib[i] = (uint8_t)n;
    d[i] = fmaf(-q, s, y[i]);
  }
  float a = d[0] * d[0], b = d[1] * d[1];
  for (int i = 2; i < 16; i += 2) a = fmaf(d[i], d[i], a);
  for (int i = 3; i < 16; i += 2) b = fmaf(d[i], d[i], b);
  return a + b;
}

/* For each of n blocks y[16]: out_c0, out_cstar, out_best / out_base (loss
 * bits as floats), out_nib[16] (winner nibbles). */
void brute_search(const float* y, int64_t n, int fmin, int fmax, int32_t* out_c0, int32_t* out_cstar,
                  float* out_best, float* out_base, uint8_t* out_nib) {
  const float k6 = 1.0f / 6.0f;
  for (int64_t b = 0; b < n; b++) {
    const float* x = y + 16 * b;
    float m = 0.0f;
    for (int i = 0; i < 16; i++) m = fmaxf(m, fabsf(x[i]));
    const int c0 = scale_code(m * k6);
    int lo = c0 + fmin, hi = c0 + fmax;
    if (lo < 0) lo = 0;
    if (hi > 126) hi = 126;
    float best = 0.0f, base = NAN;
    int cstar = -1;
    uint8_t nib[16], bn[16];
    for (int c = lo; c <= hi; c++) {
      float s, rho;
      if (c == 0) {
        if (c0 != 0) continue; /* code 0 is only the zero-scale candidate of c0 == 0 */
        s = 0.0f;
        rho = 0.0f;
      } else {
        s = scale_value(c);
        rho = 1.0f / s;
      }
      const float l = loss_of(x, s, rho, nib);
      if (c == c0) base = l;
      if (cstar < 0 || l < best || (l == best && c < cstar)) { /* lexicographic (loss, code) */
        best = l;
        cstar = c;
        memcpy(bn, nib, 16);
      }
    }
    out_c0[b] = c0;
    out_cstar[b] = cstar;
    out_best[b] = best;
    out_base[b] = base;
    memcpy(out_nib + 16 * b, bn, 16);
  }
}
