/*
 * attn_oracle.c — plain, slow, obviously-correct fp64 attention (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: nothing in the product path links or calls this file.
 * It shares no code, header, table or constant with paper_2504_17577_b200/csrc.
 *
 * Each function cites the passage it follows:
 *   - definition of the result: exact softmax attention, PAPER.md P:L424 (ref [12]);
 *     the online recurrence of Fig. 18 computes the same value, so the
 *     oracle is the plain two-pass definition (max, exp, sum, normalise), fp64.
 *   - GQA head grouping: cur_kv_head = by // (kv_group_num // block_H)
 *     -> g = h / (Hq / Hkv) (reading R7).
 *   - causal flag: Table 3; alignment is bottom-right (R3).
 *   - tensor layout KV[batch, seqlen_kv, kv_head_num, dim], P:L583 (R6).
 * Build: gcc -O2 (no -ffast-math), single-threaded, libm only.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* IEEE binary16 / bfloat16 -> double, exact (every 16-bit value is a double). */
double oracle_widen(uint16_t bits, int dtype) {
  if (dtype == ORACLE_BF16) {
    /* bfloat16 is the top half of an IEEE binary32. */
    uint32_t u = ((uint32_t)bits) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
  }
  /* binary16: 1 sign, 5 exponent (bias 15), 10 mantissa bits. */
  int sign = (bits >> 15) & 1;
  int e = (bits >> 10) & 0x1f;
  int m = bits & 0x3ff;
  double mag;
  if (e == 0) {
    mag = ldexp((double)m, -24); /* subnormal: m * 2^-24 */
  } else if (e == 31) {
    mag = (m == 0) ? INFINITY : NAN;
  } else {
    mag = ldexp((double)(1024 + m), e - 25); /* (1 + m/1024) * 2^(e-15) */
  }
  return sign ? -mag : mag;
}

static int check_args(int dtype, long B, long Hq, long Hkv, long Sq, long Skv, long D,
                      int causal) {
  if (dtype != ORACLE_F16 && dtype != ORACLE_BF16) return 1;
  if (B < 1 || Hq < 1 || Hkv < 1 || Sq < 1 || Skv < 1 || D < 1) return 1;
  if (Hq % Hkv != 0) return 1;
  if (causal != 0 && causal != 1) return 1;
  return 0;
}

/* Index of element (b, s, h, d) in a contiguous BSHD tensor. */
static long bshd(long b, long s, long h, long d, long S, long H, long D) {
  return ((b * S + s) * H + h) * D + d;
}

/* Is key j allowed for query row i?  J_i = { j < Skv : !causal || j <= i + Skv - Sq }. */
static int allowed(long i, long j, long Sq, long Skv, int causal) {
  if (j >= Skv) return 0;
  if (causal && j > i + Skv - Sq) return 0;
  return 1;
}

int oracle_attn_rows(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                     long B, long Hq, long Hkv, long Sq, long Skv, long D,
                     int causal, double scale, long b, long h,
                     const long* rows, long nrows, double* o_out, double* lse_out) {
  if (!q || !k || !v || !o_out || (nrows > 0 && !rows)) return 1;
  if (check_args(dtype, B, Hq, Hkv, Sq, Skv, D, causal)) return 1;
  if (b < 0 || b >= B || h < 0 || h >= Hq || nrows < 0) return 1;
  for (long r = 0; r < nrows; ++r)
    if (rows[r] < 0 || rows[r] >= Sq) return 1;

  const long g = h / (Hq / Hkv);
  double* s = (double*)malloc(sizeof(double) * (size_t)Skv);
  double* qd = (double*)malloc(sizeof(double) * (size_t)D);
  if (!s || !qd) { free(s); free(qd); return 1; }

  for (long r = 0; r < nrows; ++r) {
    const long i = rows[r];
    double* o = o_out + r * D;
    for (long d = 0; d < D; ++d) qd[d] = oracle_widen(q[bshd(b, i, h, d, Sq, Hq, D)], dtype);

    /* pass 1: scores s_j = scale * sum_d q_d k_{j,d} (sequential d), and their max */
    double m = -INFINITY;
    long nallowed = 0;
    for (long j = 0; j < Skv; ++j) {
      if (!allowed(i, j, Sq, Skv, causal)) continue;
      double acc = 0.0;
      for (long d = 0; d < D; ++d) acc += qd[d] * oracle_widen(k[bshd(b, j, g, d, Skv, Hkv, D)], dtype);
      s[j] = scale * acc;
      if (s[j] > m) m = s[j];
      ++nallowed;
    }
    if (nallowed == 0) { /* DESIGN.md R4: empty key set */
      for (long d = 0; d < D; ++d) o[d] = 0.0;
      if (lse_out) lse_out[r] = -INFINITY;
      continue;
    }
    /* pass 2: w_j = exp(s_j - m), l = sum w_j, o = sum w_j v_j / l, lse = m + log l */
    double l = 0.0;
    for (long d = 0; d < D; ++d) o[d] = 0.0;
    for (long j = 0; j < Skv; ++j) {
      if (!allowed(i, j, Sq, Skv, causal)) continue;
      double w = exp(s[j] - m);
      l += w;
      for (long d = 0; d < D; ++d) o[d] += w * oracle_widen(v[bshd(b, j, g, d, Skv, Hkv, D)], dtype);
    }
    for (long d = 0; d < D; ++d) o[d] /= l;
    if (lse_out) lse_out[r] = m + log(l);
  }
  free(s);
  free(qd);
  return 0;
}

int oracle_attn_full(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                     long B, long Hq, long Hkv, long Sq, long Skv, long D,
                     int causal, double scale, double* o_out, double* lse_out) {
  if (!o_out) return 1;
  if (check_args(dtype, B, Hq, Hkv, Sq, Skv, D, causal)) return 1;
  long* rows = (long*)malloc(sizeof(long) * (size_t)Sq);
  double* o = (double*)malloc(sizeof(double) * (size_t)(Sq * D));
  if (!rows || !o) { free(rows); free(o); return 1; }
  for (long i = 0; i < Sq; ++i) rows[i] = i;
  int rc = 0;
  for (long b = 0; b < B && !rc; ++b) {
    for (long h = 0; h < Hq && !rc; ++h) {
      double* lse = lse_out ? lse_out + (b * Hq + h) * Sq : NULL;
      rc = oracle_attn_rows(q, k, v, dtype, B, Hq, Hkv, Sq, Skv, D, causal, scale, b, h,
                            rows, Sq, o, lse);
      for (long i = 0; i < Sq && !rc; ++i)
        for (long d = 0; d < D; ++d) o_out[bshd(b, i, h, d, Sq, Hq, D)] = o[i * D + d];
    }
  }
  free(rows);
  free(o);
  return rc;
}

int oracle_brute_force(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                       long B, long Hq, long Hkv, long Sq, long Skv, long D,
                       int causal, double scale, long b, long h,
                       double* s_out, double* p_out, double* o_out, double* lse_out) {
  if (!q || !k || !v || !o_out) return 1;
  if (check_args(dtype, B, Hq, Hkv, Sq, Skv, D, causal)) return 1;
  if (b < 0 || b >= B || h < 0 || h >= Hq) return 1;
  const long g = h / (Hq / Hkv);
  double* S = (double*)malloc(sizeof(double) * (size_t)(Sq * Skv));
  double* P = (double*)malloc(sizeof(double) * (size_t)(Sq * Skv));
  if (!S || !P) { free(S); free(P); return 1; }

  /* S = scale * Q K^T as an explicit matrix, -inf where masked */
  for (long i = 0; i < Sq; ++i)
    for (long j = 0; j < Skv; ++j) {
      if (!allowed(i, j, Sq, Skv, causal)) { S[i * Skv + j] = -INFINITY; continue; }
      double acc = 0.0;
      for (long d = 0; d < D; ++d)
        acc += oracle_widen(q[bshd(b, i, h, d, Sq, Hq, D)], dtype) *
               oracle_widen(k[bshd(b, j, g, d, Skv, Hkv, D)], dtype);
      S[i * Skv + j] = scale * acc;
    }
  /* P_ij = 1 / sum_k exp(s_ik - s_ij): no max subtraction, different algebra */
  for (long i = 0; i < Sq; ++i)
    for (long j = 0; j < Skv; ++j) {
      double sij = S[i * Skv + j];
      if (sij == -INFINITY) { P[i * Skv + j] = 0.0; continue; }
      long double den = 0.0L;
      for (long kk = 0; kk < Skv; ++kk) {
        double sik = S[i * Skv + kk];
        if (sik == -INFINITY) continue;
        den += expl((long double)sik - (long double)sij);
      }
      P[i * Skv + j] = (double)(1.0L / den);
    }
  /* O = P V (explicit matrix product); lse_i = s_ij* - log P_ij* with j* = argmax_j P_ij
     (since P_ij = exp(s_ij) / sum_k exp(s_ik), log sum_k exp(s_ik) = s_ij - log P_ij) */
  for (long i = 0; i < Sq; ++i) {
    for (long d = 0; d < D; ++d) {
      long double acc = 0.0L;
      for (long j = 0; j < Skv; ++j)
        acc += (long double)P[i * Skv + j] * (long double)oracle_widen(v[bshd(b, j, g, d, Skv, Hkv, D)], dtype);
      o_out[i * D + d] = (double)acc;
    }
    if (lse_out) {
      long jstar = -1;
      for (long j = 0; j < Skv; ++j)
        if (P[i * Skv + j] > 0.0 && (jstar < 0 || P[i * Skv + j] > P[i * Skv + jstar])) jstar = j;
      lse_out[i] = (jstar < 0) ? -INFINITY : S[i * Skv + jstar] - log(P[i * Skv + jstar]);
    }
  }
  if (s_out) memcpy(s_out, S, sizeof(double) * (size_t)(Sq * Skv));
  if (p_out) memcpy(p_out, P, sizeof(double) * (size_t)(Sq * Skv));
  free(S);
  free(P);
  return 0;
}
