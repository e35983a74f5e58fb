/*
 * mla_oracle.c — plain, slow, obviously-correct fp64 MLA decode attention (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: nothing in the product path links or calls this file.
 * It shares no code, header, table or constant with paper_2504_17577_b200/csrc.
 *
 * What it follows: PAPER.md Appendix B.3, Fig. 18 "FlashMLA":
 *   - tensors Q[batch, heads, dim], Q_pe[batch, heads, pe_dim], KV[batch, seqlen_kv,
 *     kv_head_num, dim], K_pe[batch, seqlen_kv, kv_head_num, pe_dim], Output[batch,
 *     heads, dim];
 *   - scores = Q KV^T + Q_pe K_pe^T: two T.gemm calls into the same acc_s;
 *   - softmax over the keys and O = softmax . KV: the value operand of the
 *     second T.gemm is KV_shared itself, i.e. V = KV (the latent cache);
 *   - kv head of query head h: cur_kv_head = by // (kv_group_num // block_H)
 *     -> g = h / (H / Hkv) (reading R7 / M2).
 * The Fig. 18 loop is the online (running max / sum) form; this oracle evaluates the plain
 * two-pass definition it computes exactly: max, exp, sum, normalise, in fp64.
 * Reading M1: Fig. 18 has one seqlen_kv for all batches; the ABI adds an
 * optional per-batch cache length n_b <= Skv (keys j >= n_b do not take part). n_b = 0
 * gives o = 0 and lse = -inf (as R4 for empty key sets).
 * Build: gcc -O2 (no -ffast-math), single-threaded, libm only.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>

static int mla_check(int dtype, long B, long H, long Hkv, long Skv, long Dl, long Dr,
                     const int32_t* seqlens) {
  if (dtype != ORACLE_F16 && dtype != ORACLE_BF16) return 1;
  if (B < 1 || H < 1 || Hkv < 1 || Skv < 1 || Dl < 1 || Dr < 0) return 1;
  if (H % Hkv != 0) return 1;
  if (seqlens)
    for (long b = 0; b < B; ++b)
      if (seqlens[b] < 0 || seqlens[b] > Skv) return 1;
  return 0;
}

/* Two-pass definition for every (b, h). o_out [B][H][Dl], lse_out [B][H] (may be NULL). */
int oracle_mla_decode(const uint16_t* q, const uint16_t* q_pe, const uint16_t* kv,
                      const uint16_t* k_pe, int dtype, const int32_t* seqlens, long B, long H,
                      long Hkv, long Skv, long Dl, long Dr, double scale, double* o_out,
                      double* lse_out) {
  if (!q || !kv || !o_out || (Dr > 0 && (!q_pe || !k_pe))) return 1;
  if (mla_check(dtype, B, H, Hkv, Skv, Dl, Dr, seqlens)) return 1;
  double* s = (double*)malloc(sizeof(double) * (size_t)Skv);
  if (!s) return 1;
  for (long b = 0; b < B; ++b) {
    const long n = seqlens ? (long)seqlens[b] : Skv;
    for (long h = 0; h < H; ++h) {
      const long g = h / (H / Hkv);
      double* o = o_out + (b * H + h) * Dl;
      for (long d = 0; d < Dl; ++d) o[d] = 0.0;
      if (n == 0) {
        if (lse_out) lse_out[b * H + h] = -INFINITY;
        continue;
      }
      /* s_j = scale * (q . kv_j + q_pe . kpe_j) */
      for (long j = 0; j < n; ++j) {
        double acc = 0.0;
        for (long d = 0; d < Dl; ++d)
          acc += oracle_widen(q[(b * H + h) * Dl + d], dtype) *
                 oracle_widen(kv[((b * Skv + j) * Hkv + g) * Dl + d], dtype);
        for (long e = 0; e < Dr; ++e)
          acc += oracle_widen(q_pe[(b * H + h) * Dr + e], dtype) *
                 oracle_widen(k_pe[((b * Skv + j) * Hkv + g) * Dr + e], dtype);
        s[j] = scale * acc;
      }
      /* softmax, two-pass: m = max s, w_j = exp(s_j - m), l = sum w */
      double m = -INFINITY;
      for (long j = 0; j < n; ++j)
        if (s[j] > m) m = s[j];
      double l = 0.0;
      for (long j = 0; j < n; ++j) {
        const double w = exp(s[j] - m);
        s[j] = w;
        l += w;
      }
      /* o = sum_j w_j kv_j / l   (V = KV; acc_o /= logsum) */
      for (long j = 0; j < n; ++j)
        for (long d = 0; d < Dl; ++d)
          o[d] += s[j] * oracle_widen(kv[((b * Skv + j) * Hkv + g) * Dl + d], dtype);
      for (long d = 0; d < Dl; ++d) o[d] /= l;
      if (lse_out) lse_out[b * H + h] = m + log(l);
    }
  }
  free(s);
  return 0;
}

/* Independent formulation for tiny shapes, one batch b (all heads): concatenate the
 * operands explicitly, Qc = [Q | Q_pe] (H x (Dl+Dr)) and Kc = [KV | K_pe] (n x (Dl+Dr)),
 * S = scale Qc Kc^T materialised, P_hj = 1 / sum_k exp(s_hk - s_hj) (no max subtraction),
 * O = P KV as a matrix product, lse_h = s_hj* - log P_hj* at j* = argmax_j P_hj.
 * s_out/p_out (H x n) may be NULL. o_out H x Dl, lse_out H (may be NULL). */
int oracle_mla_brute(const uint16_t* q, const uint16_t* q_pe, const uint16_t* kv,
                     const uint16_t* k_pe, int dtype, const int32_t* seqlens, long B, long H,
                     long Hkv, long Skv, long Dl, long Dr, double scale, long b, double* s_out,
                     double* p_out, double* o_out, double* lse_out) {
  if (!q || !kv || !o_out || (Dr > 0 && (!q_pe || !k_pe))) return 1;
  if (mla_check(dtype, B, H, Hkv, Skv, Dl, Dr, seqlens) || b < 0 || b >= B) return 1;
  const long n = seqlens ? (long)seqlens[b] : Skv;
  const long Dc = Dl + Dr;
  double* Qc = (double*)malloc(sizeof(double) * (size_t)(H * Dc));
  double* Kc = (double*)malloc(sizeof(double) * (size_t)((Hkv * n + 1) * Dc));
  double* S = (double*)malloc(sizeof(double) * (size_t)(H * n + 1));
  double* P = (double*)malloc(sizeof(double) * (size_t)(H * n + 1));
  if (!Qc || !Kc || !S || !P) {
    free(Qc);
    free(Kc);
    free(S);
    free(P);
    return 1;
  }
  for (long h = 0; h < H; ++h)
    for (long c = 0; c < Dc; ++c)
      Qc[h * Dc + c] = c < Dl ? oracle_widen(q[(b * H + h) * Dl + c], dtype)
                              : oracle_widen(q_pe[(b * H + h) * Dr + (c - Dl)], dtype);
  for (long g = 0; g < Hkv; ++g)
    for (long j = 0; j < n; ++j)
      for (long c = 0; c < Dc; ++c)
        Kc[(g * n + j) * Dc + c] =
            c < Dl ? oracle_widen(kv[((b * Skv + j) * Hkv + g) * Dl + c], dtype)
                   : oracle_widen(k_pe[((b * Skv + j) * Hkv + g) * Dr + (c - Dl)], dtype);
  for (long h = 0; h < H; ++h) {
    const long g = h / (H / Hkv);
    for (long j = 0; j < n; ++j) {
      double acc = 0.0;
      for (long c = 0; c < Dc; ++c) acc += Qc[h * Dc + c] * Kc[(g * n + j) * Dc + c];
      S[h * n + j] = scale * acc;
    }
  }
  for (long h = 0; h < H; ++h) {
    for (long j = 0; j < n; ++j) {
      double den = 0.0;
      for (long k = 0; k < n; ++k) den += exp(S[h * n + k] - S[h * n + j]);
      P[h * n + j] = 1.0 / den;
    }
  }
  for (long h = 0; h < H; ++h) {
    const long g = h / (H / Hkv);
    for (long d = 0; d < Dl; ++d) {
      double acc = 0.0;
      for (long j = 0; j < n; ++j) acc += P[h * n + j] * Kc[(g * n + j) * Dc + d];
      o_out[h * Dl + d] = acc;
    }
    if (lse_out) {
      if (n == 0) {
        lse_out[h] = -INFINITY;
      } else {
        long js = 0;
        for (long j = 1; j < n; ++j)
          if (P[h * n + j] > P[h * n + js]) js = j;
        lse_out[h] = S[h * n + js] - log(P[h * n + js]);
      }
    }
  }
  if (s_out)
    for (long i = 0; i < H * n; ++i) s_out[i] = S[i];
  if (p_out)
    for (long i = 0; i < H * n; ++i) p_out[i] = P[i];
  free(Qc);
  free(Kc);
  free(S);
  free(P);
  return 0;
}
