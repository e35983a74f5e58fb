/*
 * ssd_oracle.c — plain, slow, obviously-correct fp64 Mamba-2 SSD chunk kernels (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: nothing in the product path links or calls this file.
 * It shares no code, header, table or constant with paper_2504_17577_b200/csrc.
 *
 * What it follows: PAPER.md §5.2 "Linear Attention Performance": "the chunk-scan
 * and chunk-state functions from Mamba-2", benchmarked on the shapes of Table 4
 * (batch, nheads, seq_len, head_dim, d_state). The paper prints no formula;
 * the functions are the two chunked kernels of the Mamba-2 state-space-duality (SSD)
 * algorithm for the scalar-decay SSM (readings L1-L8):
 *
 *   recurrence (per batch b, head h, group g = h / (H/G)):
 *     h_t = exp(dt_t * A_h) h_{t-1} + dt_t * B_t x_t^T          (h_t in R^{N x P})
 *     y_t = C_t^T h_t + D_h x_t
 *   chunked (chunk length Q, chunk c = positions [cQ, cQ + len_c), len_c = min(Q, L - cQ)):
 *     dA[b,h,c,i] = sum_{j <= i} dt_{cQ+j} A_h   (inclusive cumulative sum inside the chunk)
 *     chunk_state: states[b,c,h,p,n] = sum_{i < len_c} x[b,cQ+i,h,p] B[b,cQ+i,g,n]
 *                                        * exp(dA[b,h,c,len_c-1] - dA[b,h,c,i]) * dt[b,h,c,i]
 *     chunk_scan:  out[b,cQ+i,h,p] = exp(dA[b,h,c,i]) * sum_n C[b,cQ+i,g,n] prev[b,c,h,p,n]
 *                     + sum_{j <= i} cb[b,c,g,i,j] exp(dA[b,h,c,i] - dA[b,h,c,j]) dt[b,h,c,j]
 *                                    * x[b,cQ+j,h,p]
 *                     + D_h x[b,cQ+i,h,p]
 *     with cb[b,c,g,i,j] = sum_n C[b,cQ+i,g,n] B[b,cQ+j,g,n] and prev[b,c] the state entering
 *     chunk c (prev[b,0] = 0, prev[b,c+1] = exp(dA[b,h,c,len_c-1]) prev[b,c] + states[b,c]).
 *
 * Layouts: x[B][L][H][P], Bm / C [B][L][G][N], dt / dA [B][H][nchunks][Q] (entries i >=
 * len_c of the last chunk are ignored), cb [B][nchunks][G][Q][Q], states / prev
 * [B][nchunks][H][P][N], D[H] (or NULL = 0), out / y [B][L][H][P]. All double.
 * Build: gcc -O2 (no -ffast-math), single-threaded, libm only. Return 0 ok, 1 bad argument.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>

static int ssd_check(long Bn, long L, long H, long G, long P, long N, long Q) {
  if (Bn < 1 || L < 1 || H < 1 || G < 1 || P < 1 || N < 1 || Q < 1) return 1;
  if (H % G != 0) return 1;
  return 0;
}

static long chunk_len(long c, long L, long Q) { return (L - c * Q) < Q ? (L - c * Q) : Q; }

int oracle_ssd_chunk_state(const double* x, const double* Bm, const double* dt, const double* dA,
                           long Bn, long L, long H, long G, long P, long N, long Q,
                           double* states) {
  if (!x || !Bm || !dt || !dA || !states || ssd_check(Bn, L, H, G, P, N, Q)) return 1;
  const long nc = (L + Q - 1) / Q;
  for (long b = 0; b < Bn; ++b)
    for (long c = 0; c < nc; ++c) {
      const long len = chunk_len(c, L, Q);
      for (long h = 0; h < H; ++h) {
        const long g = h / (H / G);
        const double* dtc = dt + ((b * H + h) * nc + c) * Q;
        const double* dAc = dA + ((b * H + h) * nc + c) * Q;
        for (long p = 0; p < P; ++p)
          for (long n = 0; n < N; ++n) {
            double acc = 0.0;
            for (long i = 0; i < len; ++i) {
              const long t = c * Q + i;
              acc += x[((b * L + t) * H + h) * P + p] * Bm[((b * L + t) * G + g) * N + n] *
                     exp(dAc[len - 1] - dAc[i]) * dtc[i];
            }
            states[(((b * nc + c) * H + h) * P + p) * N + n] = acc;
          }
      }
    }
  return 0;
}

int oracle_ssd_chunk_scan(const double* cb, const double* x, const double* dt, const double* dA,
                          const double* C, const double* prev, const double* D, long Bn, long L,
                          long H, long G, long P, long N, long Q, double* out) {
  if (!cb || !x || !dt || !dA || !C || !prev || !out || ssd_check(Bn, L, H, G, P, N, Q)) return 1;
  const long nc = (L + Q - 1) / Q;
  for (long b = 0; b < Bn; ++b)
    for (long c = 0; c < nc; ++c) {
      const long len = chunk_len(c, L, Q);
      for (long h = 0; h < H; ++h) {
        const long g = h / (H / G);
        const double* dtc = dt + ((b * H + h) * nc + c) * Q;
        const double* dAc = dA + ((b * H + h) * nc + c) * Q;
        const double* cbc = cb + ((b * nc + c) * G + g) * Q * Q;
        const double* pv = prev + ((b * nc + c) * H + h) * P * N;
        for (long i = 0; i < len; ++i) {
          const long t = c * Q + i;
          for (long p = 0; p < P; ++p) {
            double inter = 0.0;  /* state entering the chunk, decayed to position i */
            for (long n = 0; n < N; ++n) inter += C[((b * L + t) * G + g) * N + n] * pv[p * N + n];
            inter *= exp(dAc[i]);
            double intra = 0.0;  /* positions j <= i of this chunk */
            for (long j = 0; j <= i; ++j)
              intra += cbc[i * Q + j] * exp(dAc[i] - dAc[j]) * dtc[j] *
                       x[((b * L + c * Q + j) * H + h) * P + p];
            const double skip = D ? D[h] * x[((b * L + t) * H + h) * P + p] : 0.0;
            out[((b * L + t) * H + h) * P + p] = inter + intra + skip;
          }
        }
      }
    }
  return 0;
}

/* The SSM recurrence itself, position by position (an independent formulation: no
 * chunks, no cumulative sums). dtv[B][L][H] (per position), A[H], Bm / C [B][L][G][N],
 * x [B][L][H][P], D[H] or NULL. y_out [B][L][H][P]; h_out [B][H][P][N] = final state
 * (may be NULL). Work space: one N x P state per (b, h). */
int oracle_ssd_recurrence(const double* x, const double* dtv, const double* A, const double* Bm,
                          const double* C, const double* D, long Bn, long L, long H, long G,
                          long P, long N, double* y_out, double* h_out) {
  if (!x || !dtv || !A || !Bm || !C || !y_out || ssd_check(Bn, L, H, G, P, N, 1)) return 1;
  double* hs = (double*)calloc((size_t)(N * P), sizeof(double));
  if (!hs) return 1;
  for (long b = 0; b < Bn; ++b)
    for (long h = 0; h < H; ++h) {
      const long g = h / (H / G);
      for (long e = 0; e < N * P; ++e) hs[e] = 0.0;
      for (long t = 0; t < L; ++t) {
        const double d = dtv[(b * L + t) * H + h];
        const double decay = exp(d * A[h]);
        for (long n = 0; n < N; ++n)
          for (long p = 0; p < P; ++p)
            hs[n * P + p] = decay * hs[n * P + p] +
                            d * Bm[((b * L + t) * G + g) * N + n] * x[((b * L + t) * H + h) * P + p];
        for (long p = 0; p < P; ++p) {
          double acc = 0.0;
          for (long n = 0; n < N; ++n) acc += C[((b * L + t) * G + g) * N + n] * hs[n * P + p];
          y_out[((b * L + t) * H + h) * P + p] =
              acc + (D ? D[h] * x[((b * L + t) * H + h) * P + p] : 0.0);
        }
      }
      if (h_out)
        for (long p = 0; p < P; ++p)
          for (long n = 0; n < N; ++n) h_out[((b * H + h) * P + p) * N + n] = hs[n * P + p];
    }
  free(hs);
  return 0;
}
