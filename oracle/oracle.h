/*
 * oracle.h — fp64 CPU oracle for the fused attention forward.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (libtlattn) never links, loads or calls it, and the two share no code.
 *
 * What it computes (ref [12] "exact attention"; the recurrence of
 * Fig. 18, is an exact reformulation of the same result):
 *
 *   o[b,i,h,:] = sum_{j in J_i} softmax_j(scale * q[b,i,h,:].k[b,j,g,:]) * v[b,j,g,:]
 *   g   = h / (Hq / Hkv)                        (GQA grouping; R7)
 *   J_i = { j < Skv : !causal || j <= i + Skv - Sq }   (bottom-right causal, R3)
 *   lse[b,h,i] = log sum_{j in J_i} exp(scale * q.k_j)  (natural log, R5)
 *   J_i empty -> o = 0, lse = -inf                       (R4)
 *
 * Layout (R6): q[B][Sq][Hq][D], k,v[B][Skv][Hkv][D] as raw 16-bit patterns
 * (dtype 0 = IEEE fp16, 1 = bfloat16), widened exactly to double.
 *
 * Return codes: 0 ok, 1 invalid argument (nothing written).
 */
#ifndef TLATTN_ORACLE_H
#define TLATTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_F16 = 0, ORACLE_BF16 = 1 };

/* Exact widening of one 16-bit pattern to double (IEEE binary16 / bfloat16). */
double oracle_widen(uint16_t bits, int dtype);

/* Plain-definition attention for selected query rows of one (b, h).
 * rows[nrows] are query indices in [0, Sq). o_out is nrows x D (row-major),
 * lse_out is nrows (may be NULL). Two-pass form: max, then exp/sum/normalise. */
int oracle_attn_rows(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                     long B, long Hq, long Hkv, long Sq, long Skv, long D,
                     int causal, double scale, long b, long h,
                     const long* rows, long nrows, double* o_out, double* lse_out);

/* All rows of all (b, h): o_out is BSHD [B][Sq][Hq][D], lse_out is [B][Hq][Sq]. */
int oracle_attn_full(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                     long B, long Hq, long Hkv, long Sq, long Skv, long D,
                     int causal, double scale, double* o_out, double* lse_out);

/* Independent brute-force formulation for tiny shapes (one (b, h)):
 * materialises S (Sq x Skv, -inf where masked), P_ij = 1 / sum_k exp(s_ik - s_ij)
 * (no max subtraction), O = P V as an explicit matrix product.
 * s_out/p_out (Sq x Skv) may be NULL; o_out is Sq x D; lse_out is Sq (may be NULL). */
int oracle_brute_force(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                       long B, long Hq, long Hkv, long Sq, long Skv, long D,
                       int causal, double scale, long b, long h,
                       double* s_out, double* p_out, double* o_out, double* lse_out);

/* Plain GEMM (Fig. 16 Matmul): rows[nrows] of C = A[M][K] B[K][N] in fp64,
 * c_out is nrows x N. */
int oracle_gemm_rows(const uint16_t* a, const uint16_t* b, int dtype, long M, long N, long K,
                     const long* rows, long nrows, double* c_out);

/* MLA decode attention (Appendix B.3, Fig. 18), see mla_oracle.c.
 * q[B][H][Dl], q_pe[B][H][Dr], kv[B][Skv][Hkv][Dl], k_pe[B][Skv][Hkv][Dr] (16-bit patterns),
 * seqlens[B] (int32, each in [0, Skv]) or NULL (= Skv for every batch).
 *   s_j  = scale * (q . kv_j + q_pe . k_pe_j),  j < n_b
 *   o    = sum_j softmax(s)_j kv_j   (V = KV)   o_out [B][H][Dl]
 *   lse  = log sum_j exp(s_j)                                    lse_out [B][H] or NULL
 *   g    = h / (H / Hkv) */
int oracle_mla_decode(const uint16_t* q, const uint16_t* q_pe, const uint16_t* kv,
                      const uint16_t* k_pe, int dtype, const int32_t* seqlens, long B, long H,
                      long Hkv, long Skv, long Dl, long Dr, double scale, double* o_out,
                      double* lse_out);

/* Independent explicit-matrix formulation for batch b (tiny shapes): concatenated
 * operands, S materialised, P_hj = 1/sum_k exp(s_hk - s_hj), O = P KV. s_out/p_out are
 * H x n_b (may be NULL), o_out H x Dl, lse_out H (may be NULL). */
int oracle_mla_brute(const uint16_t* q, const uint16_t* q_pe, const uint16_t* kv,
                     const uint16_t* k_pe, int dtype, const int32_t* seqlens, long B, long H,
                     long Hkv, long Skv, long Dl, long Dr, double scale, long b, double* s_out,
                     double* p_out, double* o_out, double* lse_out);

/* Mamba-2 SSD chunk kernels (Table 4), see ssd_oracle.c for
 * the definitions and readings L1-L8. All arrays double; layouts:
 *   x[B][L][H][P], Bm / C [B][L][G][N], dt / dA [B][H][nchunks][Q], cb [B][nchunks][G][Q][Q],
 *   states / prev [B][nchunks][H][P][N], D[H] (or NULL), out / y [B][L][H][P].
 * nchunks = ceil(L / Q); group of head h: h / (H / G). */
int oracle_ssd_chunk_state(const double* x, const double* Bm, const double* dt, const double* dA,
                           long B, long L, long H, long G, long P, long N, long Q,
                           double* states);
int oracle_ssd_chunk_scan(const double* cb, const double* x, const double* dt, const double* dA,
                          const double* C, const double* prev, const double* D, long B, long L,
                          long H, long G, long P, long N, long Q, double* out);
/* The SSM recurrence position by position (no chunks): dtv[B][L][H], A[H];
 * y_out [B][L][H][P], h_out [B][H][P][N] (final state) or NULL. */
int oracle_ssd_recurrence(const double* x, const double* dtv, const double* A, const double* Bm,
                          const double* C, const double* D, long B, long L, long H, long G,
                          long P, long N, double* y_out, double* h_out);

#ifdef __cplusplus
}
#endif
#endif
