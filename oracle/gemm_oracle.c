/*
 * gemm_oracle.c — plain fp64 GEMM, the definition of the paper's Matmul (Fig. 1 /
 * Fig. 16: C = A · B with A [M][K], B [K][N]):
 *
 *   C[i][j] = sum_{k=0}^{K-1} A[i][k] * B[k][j]      (sequential k, fp64)
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h); shares no code with the CUDA path.
 */
#include "oracle.h"

int oracle_gemm_rows(const uint16_t* a, const uint16_t* b, int dtype, long M, long N, long K,
                     const long* rows, long nrows, double* c_out) {
  if (!a || !b || !c_out || (nrows > 0 && !rows)) return 1;
  if (dtype != ORACLE_F16 && dtype != ORACLE_BF16) return 1;
  if (M < 1 || N < 1 || K < 1 || nrows < 0) return 1;
  for (long r = 0; r < nrows; ++r)
    if (rows[r] < 0 || rows[r] >= M) return 1;
  for (long r = 0; r < nrows; ++r) {
    const long i = rows[r];
    for (long j = 0; j < N; ++j) {
      double acc = 0.0;
      for (long k = 0; k < K; ++k)
        acc += oracle_widen(a[i * K + k], dtype) * oracle_widen(b[k * N + j], dtype);
      c_out[r * N + j] = acc;
    }
  }
  return 0;
}
