// gemv_sm100.cuh — the M = 1 rows of tl_gemm: c[N] = a[K] · B[K][N] (the "V" GEMV shapes of
// the paper's Table 2; Matmul Fig. 16 with block_M = 1).
//
// A GEMV reads every element of B exactly once and does 2 FLOP per 2-byte element: it is
// HBM-bound (1 FLOP/B against a ~250 FLOP/B ridge), so there is nothing for the tensor
// cores to do. The design is a bandwidth kernel:
//   * a cluster of CS CTAs owns TC output columns and splits K into CS contiguous ranges;
//     each thread streams 16-byte vectors (8 columns) of its rows of B with read-once
//     (L1::no_allocate) loads, U rows in flight per thread, fp32 FMA into 8 accumulators;
//   * the CTA reduces its row groups in shared memory, then the cluster's leader sums the
//     CS partial rows through distributed shared memory (fixed order: deterministic) and
//     writes c rounded RN — no workspace, one launch.
//   * grid = (N / TC) x CS clusters, sized so at least ~2 CTAs per SM stream at once.
#pragma once
#include "attn_fwd_sm100.cuh"

namespace tlattn {

struct GemvParams {
  const uint16_t* a;  // [K]
  const uint16_t* b;  // [K][N] row-major
  uint16_t* c;        // [N]
  int N, K;
  int tc;             // output columns per cluster (multiple of 8, <= 256)
};

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_CS = 8;      // CTAs per cluster (K split)
#ifndef TLATTN_GEMV_U
#define TLATTN_GEMV_U 8
#endif
constexpr int GEMV_U = TLATTN_GEMV_U;  // 16-byte row vectors in flight per thread (8 or 16)

template <bool BF16>
__device__ __forceinline__ float h2f(uint16_t x) {
  if constexpr (BF16) return __uint_as_float(static_cast<uint32_t>(x) << 16);
  else return __half2float(__ushort_as_half(x));
}

__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Four read-once 16-byte loads in ONE asm statement, so all four are in flight before any
// of their values is used (separate loads were interleaved with the FMAs by the compiler,
// leaving one load in flight per thread).
__device__ __forceinline__ void ld_stream_v4x4(const void* p0, const void* p1, const void* p2,
                                               const void* p3, uint4 (&r)[4]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%16];\n\t"
      "ld.global.nc.L1::no_allocate.v4.u32 {%4, %5, %6, %7}, [%17];\n\t"
      "ld.global.nc.L1::no_allocate.v4.u32 {%8, %9, %10, %11}, [%18];\n\t"
      "ld.global.nc.L1::no_allocate.v4.u32 {%12, %13, %14, %15}, [%19];"
      : "=r"(r[0].x), "=r"(r[0].y), "=r"(r[0].z), "=r"(r[0].w), "=r"(r[1].x), "=r"(r[1].y),
        "=r"(r[1].z), "=r"(r[1].w), "=r"(r[2].x), "=r"(r[2].y), "=r"(r[2].z), "=r"(r[2].w),
        "=r"(r[3].x), "=r"(r[3].y), "=r"(r[3].z), "=r"(r[3].w)
      : "l"(p0), "l"(p1), "l"(p2), "l"(p3));
}

template <bool BF16>
__device__ __forceinline__ void fma8(float (&acc)[8], float s, const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] = fmaf(s, h2f<BF16>(static_cast<uint16_t>(w[i] & 0xFFFFu)), acc[2 * i]);
    acc[2 * i + 1] = fmaf(s, h2f<BF16>(static_cast<uint16_t>(w[i] >> 16)), acc[2 * i + 1]);
  }
}

template <bool BF16>
__global__ void __cluster_dims__(1, GEMV_CS, 1) __launch_bounds__(GEMV_THREADS)
tl_gemv_kernel(const __grid_constant__ GemvParams p) {
  __shared__ float red[GEMV_THREADS * 8];  // [row group][column] partial sums
  const int vpr = p.tc / 8;                 // 16-byte vectors per row of the tile
  const int rpp = GEMV_THREADS / vpr;       // rows per pass (row groups)
  const int tid = threadIdx.x;
  const int cv = tid % vpr;                 // this thread's column vector
  const int rg = tid / vpr;                 // this thread's row group
  const int n0 = blockIdx.x * p.tc + cv * 8;
  const uint32_t rank = cluster_ctarank();  // K split index
  const int kc = (p.K + GEMV_CS - 1) / GEMV_CS;
  const int k_begin = static_cast<int>(rank) * kc;
  const int k_end = min(p.K, k_begin + kc);
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  const bool active = rg < rpp && n0 < p.N;
  if (active) {
    const uint16_t* bcol = p.b + n0;
    int k = k_begin + rg;
    // U independent 16-byte loads in flight, then their FMAs (rows k, k + rpp, ...)
    for (; k + (GEMV_U - 1) * rpp < k_end; k += GEMV_U * rpp) {
      static_assert(GEMV_U % 4 == 0, "groups of four loads");
      uint4 v[GEMV_U / 4][4];
      const uint16_t* r0 = bcol + (size_t)k * p.N;
      const size_t step = (size_t)rpp * p.N;
#pragma unroll
      for (int g4 = 0; g4 < GEMV_U / 4; ++g4) {
        const uint16_t* rg4 = r0 + (size_t)(4 * g4) * step;
        ld_stream_v4x4(rg4, rg4 + step, rg4 + 2 * step, rg4 + 3 * step, v[g4]);
      }
      float s[GEMV_U];
#pragma unroll
      for (int u = 0; u < GEMV_U; ++u) s[u] = h2f<BF16>(p.a[k + u * rpp]);
#pragma unroll
      for (int u = 0; u < GEMV_U; ++u) fma8<BF16>(acc, s[u], v[u >> 2][u & 3]);
    }
    for (; k < k_end; k += rpp) fma8<BF16>(acc, h2f<BF16>(p.a[k]), ld_stream_v4(bcol + (size_t)k * p.N));
  }
  // CTA: sum the row groups of each column (fixed order)
#pragma unroll
  for (int i = 0; i < 8; ++i) red[rg * p.tc + cv * 8 + i] = acc[i];
  __syncthreads();
  for (int col = tid; col < p.tc; col += GEMV_THREADS) {
    float sum = 0.f;
    for (int r = 0; r < rpp; ++r) sum += red[r * p.tc + col];
    red[col] = sum;  // row group 0's slot now holds the CTA's partial for column col
  }
  cluster_sync();  // every CTA's partial row is in its shared memory
  if (rank == 0) {
    const uint32_t base = smem_u32(red);
    for (int col = tid; col < p.tc; col += GEMV_THREADS) {
      float sum = red[col];
      for (int r = 1; r < GEMV_CS; ++r) {
        float x;
        asm volatile("ld.shared::cluster.f32 %0, [%1];"
                     : "=f"(x)
                     : "r"(mapa_shared(base + 4u * col, static_cast<uint32_t>(r))));
        sum += x;
      }
      const int n = blockIdx.x * p.tc + col;
      if (n < p.N) {
        const uint32_t pk = pack2<BF16>(sum, 0.f);
        p.c[n] = static_cast<uint16_t>(pk & 0xFFFFu);
      }
    }
  }
  cluster_sync();  // peers keep their shared memory until the leader has read it
}

}  // namespace tlattn
