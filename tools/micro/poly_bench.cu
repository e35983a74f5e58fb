// Throughput of the kernel's FMA-pipe exp2 (Exp2Poly: clamp, magic-add range reduction,
// degree-3 FFMA2 polynomial, exponent insert) vs MUFU.EX2, per pair of values, and a mix.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_17577_b200/csrc/attn_fwd_sm100.cuh"
using namespace tlattn;
template <int MODE>  // 0: MUFU pairs, 1: poly pairs, 2: 3 of 8 pairs poly
__global__ void k(float* out, int iters, long long* clk) {
  constexpr int CH = 16;
  float v[2 * CH];
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) v[i] = -0.001f * (threadIdx.x + i);
  const Exp2Poly poly;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      float a = v[2 * i], b = v[2 * i + 1];
      const bool emu = MODE == 1 || (MODE == 2 && ((i & 7) == 2 || (i & 7) == 5 || (i & 7) == 7));
      if (emu) poly(f2pack(a, b), a, b);
      else { a = ex2(a); b = ex2(b); }
      v[2 * i] = a - 1.5f; v[2 * i + 1] = b - 1.5f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(int sms, float* out, long long* clk) {
  for (int wps : {1, 2, 4}) {
    int threads = 128 * wps, iters = 1000;
    k<MODE><<<sms, threads>>>(out, iters, clk); cudaDeviceSynchronize();
    k<MODE><<<sms, threads>>>(out, iters, clk); long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("mode %d warps/SMSP=%d: %.2f exp/clk/SM\n", MODE, wps, 2.0 * threads * iters * 16 / c);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  run<0>(sms, out, clk); run<1>(sms, out, clk); run<2>(sms, out, clk);
  return 0;
}
