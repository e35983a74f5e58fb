// Does MUFU.EX2 (ex2.approx.ftz.f32) run slower on special inputs (-inf, large negative)?
// 8 warps x 64 independent ex2 per iteration, one CTA per SM; clocks per iteration.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void k(float base, int frac_inf, float* out, int iters, long long* clk) {
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = (i < frac_inf) ? -INFINITY : base - 0.01f * ((threadIdx.x + i) & 15);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 64; ++i) acc += ex2(v[i] - 1e-9f * it);
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&clk, 148 * 8);
  struct { const char* n; float base; int finf; } cases[] = {
      {"normal (-3)", -3.f, 0}, {"all -inf", -3.f, 64}, {"half -inf", -3.f, 32},
      {"large negative (-200)", -200.f, 0}, {"-130 (denormal range)", -130.f, 0}};
  for (auto& c : cases) {
    k<<<148, 256>>>(c.base, c.finf, out, 200, clk);
    k<<<148, 256>>>(c.base, c.finf, out, 200, clk);
    cudaDeviceSynchronize();
    long long t; cudaMemcpy(&t, clk, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %8.1f clk/iter (8 warps x 64 ex2) = %.2f ex2/clk/SM\n", c.n, t / 200.0, 256.0 * 64 * 200 / t);
  }
  return 0;
}
