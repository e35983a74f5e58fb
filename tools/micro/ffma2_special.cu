// Is fp32x2 FMA (FFMA2) or F2FP slow on infinite operands? 8 warps x 32 independent FFMA2
// chains per thread; clocks per iteration for finite vs -inf inputs.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2pack(float a, float b) { unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) { unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int MODE>
__global__ void k(float v0, float* out, int iters, long long* clk) {
  unsigned long long x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = f2pack(v0 + i, v0 - i);
  const unsigned long long c = f2pack(0.5f, 0.5f), m = f2pack(-1e-3f, -1e-3f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = ffma2(x[i], c, m);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 32; ++i) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(x[i])); s += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&clk, 148 * 8);
  float vals[] = {1.0f, -INFINITY, 1e-40f};
  const char* names[] = {"finite", "-inf", "denormal"};
  for (int v = 0; v < 3; ++v) {
    k<0><<<148, 256>>>(vals[v], out, 200, clk); k<0><<<148, 256>>>(vals[v], out, 200, clk);
    cudaDeviceSynchronize(); long long t; cudaMemcpy(&t, clk, 8, cudaMemcpyDeviceToHost);
    printf("FFMA2 %-9s %8.1f clk/iter (8 warps x 32 FFMA2)\n", names[v], t / 200.0);
  }
  return 0;
}
