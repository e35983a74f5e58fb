// MUFU.EX2 throughput micro-benchmark (calibration): each thread runs
// N independent ex2.approx chains; one CTA per SM; warps per CTA = 4 x WPS (WPS warps per
// SM sub-partition). Prints ex2 per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int CH>
__global__ void k(float* out, int iters, long long* clk) {
  float v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = ex2(v[i]) - 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 2000;
  for (int wps : {1, 2, 4, 8}) {
    int threads = 128 * wps;
    k<16><<<sms, threads>>>(out, iters, clk);
    cudaDeviceSynchronize();
    k<16><<<sms, threads>>>(out, iters, clk);
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 16;
    printf("warps/SMSP=%d: %.2f ex2/clk/SM (%lld clk)\n", wps, ops / c, c);
  }
  return 0;
}
