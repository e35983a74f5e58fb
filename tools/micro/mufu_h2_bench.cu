// MUFU.EX2 throughput for f16x2 / bf16x2 / f32 operands (does a packed 16-bit exp2 raise the
// softmax exp rate?). One CTA per SM, 16 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
__device__ __forceinline__ unsigned ex2h2(unsigned x) { unsigned y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ unsigned ex2b2(unsigned x) { unsigned y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE, int CH>
__global__ void k(unsigned* out, int iters, long long* clk) {
  unsigned v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = 0x3c00bc00u ^ (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) v[i] = ex2h2(v[i]) ^ 0x80008000u;
      else if (MODE == 1) v[i] = ex2b2(v[i]) ^ 0x80008000u;
      else v[i] = __float_as_uint(ex2f(__uint_as_float(v[i]))) ^ 0x80000000u;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(const char* name, unsigned* out, long long* clk, int sms) {
  const int iters = 2000;
  for (int wps : {1, 2, 4}) {
    int threads = 128 * wps;
    k<MODE, 16><<<sms, threads>>>(out, iters, clk);
    cudaDeviceSynchronize();
    k<MODE, 16><<<sms, threads>>>(out, iters, clk);
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 16;
    printf("%s warps/SMSP=%d: %.2f instr-lanes/clk/SM (x%d exps)\n", name, wps, ops / c, MODE == 2 ? 1 : 2);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  run<0>("f16x2", out, clk, sms); run<1>("bf16x2", out, clk, sms); run<2>("f32", out, clk, sms);
  return 0;
}
