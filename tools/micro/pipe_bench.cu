// Which pipe does the softmax's fp32->bf16x2 pack (F2FP) use? Loop bodies per pair of
// values: A = 2 x MUFU.EX2; B = A + F2FP.BF16.PACK_AB; C = B + FFMA2 + FADD2 (the full
// softmax element mix). One CTA per SM, 1 or 2 warps per SMSP. Prints pairs/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pk(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ uint64_t f2(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void uf2(uint64_t v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
  constexpr int CH = 16;
  float v[2 * CH]; uint32_t acc = 0; uint64_t s2 = f2(0.f, 0.f);
  const uint64_t c2 = f2(1.0001f, 1.0001f), m2 = f2(-0.5f, -0.5f);
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      float a = v[2 * i], b = v[2 * i + 1];
      a = ex2(a); b = ex2(b);
      if (MODE >= 1) acc ^= pk(a, b);
      if (MODE >= 2) {
        uint64_t x; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x) : "l"(f2(a, b)), "l"(c2), "l"(m2));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(s2) : "l"(x));
        uf2(x, a, b);
      } else { a -= 0.5f; b -= 0.5f; }
      v[2 * i] = a; v[2 * i + 1] = b;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0, s0, s1; uf2(s2, s0, s1);
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc + s0 + s1;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(int sms, float* out, long long* clk) {
  for (int wps : {1, 2}) {
    int threads = 128 * wps, iters = 1000;
    k<MODE><<<sms, threads>>>(out, iters, clk); cudaDeviceSynchronize();
    k<MODE><<<sms, threads>>>(out, iters, clk); long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("mode %d warps/SMSP=%d: %.2f pairs/clk/SM (ex2 %.2f/clk/SM)\n", MODE, wps, (double)threads * iters * 16 / c, 2.0 * threads * iters * 16 / c);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  run<0>(sms, out, clk); run<1>(sms, out, clk); run<2>(sms, out, clk);
  return 0;
}
