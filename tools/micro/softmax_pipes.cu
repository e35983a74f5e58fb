// Which pipe bounds the softmax element loop? Variants of the per-element sequence
// x = s*c - m (FFMA2), p = ex2(x) (MUFU), sum += p (FADD2), P = cvt.rn.bf16x2 (F2FP),
// each removing one instruction class. 8 warps x 64 columns per block (one 128x128 tile).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2504_17577_b200/csrc/attn_fwd_sm100.cuh"
using namespace tlattn;

template <int MODE>  // 0 full, 1 no F2FP, 2 no MUFU, 3 no FADD2, 4 no FFMA2, 5 F2FP on f16x2
__global__ void kern(float* out, int iters, long long* clk) {
  constexpr int NC = 64;
  float s[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) s[i] = 0.01f * ((threadIdx.x * 7 + i * 13) % 97) - 0.5f;
  uint32_t keep = 0;
  uint64_t acc[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) acc[a] = f2pack(0.f, 0.f);
  const uint64_t c2 = f2pack(0.1275f, 0.1275f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float mm = 1e-7f * it;
    const uint64_t nm2 = f2pack(-mm, -mm);
    float x[NC];
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      if (MODE == 4) { x[2 * q] = s[2 * q] - mm; x[2 * q + 1] = s[2 * q + 1]; }
      else { uint64_t x2 = ffma2(f2pack(s[2 * q], s[2 * q + 1]), c2, nm2); f2unpack(x2, x[2 * q], x[2 * q + 1]); }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) if (MODE != 2) x[i] = ex2(x[i]);
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      if (MODE != 3) acc[q & 3] = fadd2(acc[q & 3], f2pack(x[2 * q], x[2 * q + 1]));
      if (MODE == 1) keep += __float_as_uint(x[2 * q]) ^ __float_as_uint(x[2 * q + 1]);
      else if (MODE == 5) keep ^= pack2<false>(x[2 * q], x[2 * q + 1]);
      else keep ^= pack2<true>(x[2 * q], x[2 * q + 1]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float a0, a1; f2unpack(acc[0], a0, a1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + (float)keep;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk;
  cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&clk, sms * 8);
  const int iters = 400, warps = 8;
  kern<MODE><<<sms, 32 * warps>>>(out, iters, clk);
  kern<MODE><<<sms, 32 * warps>>>(out, iters, clk);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %7.1f clk/block (64 elem/thread, 8 warps)\n", name, (double)c / iters);
  cudaFree(out); cudaFree(clk);
}

int main() {
  run<0>("full (MUFU only)");
  run<1>("no F2FP");
  run<2>("no MUFU");
  run<3>("no FADD2");
  run<4>("no FFMA2");
  run<5>("F2FP f16x2");
  return 0;
}
