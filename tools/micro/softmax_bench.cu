// Softmax block micro-benchmark: the exact per-block register code of the D=128 pair kernel
// (mask_max_cols + exp_cols from attn_fwd_sm100.cuh) on register data, no TMEM / barriers.
// One CTA per SM with WARPS warps; each thread processes NC columns per "block", ITERS
// blocks. Prints SM clocks per block (the softmax compute floor of one tile-block when
// 128 rows x 128 columns are split over the CTA's threads).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2504_17577_b200/csrc/attn_fwd_sm100.cuh"
using namespace tlattn;

template <int NC, int EMU, int MODE>
__global__ void __launch_bounds__(256, 1) kern(float* out, int iters, long long* clk) {
  float s[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) s[i] = 0.01f * ((threadIdx.x * 7 + i * 13) % 97) - 0.5f;
  float m = 0.f, l = 0.f;
  uint32_t keep = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float sl[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) sl[i] = s[i] + 1e-7f * it;  // fresh "S" every block
    float mx = 0.f;
    if (MODE == 3) mx = mask_max_cols<0, NC>(sl, 0, (threadIdx.x & 127) * NC / 128, true);  // diagonal block
    else if (MODE == 4) mx = mask_max_cols<0, NC>(sl, 0, -1, true);  // fully masked rows
    else if (MODE == 5) mx = mask_max_cols<0, NC>(sl, 0, (threadIdx.x & 127) * NC / 128 - 64, true);
    else if (MODE != 2) mx = mask_max_cols<0, NC>(sl, 0, 1 << 30, false);
    float m_new, alpha, m_use;
    row_max_finish(mx, 1.4426950408889634f * 0.0883883f, m, m_new, alpha, m_use);
    uint64_t acc[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) acc[a] = f2pack(0.f, 0.f);
    uint32_t pk[NC / 2];
    exp_cols<true, 0, NC, EMU>(sl, 1.4426950408889634f * 0.0883883f, m_use, pk, acc);
#pragma unroll
    for (int i = 0; i < NC / 2; ++i) keep ^= pk[i];
    float a0, a1, b0, b1;
    f2unpack(fadd2(acc[0], acc[1]), a0, a1);
    f2unpack(fadd2(acc[2], acc[3]), b0, b1);
    l = l * alpha + (a0 + b0) + (a1 + b1);
    m = m_new;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + m + (float)keep;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int NC, int EMU, int MODE>
void run(const char* name, int warps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk;
  cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&clk, sms * 8);
  const int iters = 400;
  kern<NC, EMU, MODE><<<sms, 32 * warps>>>(out, iters, clk);
  kern<NC, EMU, MODE><<<sms, 32 * warps>>>(out, iters, clk);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  // elements per block per SM = warps*32*NC
  printf("%-28s warps=%2d NC=%3d: %7.1f clk/block  %5.2f exp/clk/SM\n", name, warps, NC,
         (double)c / iters, (double)warps * 32 * NC * iters / c);
  cudaFree(out); cudaFree(clk);
}

int main() {
  run<64, 0, 0>("64col emu0", 8);
  run<128, 0, 3>("128col emu0 masked (2 tiles)", 8);
  run<128, 0, 4>("128col emu0 all -inf (2 tiles)", 8);
  run<128, 0, 5>("128col emu0 masked-64 (2 tiles)", 8);
  run<128, 0, 0>("128col emu0 unmasked (2 tiles)", 8);
  run<64, 1, 0>("64col emu1", 8);
  run<64, 2, 0>("64col emu2", 8);
  run<64, 3, 0>("64col emu3", 8);
  run<64, 2, 2>("64col emu2 nomax", 8);
  run<128, 0, 0>("128col emu0", 4);
  run<128, 2, 0>("128col emu2", 4);
  run<128, 0, 0>("128col emu0 (2 tiles)", 8);
  run<64, 2, 0>("64col emu2 16w (2 tiles)", 16);
  run<64, 0, 0>("64col emu0 16w (2 tiles)", 16);
  run<64, 3, 0>("64col emu3 16w (2 tiles)", 16);
  run<64, 2, 0>("64col emu2 20w", 20);
  run<32, 2, 0>("32col emu2 16w", 16);
  return 0;
}
