// mbar_handoff_race.cu — does compute-sanitizer racecheck model an mbarrier hand-off of
// ordinary shared-memory data between warps?
//
// The SSD chunk_scan kernel passes the per-unit decay vectors from one warp (st.shared) to
// others (ld.shared) through a double-buffered pair of mbarriers (full: writer lane 0
// arrives after __syncwarp; empty: every reader warp's lane 0 arrives after __syncwarp),
// the pattern CUTLASS pipelines use. racecheck reports it as a RAW/WAR hazard. This kernel is
// that hand-off alone, repeated over "units" with two buffers:
//   variant 0: mbarrier hand-off (full / empty barriers, as the kernel)
//   variant 1: the same data flow ordered by __syncthreads() instead
// If variant 0 reports hazards and variant 1 does not, the report is about the sanitizer's
// model of mbarrier ordering, not a missing synchronisation.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mbar_handoff_race mbar_handoff_race.cu
//   compute-sanitizer --tool racecheck ./mbar_handoff_race <0|1>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

constexpr int UNITS = 16, NV = 256, READERS = 4;

template <int VARIANT>
__global__ void __launch_bounds__(32 * (1 + READERS), 1) handoff_kernel(float* out) {
  __shared__ __align__(16) float vec[2][NV];
  __shared__ __align__(8) uint64_t bars[4];  // full[2], empty[2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[2]);
  if (threadIdx.x == 0) {
    mbar_init(full0, 1);
    mbar_init(full0 + 8, 1);
    mbar_init(empty0, READERS);
    mbar_init(empty0 + 8, READERS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  for (int u = 0; u < UNITS; ++u) {
    const int vb = u & 1;
    if (VARIANT == 0) {
      if (warp == 0) {
        if (u >= 2) mbar_wait(empty0 + 8 * vb, ((u >> 1) - 1) & 1);
        for (int i = lane; i < NV; i += 32) vec[vb][i] = float(u * NV + i);
        __syncwarp();
        if (lane == 0) mbar_arrive(full0 + 8 * vb);
      } else {
        mbar_wait(full0 + 8 * vb, (u >> 1) & 1);
        for (int i = lane; i < NV; i += 32) acc += vec[vb][i];
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * vb);
      }
    } else {
      if (warp == 0)
        for (int i = lane; i < NV; i += 32) vec[vb][i] = float(u * NV + i);
      __syncthreads();
      if (warp != 0)
        for (int i = lane; i < NV; i += 32) acc += vec[vb][i];
      __syncthreads();
    }
  }
  out[threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? std::atoi(argv[1]) : 0;
  float* d = nullptr;
  cudaMalloc(&d, 32 * (1 + READERS) * sizeof(float));
  if (variant == 0) handoff_kernel<0><<<1, 32 * (1 + READERS)>>>(d);
  else handoff_kernel<1><<<1, 32 * (1 + READERS)>>>(d);
  const cudaError_t e = cudaDeviceSynchronize();
  float h[64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  // reader lane l sums u*NV + i over u < UNITS, i = l mod 32 (8 values per unit)
  double want = 0.0;
  for (int u = 0; u < UNITS; ++u)
    for (int i = 0; i < NV; i += 32) want += double(u * NV + i);
  std::printf("variant %d: %s, reader lane 0 sum %.0f (expected %.0f)\n", variant,
              cudaGetErrorString(e), h[32], want);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 1;
}
