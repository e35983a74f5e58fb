// alloc2sm_race.cu — minimal kernels for the compute-sanitizer racecheck report that the
// CTA-pair attention kernel shows once per launch ("potential RAW hazard" between a thread of
// warp 0 and tcgen05.alloc.cta_group::2 of warp 1, profiles/r01_sanitizer.md).
//
// Each kernel is a 2-CTA cluster that only sets up and tears down, in the attention kernel's
// order: warp 0 lane 0 initialises mbarriers in dynamic smem (variant 0) or writes nothing
// (variant 1); warp 1 allocates TMEM (cta_group::2, or cta_group::1 for variant 2) writing
// the address to an smem word; fence, cluster barrier, every thread reads the address;
// dealloc. If racecheck reports the hazard here too — with no data exchanged at all — the
// report belongs to the allocation instruction's own smem write, not to the kernel's logic.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o alloc2sm_race alloc2sm_race.cu
//   compute-sanitizer --tool racecheck ./alloc2sm_race <variant 0|1|2>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int VARIANT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) alloc_kernel(int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (VARIANT != 1 && warp == 0 && lane == 0) {
    for (int i = 0; i < 8; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bars + i)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (VARIANT == 2) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                       smem_u32(tptr))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                       smem_u32(tptr))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = *tptr;
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(taddr);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (VARIANT == 2)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(taddr) : "memory");
  }
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? std::atoi(argv[1]) : 0;
  int* d = nullptr;
  cudaMalloc(&d, 2 * sizeof(int));
  const int smem = 2048;
  if (variant == 0) alloc_kernel<0><<<2, 128, smem>>>(d);
  else if (variant == 1) alloc_kernel<1><<<2, 128, smem>>>(d);
  else alloc_kernel<2><<<2, 128, smem>>>(d);
  const cudaError_t e = cudaDeviceSynchronize();
  int h[2] = {-1, -1};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("variant %d: %s, tmem addresses %d %d\n", variant, cudaGetErrorString(e), h[0], h[1]);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 1;
}
