// gen.cu — libtlgen.so: the seeded synthetic-input generator of paper_2504_17577_b200/inputs.py
// as ONE CUDA kernel per tensor (test / bench infrastructure; holds none of the method's
// arithmetic). It reproduces inputs.normal_from_index bit for bit: counter-based lowbias32
// hash of (seed key, global element index), uniforms from the top 24 bits, Box-Muller in fp32
// with the same IEEE operations torch performs (logf, sqrtf, cosf without fast-math), then
// RN conversion to the tensor dtype. A tensor may be a sub-block (slice) of a global tensor
// of up to 6 dimensions: element i of the output has the global index of its coordinates.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace {
constexpr int kMaxDims = 6;
struct GenParams {
  int64_t out_stride[kMaxDims];  // contiguous strides of the output (sub-block)
  int64_t glob_stride[kMaxDims]; // contiguous strides of the global tensor
  int64_t start[kMaxDims];       // sub-block start per dimension
  int ndim;
  int64_t n;                     // elements of the output
  uint32_t key;                  // inputs._key(seed, tensor id), host-computed
  int dtype;                     // 0 fp16, 1 bf16, 2 fp32
  void* out;
};

__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__global__ void tl_gen_normal_kernel(const GenParams p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i, g = 0;
    for (int d = 0; d < p.ndim; ++d) {
      const int64_t c = rem / p.out_stride[d];
      rem -= c * p.out_stride[d];
      g += (c + p.start[d]) * p.glob_stride[d];
    }
    const uint32_t c0 = static_cast<uint32_t>(g * 2);
    const uint32_t c1 = static_cast<uint32_t>(g * 2 + 1);
    const uint32_t hi = static_cast<uint32_t>(g >> 31);
    const uint32_t h0 = lowbias32(lowbias32(c0 ^ p.key) ^ hi);
    const uint32_t h1 = lowbias32(lowbias32(c1 ^ p.key) ^ hi);
    const float u1 = (static_cast<float>(h0 >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = (static_cast<float>(h1 >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float r = sqrtf(-2.0f * logf(u1));
    const float z = r * cosf(6.28318548202514648f * u2);  // fp32(2 pi), as torch's scalar
    if (p.dtype == 0) reinterpret_cast<__half*>(p.out)[i] = __float2half_rn(z);
    else if (p.dtype == 1) reinterpret_cast<__nv_bfloat16*>(p.out)[i] = __float2bfloat16_rn(z);
    else reinterpret_cast<float*>(p.out)[i] = z;
  }
}
}  // namespace

// out: device buffer of prod(out_shape) elements of dtype (0 fp16, 1 bf16, 2 fp32);
// shape / start / out_shape: ndim (<= 6) int64 values (global shape, sub-block start and
// size). Returns 0, 1 (bad argument) or 3 (CUDA error).
extern "C" int tl_gen_normal(void* out, int dtype, int ndim, const int64_t* shape,
                             const int64_t* start, const int64_t* out_shape, uint32_t key,
                             void* stream) {
  if (!out || ndim < 1 || ndim > kMaxDims || dtype < 0 || dtype > 2 || !shape || !start ||
      !out_shape)
    return 1;
  GenParams p{};
  p.ndim = ndim;
  p.key = key;
  p.dtype = dtype;
  p.out = out;
  int64_t so = 1, sg = 1;
  for (int d = ndim - 1; d >= 0; --d) {
    if (out_shape[d] < 0 || start[d] < 0 || start[d] + out_shape[d] > shape[d]) return 1;
    p.out_stride[d] = so;
    p.glob_stride[d] = sg;
    p.start[d] = start[d];
    so *= out_shape[d];
    sg *= shape[d];
  }
  p.n = so;
  if (p.n == 0) return 0;
  const int threads = 256;
  int64_t blocks = (p.n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  tl_gen_normal_kernel<<<static_cast<int>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
