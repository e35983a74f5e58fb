// tlattn_api.cu — host side of libtlattn: the C ABI declared in include/tlattn.h.
//
// Argument validation happens before any CUDA call (TL_ERR_* returned synchronously,
// nothing launched). Tensor maps are encoded per call (cheap host work, no device
// allocation) and passed to the kernel as __grid_constant__ parameters, so the call is
// CUDA-graph capturable. cuTensorMapEncodeTiled is resolved through the runtime's
// driver entry point (no -lcuda link).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>

#include "../../include/tlattn.h"
#include "attn_fwd_sm100.cuh"
#include "attn_fwd_sm100_2sm.cuh"
#include "gemm_sm100_2sm.cuh"
#include "gemv_sm100.cuh"
#include "mla_decode_sm100.cuh"
#include "ssd_sm100.cuh"

using namespace tlattn;

namespace {

thread_local int g_last_launches = 0;
unsigned long long* g_trace = nullptr;  // debug builds only (tl_attn_debug_trace)

// A/B experiment options (include/tlattn.h tl_attn_set_option): process-wide atomics, set
// once from the environment on first use (TLATTN_KERNEL=1cta, TLATTN_UNIT_TILES, TLATTN_LPT,
// TLATTN_GEMV_TC, TLATTN_MLA_HC, TLATTN_MLA_CL — for the tools/ A/B scripts) and changed only
// through tl_attn_set_option, so production calls do no getenv. -1 = automatic.
std::atomic<int> g_opt[TL_OPT_COUNT];
std::once_flag g_opt_once;
void init_options() {
  std::call_once(g_opt_once, [] {
    auto env = [](const char* name) {
      const char* e = std::getenv(name);
      return e ? std::atoi(e) : -1;
    };
    const char* k = std::getenv("TLATTN_KERNEL");
    g_opt[TL_OPT_FORCE_1CTA] = (k && std::strcmp(k, "1cta") == 0) ? 1 : -1;
    g_opt[TL_OPT_UNIT_TILES] = env("TLATTN_UNIT_TILES");
    g_opt[TL_OPT_LPT] = env("TLATTN_LPT");
    g_opt[TL_OPT_GEMV_TC] = env("TLATTN_GEMV_TC");
    g_opt[TL_OPT_MLA_HC] = env("TLATTN_MLA_HC");
    g_opt[TL_OPT_MLA_CL] = env("TLATTN_MLA_CL");
  });
}
int opt(int o) {
  init_options();
  return g_opt[o].load(std::memory_order_relaxed);
}


struct DeviceInfo {
  int sm_count = 0;
  int major = 0, minor = 0;
  bool ok = false;
  // per kernel instantiation: cudaFuncAttributeMaxDynamicSharedMemorySize already set.
  // Slots: attention 0-7, replicated-output attention 8-15, GEMM 16-17, SSD 18-21.
  bool smem_set[32] = {};
};

constexpr int kMaxDevices = 64;
std::mutex g_mu;
DeviceInfo g_dev[kMaxDevices];
bool g_dev_init[kMaxDevices] = {};
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return g_encode;
}

// Returns TL_OK and fills *dev, or an error code.
int current_device(int* dev_out, DeviceInfo** info_out) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceInfo& di = g_dev[dev];
  if (!g_dev_init[dev]) {
    if (cudaDeviceGetAttribute(&di.sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
      cudaGetLastError();
      return TL_ERR_CUDA;
    }
    di.ok = (di.major == 10 && di.minor == 0);  // sm_100a code runs on sm_100 only
    g_dev_init[dev] = true;
  }
  *dev_out = dev;
  *info_out = &di;
  return di.ok ? TL_OK : TL_ERR_UNSUPPORTED;
}

int validate(const void* q, const void* k, const void* v, const void* o, const float* lse, int B,
             int Hq, int Hkv, int Sq, int Skv, int D, int causal, float scale, int dtype) {
  if (!q || !k || !v || !o) return TL_ERR_INVALID_VALUE;
  if (B < 1 || Hq < 1 || Hkv < 1 || Sq < 1 || Skv < 1 || D < 1) return TL_ERR_INVALID_VALUE;
  if (causal != 0 && causal != 1) return TL_ERR_INVALID_VALUE;
  if (!std::isfinite(scale)) return TL_ERR_INVALID_VALUE;
  if (dtype != TL_DTYPE_F16 && dtype != TL_DTYPE_BF16) return TL_ERR_INVALID_VALUE;
  if (D != 64 && D != 128) return TL_ERR_UNSUPPORTED;
  if (Hq % Hkv != 0) return TL_ERR_UNSUPPORTED;
  auto al = [](const void* ptr, uintptr_t a) { return (reinterpret_cast<uintptr_t>(ptr) % a) == 0; };
  if (!al(q, 16) || !al(k, 16) || !al(v, 16) || !al(o, 16)) return TL_ERR_UNSUPPORTED;
  if (lse && !al(lse, 4)) return TL_ERR_UNSUPPORTED;
  // grid.x = B * Hq * ceil(Sq/256) must fit in int32; TMA coordinates are int32
  const long long units = (long long)B * Hq * ((Sq + 255) / 256);       // single-CTA grid
  const long long pair_grid = 2LL * B * Hq * ((Sq + 511) / 512);          // CTA-pair grid
  if (units > 0x7fffffffLL || pair_grid > 0x7fffffffLL) return TL_ERR_UNSUPPORTED;
  return TL_OK;
}

// Per-thread cache of encoded tensor maps (host-side only: a CUtensorMap is a 128-byte
// descriptor of (address, dims, strides, box); re-encoding costs host time on every call).
// Keyed by everything that goes into the descriptor.
struct TmapKey {
  const void* ptr;
  int dtype;
  cuuint64_t dims[4];
  cuuint32_t box[4];
  bool operator==(const TmapKey& o) const {
    return ptr == o.ptr && dtype == o.dtype && std::memcmp(dims, o.dims, sizeof dims) == 0 &&
           std::memcmp(box, o.box, sizeof box) == 0;
  }
};
struct TmapCache {
  static constexpr int N = 32;
  TmapKey key[N];
  CUtensorMap map[N];
  bool used[N] = {};
  int next = 0;
};
thread_local TmapCache g_tmaps;

// Rank-4 map over a contiguous 16-bit tensor, dims innermost first, SWIZZLE_128B box.
bool encode_4d_cached(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, const void* ptr,
                      int dtype, const cuuint64_t (&dims)[4], const cuuint32_t (&box)[4]) {
  TmapKey k;
  std::memset(&k, 0, sizeof k);
  k.ptr = ptr;
  k.dtype = dtype;
  std::memcpy(k.dims, dims, sizeof k.dims);
  std::memcpy(k.box, box, sizeof k.box);
  TmapCache& c = g_tmaps;
  for (int i = 0; i < TmapCache::N; ++i)
    if (c.used[i] && c.key[i] == k) {
      *m = c.map[i];
      return true;
    }
  const cuuint64_t strides[3] = {dims[0] * 2, dims[0] * dims[1] * 2, dims[0] * dims[1] * dims[2] * 2};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, dtype == TL_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   4, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  const int i = c.next;
  c.next = (c.next + 1) % TmapCache::N;
  c.key[i] = k;
  c.map[i] = *m;
  c.used[i] = true;
  return true;
}

bool encode_bshd(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, const void* ptr, int dtype,
                 int Bn, int S, int H, int D, unsigned box_rows = 128) {
  return encode_4d_cached(enc, m, ptr, dtype,
                          {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)S, (cuuint64_t)Bn},
                          {64, 1, box_rows, 1});
}

// Kernel launch with programmatic dependent launch allowed (the kernels call
// griddep_wait() before touching global memory): back-to-back calls overlap the next
// kernel's launch and prologue with this one's tail. -DTLATTN_NO_PDL: plain launches.
template <class K, class PT>
cudaError_t launch_pdl(K kern, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       const PT& prm) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
#ifndef TLATTN_NO_PDL
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelEx(&cfg, kern, prm);
}

template <bool BF16, class PT>
int launch_2sm(const PT& prm, DeviceInfo& di, int inst, cudaStream_t stream) {
  auto kern = tl_attn_fwd_kernel_2sm<BF16, PT>;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di.smem_set[inst]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               KCfg2::SMEM_BYTES) != cudaSuccess) {
        cudaGetLastError();
        return TL_ERR_CUDA;
      }
      di.smem_set[inst] = true;
    }
  }
  if (launch_pdl(kern, 2 * prm.n_units, NUM_THREADS, KCfg2::SMEM_BYTES, stream, prm) != cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  return TL_OK;
}

// Kernel selection: D=128 runs on CTA pairs (2-SM tcgen05), D=64 on single CTAs.
// TL_OPT_FORCE_1CTA = 1 forces the single-CTA kernel for D=128 (A/B comparisons only).
bool use_2sm(int D) { return D == 128 && opt(TL_OPT_FORCE_1CTA) != 1; }

template <int D, bool BF16, class PT>
int launch(const PT& prm, DeviceInfo& di, int inst, cudaStream_t stream) {
  auto kern = tl_attn_fwd_kernel<D, BF16, PT>;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di.smem_set[inst]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               KCfg<D>::SMEM_BYTES) != cudaSuccess) {
        cudaGetLastError();
        return TL_ERR_CUDA;
      }
      di.smem_set[inst] = true;
    }
  }
  if (launch_pdl(kern, prm.n_units, NUM_THREADS, KCfg<D>::SMEM_BYTES, stream, prm) != cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  return TL_OK;
}

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;  // ceil(log2 d)
  f.shr = l;
  f.mul = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  return f;
}

// Shared by tl_attn_fwd and tl_attn_fwd_replicated: input tensor maps, sizes, unit
// geometry; then the launch of the kernel instantiated for the parameter type PT.
template <class PT>
int run_attn(PT& prm, const void* q, const void* k, const void* v, int B, int Hq, int Hkv,
             int Sq, int Skv, int D, int causal, float scale, int dtype, void* stream) {
  int dev;
  DeviceInfo* di;
  int rc;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;

  const bool pair = use_2sm(D);
  if (!encode_bshd(enc, &prm.tm_q, q, dtype, B, Sq, Hq, D) ||
      !encode_bshd(enc, &prm.tm_k, k, dtype, B, Skv, Hkv, D, pair ? 64u : 128u) ||
      !encode_bshd(enc, &prm.tm_v, v, dtype, B, Skv, Hkv, D))
    return TL_ERR_CUDA;
  prm.B = B;
  prm.Hq = Hq;
  prm.Hkv = Hkv;
  prm.Sq = Sq;
  prm.Skv = Skv;
  prm.causal = causal;
  prm.c_log2 = std::fabs(scale) * 1.4426950408889634f;
  // scale = 0 (uniform attention): use a tiny positive c instead, so masked scores
  // (-inf) still map to exp2(-inf) = 0 in the kernel's single exp path; with |s| << 1e28
  // every allowed p is exactly 1 and LSE = ln|J| up to ~1e-28.
  if (prm.c_log2 == 0.f) prm.c_log2 = 1e-30f;
  // Short-sequence mode (the paper's "dynamic parameters", and its small-S point,
  // P:L362): when the 512-row pair units would fill at most half of the SM pairs, units
  // shrink to one 256-row tile so twice as many pairs work (Table 3 FA0/FA1 shapes).
  prm.unit_tiles = 2;
  if (pair) {
    const long long units512 = (long long)B * Hq * ((Sq + 511) / 512);
    if (2 * units512 <= di->sm_count / 2) prm.unit_tiles = 1;
    if (const int v = opt(TL_OPT_UNIT_TILES); v == 1 || v == 2) prm.unit_tiles = v;
  }
  const int unit_rows = pair ? 2 * BM * prm.unit_tiles : TILES * BM;
  prm.n_mblk = (Sq + unit_rows - 1) / unit_rows;
  // Unit order (the T.use_swizzle idea). Default: units of one (b, kv head) are
  // adjacent so their K/V stay L2-resident. Causal problems instead run the heaviest query
  // blocks of ALL heads first (longest-processing-time order) when either their whole K/V
  // fits in half of the 126 MB L2 (the paper's Table 3 shapes), or the heaviest unit is
  // >= 5 % of one worker's share of the work (long sequences: the last head's first unit
  // would otherwise start late and run alone). Measured: Table 3 FA4 +26 %,
  // C4 +12.6 %, C3 +1.4 %; C5 (short sequences, 2 GB of K/V) -5 %, so it keeps head-major.
  const double kv_bytes = 4.0 * B * Hkv * (double)Skv * D;
  const int workers = pair ? di->sm_count / 2 : di->sm_count;
  const double nb = std::ceil(Skv / 128.0);                    // K/V blocks of a full row
  const double tile_rows = pair ? 256.0 : 128.0;
  const double tiles_per_unit = pair ? prm.unit_tiles : TILES;
  const double heaviest = tiles_per_unit * nb;                 // tile-blocks of the top unit
  const double share = (double)B * Hq * std::ceil(Sq / tile_rows) * nb * 0.5 / workers;
  prm.lpt = (causal && (kv_bytes <= 64.0 * (1 << 20) || heaviest >= 0.05 * share)) ? 1 : 0;
  if (const int v = opt(TL_OPT_LPT); v == 0 || v == 1) prm.lpt = v;
  // grid bound re-checked after the unit-size choice (validate() bounded the default)
  const long long n_units = (long long)B * Hq * prm.n_mblk;
  if ((pair ? 2 : 1) * n_units > 0x7fffffffLL) return TL_ERR_UNSUPPORTED;
  prm.n_units = static_cast<int>(n_units);
  prm.fd_mblk = make_fastdiv(prm.n_mblk);
  prm.fd_nbh = make_fastdiv(B * Hq);
  prm.fd_hq = make_fastdiv(Hq);
  prm.fd_grp = make_fastdiv(Hq / Hkv);
  // Negative scale: the tensor core negates Q (instruction-descriptor a_negate), so the
  // kernel computes S' = -QK^T and uses c = |scale| log2(e) >= 0; scale*S == |scale|*S'.
  prm.neg = scale < 0.f ? 1 : 0;
  prm.trace = g_trace;

  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool bf = dtype == TL_DTYPE_BF16;
  const int i0 = PT::kRepl ? 8 : 0;  // per-instantiation "smem attribute set" slots
  if (pair) rc = bf ? launch_2sm<true>(prm, *di, i0 + 4, st) : launch_2sm<false>(prm, *di, i0 + 5, st);
  else if (D == 128) rc = bf ? launch<128, true>(prm, *di, i0 + 0, st) : launch<128, false>(prm, *di, i0 + 1, st);
  else rc = bf ? launch<64, true>(prm, *di, i0 + 2, st) : launch<64, false>(prm, *di, i0 + 3, st);
  if (rc == TL_OK) g_last_launches = 1;
  return rc;
}

}  // namespace

extern "C" int tl_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int B,
                           int Hq, int Hkv, int Sq, int Skv, int D, int causal, float scale,
                           int dtype, void* stream) {
  g_last_launches = 0;
  int rc = validate(q, k, v, o, lse, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype);
  if (rc != TL_OK) return rc;
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;
  AttnParams prm;
  std::memset(&prm, 0, sizeof(prm));
  if (!encode_bshd(enc, &prm.tm_o, o, dtype, B, Sq, Hq, D)) return TL_ERR_CUDA;
  prm.o = o;
  prm.lse = lse;
  return run_attn(prm, q, k, v, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype, stream);
}

extern "C" int tl_attn_fwd_replicated(const void* q, const void* k, const void* v,
                                      void* const* o_outs, float* const* lse_outs, int n_outs,
                                      int B_total, int b_off, int Hq_total, int h_off, int B,
                                      int Hq, int Hkv, int Sq, int Skv, int D, int causal,
                                      float scale, int dtype, void* stream) {
  g_last_launches = 0;
  if (!o_outs || n_outs < 1 || n_outs > kMaxOuts) return TL_ERR_INVALID_VALUE;
  for (int r = 0; r < n_outs; ++r)
    if (!o_outs[r]) return TL_ERR_INVALID_VALUE;
  int rc = validate(q, k, v, o_outs[0], nullptr, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype);
  if (rc != TL_OK) return rc;
  if (b_off < 0 || h_off < 0 || B_total < 1 || Hq_total < 1 || (long long)b_off + B > B_total ||
      (long long)h_off + Hq > Hq_total)
    return TL_ERR_INVALID_VALUE;
  for (int r = 0; r < n_outs; ++r) {
    if (reinterpret_cast<uintptr_t>(o_outs[r]) % 16 != 0) return TL_ERR_UNSUPPORTED;
    if (lse_outs && lse_outs[r] && reinterpret_cast<uintptr_t>(lse_outs[r]) % 4 != 0)
      return TL_ERR_UNSUPPORTED;
  }
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;
  AttnParamsRepl prm;
  std::memset(&prm, 0, sizeof(prm));
  for (int r = 0; r < n_outs; ++r) {
    if (!encode_bshd(enc, &prm.tm_out[r], o_outs[r], dtype, B_total, Sq, Hq_total, D))
      return TL_ERR_CUDA;
    prm.o_out[r] = o_outs[r];
    prm.lse_out[r] = lse_outs ? lse_outs[r] : nullptr;
  }
  prm.n_out = n_outs;
  prm.b_off = b_off;
  prm.h_off = h_off;
  prm.Hq_total = Hq_total;
  return run_attn(prm, q, k, v, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype, stream);
}

// ------------------------------------------------------------------ peer memory (N2)
namespace {
struct PeerFlags {
  uint32_t* ptr[kMaxOuts];
};
thread_local uint64_t g_peer_timeout_ns = 10000000000ull;  // 10 s
// One block, `world` threads: thread i publishes `epoch` into rank i's flag slot [rank]
// (system-scope release: this rank's earlier writes into rank i's memory — the replicated
// O / LSE of the previous kernels on this stream — are visible before the flag), then
// waits until its own slot [i] holds >= epoch (acquire: rank i's writes are visible). The
// wait is bounded: after timeout_ns the thread records TL_ERR_TIMEOUT in this rank's
// status word and returns (a dead peer must not hang the stream forever).
__global__ void tl_peer_barrier_kernel_v(const PeerFlags f, int world, int rank, uint32_t epoch,
                                         uint64_t timeout_ns) {
  const int i = threadIdx.x;
  if (i >= world) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.ptr[i] + rank), "r"(epoch) : "memory");
  const uint32_t* mine = f.ptr[rank] + i;
  const uint64_t t0 = globaltimer();
  uint32_t v;
  for (uint32_t n = 0;; ++n) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    if ((n & 255u) == 255u && globaltimer() - t0 > timeout_ns) {
      atomicExch(f.ptr[rank] + TL_PEER_STATUS_WORD, (uint32_t)TL_ERR_TIMEOUT);
      break;
    }
  }
}
}  // namespace

extern "C" int tl_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch,
                               void* stream) {
  g_last_launches = 0;
  if (!flags || world < 1 || world > kMaxOuts || rank < 0 || rank >= world)
    return TL_ERR_INVALID_VALUE;
  PeerFlags f;
  std::memset(&f, 0, sizeof f);
  for (int r = 0; r < world; ++r) {
    if (!flags[r] || reinterpret_cast<uintptr_t>(flags[r]) % 4 != 0) return TL_ERR_INVALID_VALUE;
    f.ptr[r] = flags[r];
  }
  int dev;
  DeviceInfo* di;
  int rc;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  tl_peer_barrier_kernel_v<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      f, world, rank, epoch, g_peer_timeout_ns);
  if (cudaGetLastError() != cudaSuccess) return TL_ERR_CUDA;
  g_last_launches = 1;
  return TL_OK;
}

extern "C" int tl_peer_barrier_set_timeout_ns(uint64_t ns) {
  if (ns == 0) return TL_ERR_INVALID_VALUE;
  g_peer_timeout_ns = ns;
  return TL_OK;
}

extern "C" int tl_peer_barrier_check(const uint32_t* own_flags) {
  if (!own_flags || reinterpret_cast<uintptr_t>(own_flags) % 4 != 0) return TL_ERR_INVALID_VALUE;
  uint32_t status = 0;
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(&status, own_flags + TL_PEER_STATUS_WORD, sizeof status, cudaMemcpyDeviceToHost) !=
          cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  return status == 0 ? TL_OK : (int)status;
}

// Handle blob = cudaIpcMemHandle_t of the allocation + the byte offset of dev_ptr inside it
// (torch's caching allocator sub-allocates, and cudaIpcOpenMemHandle maps the allocation
// base), so the opened pointer is the same tensor in the other process.
struct IpcBlob {
  cudaIpcMemHandle_t h;
  uint64_t offset;
};

extern "C" int tl_ipc_handle_bytes(void) { return (int)sizeof(IpcBlob); }

extern "C" int tl_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return TL_ERR_INVALID_VALUE;
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!get_range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000, cudaEnableDefault,
                                           &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return TL_ERR_CUDA;
      get_range = reinterpret_cast<GetRange>(fn);
    }
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return TL_ERR_CUDA;
  IpcBlob blob;
  std::memset(&blob, 0, sizeof blob);
  if (cudaIpcGetMemHandle(&blob.h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  blob.offset = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
  std::memcpy(handle_out, &blob, sizeof blob);
  return TL_OK;
}

extern "C" int tl_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return TL_ERR_INVALID_VALUE;
  IpcBlob blob;
  std::memcpy(&blob, handle, sizeof blob);
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, blob.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  *dev_ptr_out = static_cast<uint8_t*>(base) + blob.offset;
  return TL_OK;
}

// dev_ptr: the pointer tl_ipc_open_handle returned (offset into the mapped allocation)
extern "C" int tl_ipc_close_handle(void* dev_ptr) {
  if (!dev_ptr) return TL_ERR_INVALID_VALUE;
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000, cudaEnableDefault, &q) !=
          cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return TL_ERR_CUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (reinterpret_cast<GetRange>(fn)(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return TL_ERR_CUDA;
  if (cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  return TL_OK;
}

// ------------------------------------------------------------------ host-buffer entry
namespace {
struct HostPlan {
  int cb;             // batches per chunk
  size_t q_b, kv_b, o_b, lse_b;  // bytes per batch element
  size_t slot_bytes;  // one chunk slot (q, k, v, o, lse), 256-B aligned pieces
};

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

HostPlan plan_host(int B, int Hq, int Hkv, int Sq, int Skv, int D, int with_lse) {
  HostPlan pl;
  pl.cb = B <= 2 ? B : (B + 7) / 8;  // ~8 chunks so copies overlap compute
  pl.q_b = (size_t)Sq * Hq * D * 2;
  pl.kv_b = (size_t)Skv * Hkv * D * 2;
  pl.o_b = pl.q_b;
  pl.lse_b = with_lse ? (size_t)Hq * Sq * 4 : 0;
  pl.slot_bytes = al256(pl.cb * pl.q_b) + 2 * al256(pl.cb * pl.kv_b) + al256(pl.cb * pl.o_b) +
                  al256(pl.cb * pl.lse_b);
  return pl;
}

std::mutex g_stream_mu;
cudaStream_t g_copy_streams[kMaxDevices][2] = {};
}  // namespace

extern "C" uint64_t tl_attn_host_workspace_bytes(int B, int Hq, int Hkv, int Sq, int Skv, int D,
                                                 int with_lse) {
  if (B < 1 || Hq < 1 || Hkv < 1 || Sq < 1 || Skv < 1 || D < 1) return 0;
  HostPlan pl = plan_host(B, Hq, Hkv, Sq, Skv, D, with_lse);
  return 2 * (uint64_t)pl.slot_bytes;
}

extern "C" int tl_attn_fwd_host(const void* q_h, const void* k_h, const void* v_h, void* o_h,
                                float* lse_h, int B, int Hq, int Hkv, int Sq, int Skv, int D,
                                int causal, float scale, int dtype, void* ws, uint64_t ws_bytes,
                                void* stream) {
  g_last_launches = 0;
  int rc = validate(q_h, k_h, v_h, o_h, lse_h, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype);
  if (rc != TL_OK) return rc;
  if (!ws) return TL_ERR_INVALID_VALUE;
  HostPlan pl = plan_host(B, Hq, Hkv, Sq, Skv, D, lse_h != nullptr);
  if (ws_bytes < 2 * (uint64_t)pl.slot_bytes) return TL_ERR_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return TL_ERR_UNSUPPORTED;
  int dev;
  DeviceInfo* di;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t h2d, d2h;
  {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    for (int i = 0; i < 2; ++i)
      if (!g_copy_streams[dev][i] &&
          cudaStreamCreateWithFlags(&g_copy_streams[dev][i], cudaStreamNonBlocking) != cudaSuccess)
        return TL_ERR_CUDA;
    h2d = g_copy_streams[dev][0];
    d2h = g_copy_streams[dev][1];
  }
  const int nchunks = (B + pl.cb - 1) / pl.cb;
  // events: [0] start, [1..2] in, [3..4] comp, [5..6] out, [7..8] tails of the copy streams.
  // Every created event is destroyed on every exit path.
  cudaEvent_t evs[9] = {};
  int n_ev = 0;
  auto destroy_events = [&] {
    for (int i = 0; i < n_ev; ++i) cudaEventDestroy(evs[i]);
  };
  for (; n_ev < 9; ++n_ev) {
    if (cudaEventCreateWithFlags(&evs[n_ev], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      destroy_events();
      return TL_ERR_CUDA;
    }
  }
  cudaEvent_t ev_start = evs[0], ev_in[2] = {evs[1], evs[2]}, ev_comp[2] = {evs[3], evs[4]},
              ev_out[2] = {evs[5], evs[6]};
  bool ok = cudaEventRecord(ev_start, cs) == cudaSuccess;
  ok = ok && cudaStreamWaitEvent(h2d, ev_start, 0) == cudaSuccess;
  int launches = 0;
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  for (int c = 0; c < nchunks && ok; ++c) {
    const int s = c & 1;
    const int b0 = c * pl.cb;
    const int nb = (B - b0) < pl.cb ? (B - b0) : pl.cb;
    uint8_t* slot = wsb + (size_t)s * pl.slot_bytes;
    uint8_t* dq = slot;
    uint8_t* dk = dq + al256(pl.cb * pl.q_b);
    uint8_t* dv = dk + al256(pl.cb * pl.kv_b);
    uint8_t* dout = dv + al256(pl.cb * pl.kv_b);
    float* dlse = lse_h ? reinterpret_cast<float*>(dout + al256(pl.cb * pl.o_b)) : nullptr;
    if (c >= 2) ok = ok && cudaStreamWaitEvent(h2d, ev_out[s], 0) == cudaSuccess;  // slot free
    ok = ok && cudaMemcpyAsync(dq, (const uint8_t*)q_h + (size_t)b0 * pl.q_b, nb * pl.q_b, cudaMemcpyHostToDevice, h2d) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(dk, (const uint8_t*)k_h + (size_t)b0 * pl.kv_b, nb * pl.kv_b, cudaMemcpyHostToDevice, h2d) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(dv, (const uint8_t*)v_h + (size_t)b0 * pl.kv_b, nb * pl.kv_b, cudaMemcpyHostToDevice, h2d) == cudaSuccess;
    ok = ok && cudaEventRecord(ev_in[s], h2d) == cudaSuccess;
    ok = ok && cudaStreamWaitEvent(cs, ev_in[s], 0) == cudaSuccess;
    if (!ok) break;
    rc = tl_attn_fwd(dq, dk, dv, dout, dlse, nb, Hq, Hkv, Sq, Skv, D, causal, scale, dtype, cs);
    if (rc != TL_OK) break;
    ++launches;
    ok = ok && cudaEventRecord(ev_comp[s], cs) == cudaSuccess;
    ok = ok && cudaStreamWaitEvent(d2h, ev_comp[s], 0) == cudaSuccess;
    ok = ok && cudaMemcpyAsync((uint8_t*)o_h + (size_t)b0 * pl.o_b, dout, nb * pl.o_b, cudaMemcpyDeviceToHost, d2h) == cudaSuccess;
    if (lse_h)
      ok = ok && cudaMemcpyAsync((uint8_t*)lse_h + (size_t)b0 * pl.lse_b, dlse, nb * pl.lse_b, cudaMemcpyDeviceToHost, d2h) == cudaSuccess;
    ok = ok && cudaEventRecord(ev_out[s], d2h) == cudaSuccess;
  }
  // The caller's stream resumes after EVERY copy queued on the two copy streams — on the
  // error paths too, so the caller may free or reuse ws and the host buffers once its
  // stream is done.
  const bool tails = cudaEventRecord(evs[7], h2d) == cudaSuccess &&
                     cudaEventRecord(evs[8], d2h) == cudaSuccess &&
                     cudaStreamWaitEvent(cs, evs[7], 0) == cudaSuccess &&
                     cudaStreamWaitEvent(cs, evs[8], 0) == cudaSuccess;
  ok = ok && tails;
  destroy_events();
  if (rc != TL_OK) return rc;
  if (!ok) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  g_last_launches = launches;
  return TL_OK;
}

// ------------------------------------------------------------------ GEMM
namespace {
bool encode_2d(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, const void* ptr, int dtype,
               int inner, int outer, unsigned box_inner, unsigned box_outer) {
  // rank-4 map with two unit dimensions so the kernel shares the 4-D TMA instructions
  return encode_4d_cached(enc, m, ptr, dtype, {(cuuint64_t)inner, (cuuint64_t)outer, 1, 1},
                          {box_inner, box_outer, 1, 1});
}

template <bool BF16>
int launch_gemm(const GemmParams& prm, DeviceInfo& di, int inst, cudaStream_t stream) {
  auto kern = tl_gemm_kernel_2sm<BF16>;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di.smem_set[inst]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GCfg::SMEM_BYTES) !=
          cudaSuccess) {
        cudaGetLastError();
        return TL_ERR_CUDA;
      }
      di.smem_set[inst] = true;
    }
  }
  kern<<<2 * prm.tiles_m * prm.tiles_n, GCfg::THREADS, GCfg::SMEM_BYTES, stream>>>(prm);
  if (cudaGetLastError() != cudaSuccess) return TL_ERR_CUDA;
  return TL_OK;
}
}  // namespace

extern "C" int tl_gemm(const void* a, const void* b, void* c, int M, int N, int K, int dtype,
                       void* stream) {
  g_last_launches = 0;
  if (!a || !b || !c) return TL_ERR_INVALID_VALUE;
  if (M < 1 || N < 1 || K < 1) return TL_ERR_INVALID_VALUE;
  if (dtype != TL_DTYPE_F16 && dtype != TL_DTYPE_BF16) return TL_ERR_INVALID_VALUE;
  if (N % 8 != 0 || K % 8 != 0) return TL_ERR_UNSUPPORTED;
  auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0; };
  if (!al(a) || !al(b) || !al(c)) return TL_ERR_UNSUPPORTED;
  const long long tiles = (long long)((M + 255) / 256) * ((N + 255) / 256);
  if (2 * tiles > 0x7fffffffLL) return TL_ERR_UNSUPPORTED;
  int dev, rc;
  DeviceInfo* di;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  if (M == 1) {
    // GEMV (Table 2 "V" shapes): HBM-bound, no tensor cores (gemv_sm100.cuh). Column
    // tiles of 256 (128 for N >= 32768; narrower only when fewer than 18 tiles = 144 CTAs),
    // the best of 32/64/128/256 measured on the V shapes.
    GemvParams gp;
    gp.a = static_cast<const uint16_t*>(a);
    gp.b = static_cast<const uint16_t*>(b);
    gp.c = static_cast<uint16_t*>(c);
    gp.N = N;
    gp.K = K;
    int tc = N >= 32768 ? 128 : 256;  // measured: 128 is 4-5 % faster for N >= 32768
    while (tc > 32 && (N + tc - 1) / tc < 18) tc /= 2;
    if (const int v = opt(TL_OPT_GEMV_TC); v == 32 || v == 64 || v == 128 || v == 256) tc = v;
    gp.tc = tc;
    const long long tiles = (N + tc - 1) / tc;
    if (tiles > 0x7fffffffLL) return TL_ERR_UNSUPPORTED;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const dim3 grid(static_cast<unsigned>(tiles), GEMV_CS, 1);
    if (dtype == TL_DTYPE_BF16) tl_gemv_kernel<true><<<grid, GEMV_THREADS, 0, st>>>(gp);
    else tl_gemv_kernel<false><<<grid, GEMV_THREADS, 0, st>>>(gp);
    if (cudaGetLastError() != cudaSuccess) return TL_ERR_CUDA;
    g_last_launches = 1;
    return TL_OK;
  }
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;
  GemmParams prm;
  std::memset(&prm, 0, sizeof(prm));
  if (!encode_2d(enc, &prm.tm_a, a, dtype, K, M, 64, 128) ||
      !encode_2d(enc, &prm.tm_b, b, dtype, N, K, 64, 64) ||
      !encode_2d(enc, &prm.tm_c, c, dtype, N, M, 64, 128))
    return TL_ERR_CUDA;
  prm.M = M;
  prm.N = N;
  prm.K = K;
  prm.tiles_m = (M + 255) / 256;
  prm.tiles_n = (N + 255) / 256;
  prm.group_n = 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  rc = dtype == TL_DTYPE_BF16 ? launch_gemm<true>(prm, *di, 16, st) : launch_gemm<false>(prm, *di, 17, st);
  if (rc == TL_OK) g_last_launches = 1;
  return rc;
}

// ------------------------------------------------------------------ MLA decode
namespace {
struct MlaPlan {
  int HC, T, NHG, P, CL;
  size_t off_lse, off_o, bytes;
};

int mla_cluster_size(int T) {
  if (const int v = opt(TL_OPT_MLA_CL); (v == 1 || v == 2 || v == 4) && T % v == 0) return v;
  // measured on B200: multicast clusters ran slower than independent CTAs
  // (lockstep ring, no L2 relief at cluster size <= 4), so the default is 1
  (void)T;
  return 1;
}

// Clusters of `cl` MLA CTAs that fit on the device at once (cached per device and size).
int mla_max_clusters(int dev, int cl, int sm_count);

MlaPlan plan_mla(int B, int H, int Hkv, int dev, int sm_count) {
  MlaPlan pl;
  const int g = H / Hkv;
  // 64-head tiles read the latent cache half as often as 32-head tiles
  pl.HC = g >= 64 ? 64 : 32;
  if (const int v = opt(TL_OPT_MLA_HC); v == 32 || v == 64) pl.HC = v;
  pl.T = (g + pl.HC - 1) / pl.HC;
  pl.NHG = Hkv * pl.T;
  pl.CL = mla_cluster_size(pl.T);
  // all CTAs co-resident (one per SM): clusters that fit / cluster groups = partitions
  const int groups = pl.NHG / pl.CL;
  pl.P = mla_max_clusters(dev, pl.CL, sm_count) / groups;
  if (pl.P < 1) pl.P = 1;
  pl.off_lse = al256((size_t)(B + 1) * 4);
  pl.off_o = pl.off_lse + al256((size_t)pl.NHG * pl.P * 2 * pl.HC * 4);
  pl.bytes = pl.off_o + (size_t)pl.NHG * pl.P * 2 * pl.HC * mla::DL * 4;
  return pl;
}

bool encode_4d(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, const void* ptr, int dtype,
               const cuuint64_t (&dims)[4], const cuuint32_t (&box)[4]) {
  return encode_4d_cached(enc, m, ptr, dtype, dims, box);
}

std::mutex g_mla_mu;
int g_mla_clusters[kMaxDevices][5] = {};

template <int HC, bool BF16>
bool mla_attr_one() {
  auto k = mla::tl_mla_decode_kernel<HC, BF16>;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              mla::Cfg<HC>::SMEM_BYTES) == cudaSuccess &&
         cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
}

bool mla_smem_attr(int dev) {
  static bool done[kMaxDevices] = {};
  if (done[dev]) return true;
  if (!mla_attr_one<32, true>() || !mla_attr_one<32, false>() || !mla_attr_one<64, true>() ||
      !mla_attr_one<64, false>()) {
    cudaGetLastError();
    return false;
  }
  done[dev] = true;
  return true;
}

int mla_max_clusters(int dev, int cl, int sm_count) {
  std::lock_guard<std::mutex> lk(g_mla_mu);
  if (g_mla_clusters[dev][cl] > 0) return g_mla_clusters[dev][cl];
  int n = sm_count / cl;
  if (mla_smem_attr(dev)) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * (sm_count / cl), 1, 1);
    cfg.blockDim = dim3(mla::Cfg<64>::THREADS, 1, 1);
    cfg.dynamicSmemBytes = mla::Cfg<64>::SMEM_BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, mla::tl_mla_decode_kernel<64, true>, &cfg) == cudaSuccess &&
        c > 0)
      n = c;
    cudaGetLastError();
  }
  g_mla_clusters[dev][cl] = n;
  return n;
}

template <int HC, bool BF16>
int launch_mla(const mla::MlaParams& prm, int dev, int B, const int* seqlens, int Skv,
               cudaStream_t stream) {
  {
    std::lock_guard<std::mutex> lk(g_mla_mu);
    if (!mla_smem_attr(dev)) return TL_ERR_CUDA;
  }
  mla::tl_mla_meta_kernel<<<1, 1024, 0, stream>>>(seqlens, B, Skv, prm.cum);
  if (cudaGetLastError() != cudaSuccess) return TL_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(prm.Hkv * prm.T * prm.P, 1, 1);
  cfg.blockDim = dim3(mla::Cfg<HC>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = mla::Cfg<HC>::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = prm.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, mla::tl_mla_decode_kernel<HC, BF16>, prm) != cudaSuccess) {
    cudaGetLastError();
    return TL_ERR_CUDA;
  }
  mla::tl_mla_combine_kernel<BF16><<<dim3(B, prm.Hkv * prm.T), 256, 0, stream>>>(prm);
  if (cudaGetLastError() != cudaSuccess) return TL_ERR_CUDA;
  return TL_OK;
}
}  // namespace

extern "C" uint64_t tl_mla_decode_workspace_bytes(int B, int H, int Hkv) {
  if (B < 1 || H < 1 || Hkv < 1 || H % Hkv != 0) return 0;
  int dev;
  DeviceInfo* di;
  if (current_device(&dev, &di) != TL_OK) return 0;
  return plan_mla(B, H, Hkv, dev, di->sm_count).bytes;
}

extern "C" int tl_mla_decode(const void* q, const void* q_pe, const void* kv, const void* k_pe,
                             void* o, float* lse, const int* seqlens, int B, int H, int Hkv,
                             int Skv, int Dl, int Dr, float scale, int dtype, void* ws,
                             uint64_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (!q || !q_pe || !kv || !k_pe || !o || !ws) return TL_ERR_INVALID_VALUE;
  if (B < 1 || H < 1 || Hkv < 1 || Skv < 1 || Dl < 1 || Dr < 1) return TL_ERR_INVALID_VALUE;
  if (!std::isfinite(scale)) return TL_ERR_INVALID_VALUE;
  if (dtype != TL_DTYPE_F16 && dtype != TL_DTYPE_BF16) return TL_ERR_INVALID_VALUE;
  if (Dl != mla::DL || Dr != mla::DR || H % Hkv != 0) return TL_ERR_UNSUPPORTED;
  auto al = [](const void* ptr, uintptr_t a) { return (reinterpret_cast<uintptr_t>(ptr) % a) == 0; };
  if (!al(q, 16) || !al(q_pe, 16) || !al(kv, 16) || !al(k_pe, 16) || !al(o, 16) || !al(ws, 256))
    return TL_ERR_UNSUPPORTED;
  if ((lse && !al(lse, 4)) || (seqlens && !al(seqlens, 4))) return TL_ERR_UNSUPPORTED;
  if ((long long)B * H > 0x7fffffffLL || (long long)B * Skv * Hkv > 0x7fffffffLL)
    return TL_ERR_UNSUPPORTED;
  int dev, rc;
  DeviceInfo* di;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  const MlaPlan pl = plan_mla(B, H, Hkv, dev, di->sm_count);
  if (ws_bytes < pl.bytes) return TL_ERR_INVALID_VALUE;
  if ((long long)pl.NHG * pl.P > 0x7fffffffLL || B > 65535 || pl.NHG > 65535) return TL_ERR_UNSUPPORTED;
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;
  mla::MlaParams prm;
  std::memset(&prm, 0, sizeof(prm));
  const cuuint64_t HH = (cuuint64_t)H, BB = (cuuint64_t)B, SS = (cuuint64_t)Skv, GG = (cuuint64_t)Hkv;
  if (!encode_4d(enc, &prm.tm_q, q, dtype, {(cuuint64_t)mla::DL, HH, 1, BB}, {64, (cuuint32_t)pl.HC, 1, 1}) ||
      !encode_4d(enc, &prm.tm_qpe, q_pe, dtype, {(cuuint64_t)mla::DR, HH, 1, BB}, {64, (cuuint32_t)pl.HC, 1, 1}) ||
      !encode_4d(enc, &prm.tm_k, kv, dtype, {(cuuint64_t)mla::DL, GG, SS, BB}, {64, 1, mla::BLK, 1}) ||
      !encode_4d(enc, &prm.tm_kpe, k_pe, dtype, {(cuuint64_t)mla::DR, GG, SS, BB}, {64, 1, mla::BLK, 1}))
    return TL_ERR_CUDA;
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  prm.o = o;
  prm.lse = lse;
  prm.seqlens = seqlens;
  prm.cum = reinterpret_cast<int*>(wsb);
  prm.ws_lse = reinterpret_cast<float*>(wsb + pl.off_lse);
  prm.ws_o = reinterpret_cast<float*>(wsb + pl.off_o);
  prm.B = B;
  prm.H = H;
  prm.Hkv = Hkv;
  prm.Skv = Skv;
  prm.g = H / Hkv;
  prm.T = pl.T;
  prm.P = pl.P;
  prm.CL = pl.CL;
  prm.HC = pl.HC;
  prm.c_log2 = std::fabs(scale) * 1.4426950408889634f;
  if (prm.c_log2 == 0.f) prm.c_log2 = 1e-30f;  // scale = 0: see tl_attn_fwd
  prm.neg = scale < 0.f ? 1 : 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool bf = dtype == TL_DTYPE_BF16;
  if (pl.HC == 64)
    rc = bf ? launch_mla<64, true>(prm, dev, B, seqlens, Skv, st) : launch_mla<64, false>(prm, dev, B, seqlens, Skv, st);
  else
    rc = bf ? launch_mla<32, true>(prm, dev, B, seqlens, Skv, st) : launch_mla<32, false>(prm, dev, B, seqlens, Skv, st);
  if (rc == TL_OK) g_last_launches = 3;
  return rc;
}

// ------------------------------------------------------------------ SSD chunk kernels (N4)
namespace {
int ssd_validate(int batch, int seqlen, int nheads, int ngroups, int headdim, int dstate,
                 int chunk_size, int dtype) {
  if (batch < 1 || seqlen < 1 || nheads < 1 || ngroups < 1 || headdim < 1 || dstate < 1 ||
      chunk_size < 1)
    return TL_ERR_INVALID_VALUE;
  if (nheads % ngroups != 0) return TL_ERR_INVALID_VALUE;
  if (dtype != TL_DTYPE_F16 && dtype != TL_DTYPE_BF16) return TL_ERR_INVALID_VALUE;
  if (headdim != ssd::P || dstate != ssd::N || chunk_size != ssd::Q) return TL_ERR_UNSUPPORTED;
  const long long nc = (seqlen + (long long)chunk_size - 1) / chunk_size;
  if ((long long)batch * nc > 0x7fffffffLL || (long long)batch * nc * nheads > 0x7fffffffLL)
    return TL_ERR_UNSUPPORTED;
  return TL_OK;
}
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool al4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3) == 0; }

template <class K>
int ssd_launch(K kern, int smem, int threads, const ssd::SsdParams& prm, DeviceInfo& di, int inst,
               cudaStream_t stream) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di.smem_set[inst]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
          cudaSuccess) {
        cudaGetLastError();
        return TL_ERR_CUDA;
      }
      di.smem_set[inst] = true;
    }
  }
  // persistent CTAs striding over units; an odd grid makes each CTA alternate the unit
  // kinds of chunk_scan (units 2i / 2i+1 are the light / heavy row tile of one (b, c, h))
  int grid = prm.n_units < di.sm_count ? prm.n_units : di.sm_count;
  if (grid > 1 && grid % 2 == 0 && grid < prm.n_units) --grid;
  kern<<<grid, threads, smem, stream>>>(prm);
  if (cudaGetLastError() != cudaSuccess) return TL_ERR_CUDA;
  return TL_OK;
}
}  // namespace

extern "C" int tl_ssd_chunk_state(const void* x, const void* Bm, const float* dt, const float* dA,
                                  void* states, int batch, int seqlen, int nheads, int ngroups,
                                  int headdim, int dstate, int chunk_size, int dtype,
                                  void* stream) {
  g_last_launches = 0;
  if (!x || !Bm || !dt || !dA || !states) return TL_ERR_INVALID_VALUE;
  int rc = ssd_validate(batch, seqlen, nheads, ngroups, headdim, dstate, chunk_size, dtype);
  if (rc != TL_OK) return rc;
  // head pairs share a CTA and its Bm tile: both heads of a pair must be in one group
  if (nheads % 2 != 0 || (nheads / ngroups) % 2 != 0) return TL_ERR_UNSUPPORTED;
  if (!al16(x) || !al16(Bm) || !al16(states) || !al4(dt) || !al4(dA)) return TL_ERR_UNSUPPORTED;
  int dev;
  DeviceInfo* di;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;
  ssd::SsdParams prm;
  std::memset(&prm, 0, sizeof prm);
  const cuuint64_t L = seqlen, Bn = batch;
  if (!encode_4d_cached(enc, &prm.tm_x, x, dtype, {(cuuint64_t)ssd::P, (cuuint64_t)nheads, L, Bn},
                        {64, 1, 64, 1}) ||
      !encode_4d_cached(enc, &prm.tm_b, Bm, dtype, {(cuuint64_t)ssd::N, (cuuint64_t)ngroups, L, Bn},
                        {64, 1, 64, 1}))
    return TL_ERR_CUDA;
  prm.dt = dt;
  prm.dA = dA;
  prm.out = states;
  prm.B = batch;
  prm.L = seqlen;
  prm.H = nheads;
  prm.G = ngroups;
  prm.nc = (seqlen + chunk_size - 1) / chunk_size;
  prm.grp = nheads / ngroups;
  prm.trace = g_trace;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // four heads per unit (one Bm tile for four heads) when they share a group
  using S2 = ssd::StateCfg<2>;
  using S4 = ssd::StateCfg<4>;
  if ((nheads / ngroups) % 4 == 0) {
    prm.n_units = batch * prm.nc * (nheads / 4);
    rc = dtype == TL_DTYPE_BF16
             ? ssd_launch(ssd::tl_ssd_state_kernel<true, 4>, S4::SMEM_BYTES, S4::THREADS, prm, *di, 22, st)
             : ssd_launch(ssd::tl_ssd_state_kernel<false, 4>, S4::SMEM_BYTES, S4::THREADS, prm, *di, 23, st);
  } else {
    prm.n_units = batch * prm.nc * (nheads / 2);
    rc = dtype == TL_DTYPE_BF16
             ? ssd_launch(ssd::tl_ssd_state_kernel<true, 2>, S2::SMEM_BYTES, S2::THREADS, prm, *di, 18, st)
             : ssd_launch(ssd::tl_ssd_state_kernel<false, 2>, S2::SMEM_BYTES, S2::THREADS, prm, *di, 19, st);
  }
  if (rc == TL_OK) g_last_launches = 1;
  return rc;
}

extern "C" int tl_ssd_chunk_scan(const void* cb, const void* x, const float* dt, const float* dA,
                                 const void* C, const void* prev_states, const float* D, void* out,
                                 int batch, int seqlen, int nheads, int ngroups, int headdim,
                                 int dstate, int chunk_size, int dtype, void* stream) {
  g_last_launches = 0;
  if (!cb || !x || !dt || !dA || !C || !prev_states || !out) return TL_ERR_INVALID_VALUE;
  int rc = ssd_validate(batch, seqlen, nheads, ngroups, headdim, dstate, chunk_size, dtype);
  if (rc != TL_OK) return rc;
  if (!al16(cb) || !al16(x) || !al16(C) || !al16(prev_states) || !al16(out) || !al4(dt) ||
      !al4(dA) || (D && !al4(D)))
    return TL_ERR_UNSUPPORTED;
  int dev;
  DeviceInfo* di;
  if ((rc = current_device(&dev, &di)) != TL_OK) return rc;
  auto enc = get_encode();
  if (!enc) return TL_ERR_CUDA;
  ssd::SsdParams prm;
  std::memset(&prm, 0, sizeof prm);
  const int nc = (seqlen + chunk_size - 1) / chunk_size;
  const cuuint64_t L = seqlen, Bn = batch, BNC = (cuuint64_t)batch * nc;
  if (!encode_4d_cached(enc, &prm.tm_x, x, dtype, {(cuuint64_t)ssd::P, (cuuint64_t)nheads, L, Bn},
                        {64, 1, 128, 1}) ||
      !encode_4d_cached(enc, &prm.tm_c, C, dtype, {(cuuint64_t)ssd::N, (cuuint64_t)ngroups, L, Bn},
                        {64, 1, 128, 1}) ||
      !encode_4d_cached(enc, &prm.tm_cb, cb, dtype,
                        {(cuuint64_t)ssd::Q, (cuuint64_t)ssd::Q, (cuuint64_t)ngroups, BNC},
                        {64, 128, 1, 1}) ||
      !encode_4d_cached(enc, &prm.tm_s, prev_states, dtype,
                        {(cuuint64_t)ssd::N, (cuuint64_t)ssd::P, (cuuint64_t)nheads, BNC},
                        {64, 64, 1, 1}))
    return TL_ERR_CUDA;
  prm.dt = dt;
  prm.dA = dA;
  prm.D = D;
  prm.x = x;
  prm.out = out;
  prm.B = batch;
  prm.L = seqlen;
  prm.H = nheads;
  prm.G = ngroups;
  prm.nc = nc;
  prm.grp = nheads / ngroups;
  prm.n_units = batch * nc * nheads * 2;  // (b, c, h, 128-row tile)
  prm.trace = g_trace;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  rc = dtype == TL_DTYPE_BF16
           ? ssd_launch(ssd::tl_ssd_scan_kernel<true>, ssd::ScanCfg::SMEM_BYTES, ssd::ScanCfg::THREADS, prm, *di, 20, st)
           : ssd_launch(ssd::tl_ssd_scan_kernel<false>, ssd::ScanCfg::SMEM_BYTES, ssd::ScanCfg::THREADS, prm, *di, 21, st);
  if (rc == TL_OK) g_last_launches = 1;
  return rc;
}

extern "C" const char* tl_attn_strerror(int status) {
  switch (status) {
    case TL_OK: return "TL_OK: success";
    case TL_ERR_INVALID_VALUE: return "TL_ERR_INVALID_VALUE: invalid argument (null pointer, size < 1, causal not 0/1, non-finite scale, unknown dtype, or workspace too small)";
    case TL_ERR_UNSUPPORTED: return "TL_ERR_UNSUPPORTED: unsupported configuration (D not 64/128, Hq % Hkv != 0, misaligned pointer, size limit, or device is not sm_100)";
    case TL_ERR_CUDA: return "TL_ERR_CUDA: a CUDA runtime/driver call failed";
    case TL_ERR_TIMEOUT: return "TL_ERR_TIMEOUT: a peer did not reach the device barrier before its timeout";
    default: return "unknown tl_status code";
  }
}

extern "C" int tl_attn_version(void) { return TLATTN_VERSION; }

extern "C" int tl_attn_set_option(int option, int value) {
  if (option < 0 || option >= TL_OPT_COUNT) return TL_ERR_INVALID_VALUE;
  init_options();
  g_opt[option].store(value < 0 ? -1 : value, std::memory_order_relaxed);
  return TL_OK;
}

extern "C" int tl_attn_get_option(int option) {
  if (option < 0 || option >= TL_OPT_COUNT) return -2;
  return opt(option);
}

// Debug hook (not part of include/tlattn.h): device buffer of >= 8000 u64 that receives
// clock64 pipeline events of CTA 0 in builds compiled with -DTLATTN_TRACE.
extern "C" int tl_attn_debug_trace(void* dev_buf) {
#ifdef TLATTN_TRACE
  g_trace = static_cast<unsigned long long*>(dev_buf);
  return TL_OK;
#else
  (void)dev_buf;
  return TL_ERR_UNSUPPORTED;
#endif
}

extern "C" int tl_attn_last_launch_count(void) { return g_last_launches; }
