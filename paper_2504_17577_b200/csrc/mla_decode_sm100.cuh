// mla_decode_sm100.cuh — MLA decode attention for B200 (sm_100a), SURVEY §8(f) N1.
//
// What it computes: PAPER.md Appendix B.3, Fig. 18, see include/tlattn.h
// tl_mla_decode: per (b, h) one query against the latent cache, scores
// s_j = scale (q.kv_j + q_pe.kpe_j) (two T.gemm into acc_s), online softmax
// (P:L660-679), O = softmax . KV (the value operand is KV_shared itself).
//
// B200 design. Fig. 18 tiles heads as the GEMM M dimension with a
// [block_H x 512] fp32 accumulator in registers (Hopper wgmma). On sm_100 the accumulator
// lives in TMEM: 128 heads x 512 fp32 would fill all 512 columns of an SM, leaving no room
// for the score tile. So the tile is transposed — keys are the M dimension:
//   S^T [128 keys x HC heads] = Khat [128 keys x 576] . Qhat^T      (tcgen05, TMEM)
//   O^T [512 dv x HC heads]  += V^T  [512 x 128 keys] . P^T           (4 MMAs of M=128)
// with HC = 32 query heads per CTA: TMEM = 2 x 32 (S^T double buffer) + 4 x 32 (O^T).
// One thread per key row (TMEM lane) does the softmax; per-head (column) max and sum
// are warp transposed-butterfly reductions plus a 4-warp smem step; l is kept as
// per-thread partial sums and reduced once per segment.
//
//   warp 0     TMA producer: Qhat (8 x [32 heads x 64] + q_pe) once per segment, then per
//              key block the K_pe chunk and four "pair" slots (KV dims [128m, 128m+128) as two
//              [128 keys x 64] SWIZZLE_128B boxes). The pair slots are both the QK^T operand
//              and, unchanged, the V^T operand of PV: each KV byte crosses L2 -> SM once per
//              head tile. Five pair slots = one resident block + one prefetched pair.
//              (Measured: re-reading V from L2 instead costs 1.85x the L2 -> SM bytes, and on
//              B200 L2 -> SM traffic saturates near the HBM rate.)
//   warp 1     MMA issuer (one thread): S(j+1) part A (K_pe, pair 0) -> PV(j) -> S(j+1) part B,
//              so the tensor core computes the next scores while the softmax of block j runs.
//   warps 4-7  softmax + epilogue.
// Work split (split-KV, the FlashDecoding / FlashMLA scheme; Fig. 18 has one CTA per
// (batch, head block), which leaves most of 148 SMs idle at decode batch sizes): the key
// blocks of all batches are concatenated (cum[] from tl_mla_meta_kernel) and each CTA of a
// head tile takes an equal contiguous range; a range piece that covers a whole batch writes
// O directly, partial pieces write fp32 (O, lse) to the workspace and tl_mla_combine_kernel
// merges them.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <type_traits>

#include "attn_fwd_sm100.cuh"  // pack2
#include "ptx.cuh"

namespace tlattn {
namespace mla {

constexpr int DL = 512;             // latent (kv_lora) dim, Fig. 18 `dim`
constexpr int DR = 64;              // rope dim, Fig. 18 `pe_dim`
constexpr int BLK = 128;            // keys per block (tcgen05 M of S^T)
constexpr int NKCH = DL / 64 + 1;   // Khat chunks per block: 8 of KV + 1 of K_pe
constexpr int NPAIRS_PER_BLK = DL / 128;  // 4 pair slots per block: KV dims [128m, 128m+128)
constexpr int SLOT = 16384;         // one [128 keys x 64] 16-bit SWIZZLE_128B box
constexpr float RESCALE_LOG2 = 8.0f;  // conditional rescale threshold (as the attention kernel)
constexpr int HC_MAX = 64;

// Per head-tile width HC (query heads per CTA = tcgen05 N of both MMAs):
//  HC = 32: SMEM = 5 pair slots (one block resident + one pair prefetched) + K_pe slot +
//           Qhat 36 KB + P^T 8 KB (64-B rows, SWIZZLE_64B);
//  HC = 64: SMEM = 4 pair slots + K_pe slot + Qhat 72 KB; P^T (128-B rows, SWIZZLE_128B,
//           16 KB) shares the K_pe slot (K_pe(j) is consumed by S(j) before softmax(j)
//           writes P^T(j); K_pe(j+1) is loaded after PV(j) read it), so block j+1 is
//           loaded while PV(j) frees the pair slots (no prefetch).
template <int HC>
struct Cfg {
  static_assert(HC == 32 || HC == 64, "head tile");
  static constexpr int NSW = HC / 32;                // softmax warpgroups (32 heads each)
  static constexpr int THREADS = 128 + 128 * NSW;    // producer, MMA, 2 spare warps + softmax
  static constexpr bool PREFETCH = HC == 32;
  static constexpr int NPAIR = PREFETCH ? 5 : 4;
  static constexpr int QCH = HC * 128;               // one [HC heads x 64] SW128 chunk of Qhat
  static constexpr int PBYTES = BLK * HC * 2;        // P^T [128 keys x HC heads]
  static constexpr uint32_t P_LAYOUT = HC == 32 ? 4u : 2u;  // SWIZZLE_64B / SWIZZLE_128B
  static constexpr uint32_t P_ROW = HC * 2;          // bytes per key row of P^T
  static constexpr uint32_t TM_S = 0;                // S^T buffers at columns 0, HC
  static constexpr uint32_t TM_O = 2 * HC;           // O^T dv chunk m at 2 HC + HC m
  static constexpr uint32_t TMEM_COLS = HC == 32 ? 256 : 512;
  static constexpr int OFF_PAIR = 0;
  static constexpr int OFF_PE = OFF_PAIR + NPAIR * 2 * SLOT;
  static constexpr int OFF_Q = OFF_PE + SLOT;
  static constexpr int OFF_P = PREFETCH ? OFF_Q + NKCH * QCH : OFF_PE;
  static constexpr int OFF_RED = OFF_Q + NKCH * QCH + (PREFETCH ? PBYTES : 0);
  // per softmax group: red[2][4][32] + redl[4][32] floats, then mbc[2][2][32] floats
  static constexpr int OFF_MBC = OFF_RED + NSW * 3 * 4 * 32 * 4;
  static constexpr int OFF_BAR = OFF_MBC + NSW * 2 * 2 * 32 * 4;
  // pair_full/empty[NPAIR], pe_full, pe_empty, q_full, q_empty, s_full[2], s_free[2], p_full,
  // o_done, o_free
  static constexpr int NUM_BARS = 2 * NPAIR + 2 + 9;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget exceeded");
  static_assert(PREFETCH || PBYTES <= SLOT, "P^T must fit the K_pe slot");
};

struct MlaParams {
  CUtensorMap tm_q;    // q   [B][H][DL]       as (DL, H, 1, B),   box (64, HC, 1, 1)
  CUtensorMap tm_qpe;  // q_pe[B][H][DR]       as (DR, H, 1, B),   box (64, HC, 1, 1)
  CUtensorMap tm_k;    // kv  [B][Skv][Hkv][DL] as (DL, Hkv, Skv, B), box (64, 1, 128, 1)
  CUtensorMap tm_kpe;  // k_pe[B][Skv][Hkv][DR], box (64, 1, 128, 1)
  void* o;             // [B][H][DL]
  float* lse;          // [B][H] natural log, or nullptr
  const int* seqlens;  // [B] or nullptr (= Skv)
  int* cum;            // workspace: [B+1] prefix sums of key blocks per batch
  float* ws_o;         // workspace: [NHG][P][2][HC][DL] partial O (normalised)
  float* ws_lse;       // workspace: [NHG][P][2][HC] partial lse (log2 units)
  int HC;              // query heads per CTA (32 or 64)
  int B, H, Hkv, Skv;
  int g;               // H / Hkv (query heads per kv head)
  int T;               // head tiles per kv head = ceil(g / HC)
  int P;               // partitions (CTAs) per head tile
  int CL;              // cluster size: CL head tiles of one kv head share every K/V load
                       // (TMA multicast); 1, 2 or 4, divides T
  float c_log2;        // |scale| log2(e)
  int neg;             // scale < 0: negate Qhat (B operand) in the S^T descriptor
};

__device__ __forceinline__ int seq_len(const MlaParams& p, int b) {
  if (p.seqlens == nullptr) return p.Skv;
  const int n = p.seqlens[b];
  return n < 0 ? 0 : (n > p.Skv ? p.Skv : n);  // documented clamp (tlattn.h)
}

__device__ __forceinline__ long long part_start(int part, long long W, int P) {
  return (long long)part * W / P;
}

// last batch b with cum[b] <= s (and a non-empty key range when s < W)
__device__ __forceinline__ int batch_of(const int* cum, int B, long long s) {
  int lo = 0, hi = B;  // answer in [0, B)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((long long)cum[mid] <= s) lo = mid;
    else hi = mid;
  }
  return lo;
}

// One piece of a partition's block range that lies in one batch.
struct Seg {
  int b, k0, n;   // batch, first block (within the batch), number of blocks
  int len;        // keys of batch b
  bool partial;   // does not cover the whole batch -> workspace
  int slot;       // workspace slot (0 = first piece of the partition, 1 = later)
};

// Iterates the pieces of partition `part` (same sequence in every role).
struct SegIter {
  long long s, e;
  int b;
  bool first;
  __device__ __forceinline__ SegIter(const MlaParams& p, int part) {
    const long long W = p.cum[p.B];
    s = part_start(part, W, p.P);
    e = part_start(part + 1, W, p.P);
    b = (s < e) ? batch_of(p.cum, p.B, s) : 0;
    first = true;
  }
  __device__ __forceinline__ bool next(const MlaParams& p, Seg& sg) {
    if (s >= e) return false;
    const long long c0 = p.cum[b], c1 = p.cum[b + 1];
    const long long stop = e < c1 ? e : c1;
    sg.b = b;
    sg.k0 = (int)(s - c0);
    sg.n = (int)(stop - s);
    sg.len = seq_len(p, b);
    sg.partial = !(s == c0 && stop == c1);
    sg.slot = first ? 0 : 1;
    first = false;
    s = stop;
    ++b;
    while (s < e && b < p.B && (long long)p.cum[b + 1] <= s) ++b;  // skip empty batches
    return true;
  }
};

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                               uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;  // 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
  return d;
}

// Column reduction over the 32 lanes of a warp, "transposed butterfly": in[HC] per lane; on
// exit v[i] (i < HC/32) holds op over the warp of column lane*(HC/32) + i. Each round halves
// the columns a lane keeps (one shuffle per kept column), 31*(HC/32) shuffles in all.
template <int HC, bool MAX>
__device__ __forceinline__ void col_reduce(const float (&in)[HC], float (&v)[HC / 2], int lane) {
  {  // first round (lane distance 16) straight from `in`
    const bool up = (lane & 16) != 0;
#pragma unroll
    for (int i = 0; i < HC / 2; ++i) {
      const float send = up ? in[i] : in[i + HC / 2];
      const float keep = up ? in[i + HC / 2] : in[i];
      const float got = __shfl_xor_sync(0xffffffffu, send, 16);
      v[i] = MAX ? fmaxf(keep, got) : keep + got;
    }
  }
  int n = HC / 2;
#pragma unroll
  for (int d = 8; d >= 1; d >>= 1) {
    const int half = n / 2;
    const bool up = (lane & d) != 0;
#pragma unroll
    for (int i = 0; i < HC / 4; ++i) {
      if (i < half) {
        const float send = up ? v[i] : v[i + half];
        const float keep = up ? v[i + half] : v[i];
        const float got = __shfl_xor_sync(0xffffffffu, send, d);
        v[i] = MAX ? fmaxf(keep, got) : keep + got;
      }
    }
    n = half;
  }
}

template <int HC, bool BF16>
__global__ void __launch_bounds__(Cfg<HC>::THREADS, 1)
tl_mla_decode_kernel(const __grid_constant__ MlaParams p) {
  using C = Cfg<HC>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base = (raw_u32 + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_u32);
  const uint32_t sPair = base + C::OFF_PAIR;
  const uint32_t sPe = base + C::OFF_PE;
  const uint32_t sQ = base + C::OFF_Q;
  const uint32_t sP = base + C::OFF_P;
  float* red_all = reinterpret_cast<float*>(smem + C::OFF_RED);
  float* mbc_all = reinterpret_cast<float*>(smem + C::OFF_MBC);
  const uint32_t bar0 = base + C::OFF_BAR;
  auto bar_pair_full = [&](int s) { return bar0 + 8u * s; };
  auto bar_pair_empty = [&](int s) { return bar0 + 8u * (C::NPAIR + s); };
  const uint32_t bar_pe_full = bar0 + 8u * (2 * C::NPAIR);
  const uint32_t bar_pe_empty = bar_pe_full + 8u;
  const uint32_t bar_x = bar_pe_full + 16u;
  const uint32_t bar_q_full = bar_x;
  const uint32_t bar_q_empty = bar_x + 8u;
  auto bar_s_full = [&](int i) { return bar_x + 8u * (2 + i); };
  auto bar_s_free = [&](int i) { return bar_x + 8u * (4 + i); };
  const uint32_t bar_p_full = bar_x + 8u * 6;
  const uint32_t bar_o_done = bar_x + 8u * 7;
  const uint32_t bar_o_free = bar_x + 8u * 8;
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // cluster = CL head tiles of one kv head over the same partition of the key blocks
  const uint32_t rank = p.CL > 1 ? cluster_ctarank() : 0u;
  const int cid = blockIdx.x / p.CL;
  const int part = cid % p.P;
  const int hgi = (cid / p.P) * p.CL + rank;  // head tile id = kvh * T + t
  const uint16_t mc_mask = static_cast<uint16_t>((1u << p.CL) - 1u);
  const int kvh = hgi / p.T;
  const int t = hgi % p.T;
  const int h0 = kvh * p.g + t * HC;             // first query head of this tile
  const int nvalid = min(HC, p.g - t * HC);      // heads of this tile inside the kv group

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_q);
    prefetch_tmap(&p.tm_qpe);
    prefetch_tmap(&p.tm_k);
    prefetch_tmap(&p.tm_kpe);
    for (int s = 0; s < C::NPAIR; ++s) {
      mbar_init(bar_pair_full(s), 1);
      mbar_init(bar_pair_empty(s), p.CL);  // released by the PV MMAs of every CTA of the cluster
    }
    mbar_init(bar_pe_full, 1);
    mbar_init(bar_pe_empty, p.CL);
    mbar_init(bar_q_full, 1);
    mbar_init(bar_q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_s_full(i), 1);
      mbar_init(bar_s_free(i), 4 * C::NSW);  // every softmax warp
    }
    mbar_init(bar_p_full, 4 * C::NSW);
    mbar_init(bar_o_done, 1);
    mbar_init(bar_o_free, 4 * C::NSW);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(smem_u32(tmem_ptr_smem));
  tc_fence_before();
  if (p.CL > 1) cluster_sync();  // peers' barriers initialised before any multicast / remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr_smem;

  if (warp == 0) {
    // ================================ TMA producer ================================
    // Block j of a segment = four "pair" slots (KV dims [128m, 128m+128) as two
    // [128 keys x 64] SWIZZLE_128B boxes) + the K_pe chunk. The pair slots stay resident from
    // S(j) to PV(j) (they are both the QK^T operand and V). With CL > 1, unit number u (pairs
    // and K_pe counted separately) is loaded by CTA (u % CL) and multicast.
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_first();  // streamed once per head tile
      uint32_t pit = 0, eit = 0;
      int nseg = 0;
      SegIter si(p, part);
      Seg sg;
      auto load = [&](bool mine, uint32_t dst, const CUtensorMap* m, uint32_t fb, int c0, int c1,
                      int c2, int c3, uint64_t pol) {
        if (!mine) return;
        if (p.CL > 1) tma_load_4d_mc(dst, m, fb, c0, c1, c2, c3, mc_mask, pol);
        else tma_load_4d(dst, m, fb, c0, c1, c2, c3, pol);
      };
      auto load_pe = [&](int key0, int b) {
        if (eit >= 1u) mbar_wait(bar_pe_empty, (eit - 1) & 1);
        mbar_arrive_expect_tx(bar_pe_full, SLOT);
        load((eit % p.CL) == rank, sPe, &p.tm_kpe, bar_pe_full, 0, kvh, key0, b, pol_kv);
        ++eit;
      };
      while (si.next(p, sg)) {
        if (nseg > 0) mbar_wait(bar_q_empty, (nseg - 1) & 1);  // previous segment's S MMAs done
        mbar_arrive_expect_tx(bar_q_full, NKCH * C::QCH);
#pragma unroll 1
        for (int c = 0; c < DL / 64; ++c)
          tma_load_4d(sQ + c * C::QCH, &p.tm_q, bar_q_full, c * 64, h0, 0, sg.b, pol_q);
        tma_load_4d(sQ + (DL / 64) * C::QCH, &p.tm_qpe, bar_q_full, 0, h0, 0, sg.b, pol_q);
#pragma unroll 1
        for (int jj = 0; jj < sg.n; ++jj) {
          const int key0 = (sg.k0 + jj) * BLK;
          if constexpr (C::PREFETCH) load_pe(key0, sg.b);  // S(j) starts with K_pe
#pragma unroll 1
          for (int m = 0; m < NPAIRS_PER_BLK; ++m) {
            const int s = pit % C::NPAIR;
            if (pit >= (uint32_t)C::NPAIR) mbar_wait(bar_pair_empty(s), ((pit / C::NPAIR) - 1) & 1);
            mbar_arrive_expect_tx(bar_pair_full(s), 2 * SLOT);
            const bool mine = (pit % p.CL) == rank;
            load(mine, sPair + s * 2 * SLOT, &p.tm_k, bar_pair_full(s), (2 * m) * 64, kvh, key0, sg.b,
                 pol_kv);
            load(mine, sPair + s * 2 * SLOT + SLOT, &p.tm_k, bar_pair_full(s), (2 * m + 1) * 64, kvh,
                 key0, sg.b, pol_kv);
            ++pit;
          }
          if constexpr (!C::PREFETCH) load_pe(key0, sg.b);  // S(j) ends with K_pe (slot = P^T)
        }
        ++nseg;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // HC = 32: S(j+1) part A (K_pe, pair 0 = the prefetched slots) -> PV(j) (frees the pair
    //          slots of block j) -> S(j+1) part B (pairs 1-3): the tensor core computes the
    //          next scores while softmax(j) runs.
    // HC = 64: S(j) (pairs 0-3, then K_pe) -> PV(j) -> S(j+1) ...
    if (lane == 0) {
      constexpr uint32_t FMT = BF16 ? 1u : 0u;
      // S^T = Khat Qhat^T: A = Khat (K-major), B = Qhat (K-major), M=128 keys, N=HC heads
      const uint32_t IDESC_S = make_idesc_f16(FMT, BLK, HC, 0, 0, 0) | ((p.neg ? 1u : 0u) << 14);
      // O^T += V^T P^T: A = V^T (MN-major: dv contiguous), B = P^T (MN-major: heads
      // contiguous), M=128 dv, N=HC heads, K=128 keys
      constexpr uint32_t IDESC_PV = make_idesc_f16(FMT, 128, HC, 1, 1, 0);
      uint32_t pit = 0, eit = 0;  // pair / K_pe positions (same sequence as the producer)
      uint32_t gb = 0;            // global block counter
      int nseg = 0;
      SegIter si(p, part);
      Seg sg;
      // S^T(gs) += Khat chunk . Qhat chunk(c)
      auto s_chunk = [&](uint32_t sb, uint32_t a0, int c, bool first) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_f16_ss(tmem_base + C::TM_S + sb * HC, make_sdesc(a0 + kk * 32, 16, 1024, 2),
                     make_sdesc(sQ + c * C::QCH + kk * 32, 16, 1024, 2), IDESC_S,
                     (first && kk == 0) ? 0u : 1u);
      };
      auto s_pe = [&](uint32_t sb, bool first) {  // K_pe chunk
        mbar_wait(bar_pe_full, eit & 1);
        tc_fence_after();
        s_chunk(sb, sPe, DL / 64, first);
        if constexpr (C::PREFETCH) {  // (HC = 64: the slot is released after PV, as P^T)
          if (p.CL > 1) mma_commit_mc(bar_pe_empty, mc_mask);
          else mma_commit(bar_pe_empty);
        }
        ++eit;
      };
      auto s_pair = [&](uint32_t sb, uint32_t pos, int m, bool first) {
        const int s = pos % C::NPAIR;
        mbar_wait(bar_pair_full(s), (pos / C::NPAIR) & 1);
        tc_fence_after();
        s_chunk(sb, sPair + s * 2 * SLOT, 2 * m, first);
        s_chunk(sb, sPair + s * 2 * SLOT + SLOT, 2 * m + 1, false);
      };
      auto s_begin = [&](uint32_t gs) {
        if (gs >= 2) mbar_wait(bar_s_free(gs & 1), ((gs - 2) >> 1) & 1);
        tc_fence_after();
      };
      auto pv = [&](uint32_t g, uint32_t pos, bool first_blk) {
        mbar_wait(bar_p_full, g & 1);
        tc_fence_after();
#pragma unroll 1
        for (int m = 0; m < NPAIRS_PER_BLK; ++m) {
          const int s = (pos + m) % C::NPAIR;
          const uint32_t a0 = sPair + s * 2 * SLOT;
#pragma unroll
          for (int kk = 0; kk < BLK / 16; ++kk) {
            // A: V^T MN-major SW128, 16 keys = 16 rows of 128 B; LBO = 16 KB to the second
            // 64-wide dv atom of the pair. B: P^T MN-major, 16 keys = 16 rows of P_ROW bytes.
            mma_f16_ss(tmem_base + C::TM_O + m * HC, make_sdesc(a0 + kk * 2048, SLOT, 1024, 2),
                       make_sdesc(sP + kk * 16 * C::P_ROW, 4096, 8 * C::P_ROW, C::P_LAYOUT),
                       IDESC_PV, (!first_blk || kk > 0) ? 1u : 0u);
          }
          if (p.CL > 1) mma_commit_mc(bar_pair_empty(s), mc_mask);
          else mma_commit(bar_pair_empty(s));
        }
        if constexpr (!C::PREFETCH) {  // P^T read: the K_pe slot may be refilled
          if (p.CL > 1) mma_commit_mc(bar_pe_empty, mc_mask);
          else mma_commit(bar_pe_empty);
        }
        mma_commit(bar_o_done);
      };
      while (si.next(p, sg)) {
        mbar_wait(bar_q_full, nseg & 1);
        tc_fence_after();
        const uint32_t pit0 = pit;  // pair position of block 0 of this segment, pair 0
        if constexpr (C::PREFETCH) {
          // S(0), whole
          s_begin(gb);
          s_pe(gb & 1, true);
#pragma unroll 1
          for (int m = 0; m < NPAIRS_PER_BLK; ++m) s_pair(gb & 1, pit0 + m, m, false);
          mma_commit(bar_s_full(gb & 1));
          if (sg.n == 1) mma_commit(bar_q_empty);
#pragma unroll 1
          for (int jj = 0; jj < sg.n; ++jj) {
            const uint32_t g = gb + jj;
            const uint32_t pos = pit0 + NPAIRS_PER_BLK * jj;  // pair 0 of block jj
            const bool more = jj + 1 < sg.n;
            if (more) {  // S(j+1) part A
              s_begin(g + 1);
              s_pe((g + 1) & 1, true);
              s_pair((g + 1) & 1, pos + NPAIRS_PER_BLK, 0, false);
            }
            if (jj == 0 && nseg > 0) mbar_wait(bar_o_free, (nseg - 1) & 1);  // O^T read out
            pv(g, pos, jj == 0);
            if (more) {  // S(j+1) part B
#pragma unroll 1
              for (int m = 1; m < NPAIRS_PER_BLK; ++m)
                s_pair((g + 1) & 1, pos + NPAIRS_PER_BLK + m, m, false);
              mma_commit(bar_s_full((g + 1) & 1));
              if (jj + 2 == sg.n) mma_commit(bar_q_empty);
            }
          }
        } else {
#pragma unroll 1
          for (int jj = 0; jj < sg.n; ++jj) {
            const uint32_t g = gb + jj;
            const uint32_t pos = pit0 + NPAIRS_PER_BLK * jj;
            s_begin(g);
#pragma unroll 1
            for (int m = 0; m < NPAIRS_PER_BLK; ++m) s_pair(g & 1, pos + m, m, m == 0);
            s_pe(g & 1, false);
            mma_commit(bar_s_full(g & 1));
            if (jj + 1 == sg.n) mma_commit(bar_q_empty);
            if (jj == 0 && nseg > 0) mbar_wait(bar_o_free, (nseg - 1) & 1);  // O^T read out
            pv(g, pos, jj == 0);
          }
        }
        pit += NPAIRS_PER_BLK * sg.n;
        gb += sg.n;
        ++nseg;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ============================ softmax + epilogue ============================
    // Warpgroup sw (of HC/32) owns heads [32 sw, 32 sw + 32) of the tile: S^T columns, its
    // 16-B units of the P^T rows, O^T columns. One thread per key row (TMEM lane).
    const int sw = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;  // key within the block == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t col_s = C::TM_S + 32 * sw;   // + sb * HC
    const uint32_t col_o = C::TM_O + 32 * sw;   // + mm * HC
    const int hs = 32 * sw;                      // first head of this warpgroup in the tile
    const uint32_t bar_id = 1 + sw;
    float* red = red_all + sw * (3 * 4 * 32);    // red[2][4][32] + redl[4][32] of this group
    float* redl = red + 2 * 4 * 32;
    float* mbc = mbc_all + sw * (2 * 2 * 32);    // [2 buffers][m_use | alpha][32 heads]
    const float c = p.c_log2;
    const unsigned FULL = 0xffffffffu;
    uint32_t gb = 0;
    int nseg = 0;
    SegIter si(p, part);
    Seg sg;
    while (si.next(p, sg)) {
      float m = -INFINITY;  // running max (log2 units) of head hs + lane (same in all 4 warps)
      float lpart[32];      // this key-thread's share of l for each of the group's heads
#pragma unroll
      for (int h = 0; h < 32; ++h) lpart[h] = 0.f;
#pragma unroll 1
      for (int jj = 0; jj < sg.n; ++jj) {
        const uint32_t gs = gb + jj;
        const uint32_t sb = gs & 1;
        mbar_wait(bar_s_full(sb), (gs >> 1) & 1);
        tc_fence_after();
        float s[32];
        tmem_ld32(tmem_base + lane_off + col_s + sb * HC, *reinterpret_cast<uint32_t(*)[32]>(s));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s_free(sb));
        // tail mask: keys >= len of this batch do not take part (TMA zero-fills beyond Skv)
        if ((sg.k0 + jj) * BLK + row >= sg.len) {
#pragma unroll
          for (int h = 0; h < 32; ++h) s[h] = -INFINITY;
        }
        // per-head (column) max over the 128 keys: transposed butterfly inside the warp
        // (lane l ends with head hs + l), then the 4 warps through smem (T.reduce_max)
        float v[16];
        col_reduce<32, true>(s, v, lane);
        float* rb = red + (gs & 1) * 128;
        rb[q4 * 32 + lane] = v[0];
        named_bar_sync(bar_id, 128);
        const float mx = fmaxf(fmaxf(rb[lane], rb[32 + lane]), fmaxf(rb[64 + lane], rb[96 + lane]));
        const float mxs = (mx == -INFINITY) ? -INFINITY : mx * c;
        const float m_new = (mxs > m + RESCALE_LOG2) ? mxs : m;  // conditional rescale
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        const float alpha = ex2(m - m_use);  // scores_scale; 0 on the first block
        const bool resc = __any_sync(FULL, alpha != 1.f);
        // every thread needs m_use / alpha of all 32 heads: warp q4 == 0 publishes them
        // (the 4 warps computed identical values) and the group reads them as broadcasts
        float* mb = mbc + (gs & 1) * 64;
        if (q4 == 0) {
          mb[lane] = m_use;
          mb[32 + lane] = alpha;
        }
        named_bar_sync(bar_id, 128);
        float mu[32];
#pragma unroll
        for (int h = 0; h < 32; h += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(mb + h);
          mu[h] = t4.x; mu[h + 1] = t4.y; mu[h + 2] = t4.z; mu[h + 3] = t4.w;
        }
        if (resc) {
#pragma unroll
          for (int h = 0; h < 32; h += 4) {
            const float4 a4 = *reinterpret_cast<const float4*>(mb + 32 + h);
            lpart[h] *= a4.x; lpart[h + 1] *= a4.y; lpart[h + 2] *= a4.z; lpart[h + 3] *= a4.w;
          }
        }
        // p = exp2(s c - m_head), l partial sums from the unrounded p (R8)
        uint32_t pk[16];
#pragma unroll
        for (int h = 0; h < 32; h += 2) {
          const float p0 = ex2(fmaf(s[h], c, -mu[h]));
          const float p1 = ex2(fmaf(s[h + 1], c, -mu[h + 1]));
          lpart[h] += p0;
          lpart[h + 1] += p1;
          pk[h / 2] = pack2<BF16>(p0, p1);  // P rounded RN to the dtype (S_shared)
        }
        // the P^T buffer and O^T are free once PV(gs-1) completed
        if (gs >= 1) mbar_wait(bar_o_done, (gs - 1) & 1);
        if (resc && jj > 0) {
          // acc_o *= scores_scale: O^T columns are heads
          tc_fence_after();
#pragma unroll 1
          for (int mm = 0; mm < DL / 128; ++mm) {
            uint32_t ov[32];
            const uint32_t ta = tmem_base + lane_off + col_o + mm * HC;
            tmem_ld32(ta, ov);
            tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < 32; ++h) ov[h] = __float_as_uint(__uint_as_float(ov[h]) * mb[32 + h]);
            tmem_st32(ta, ov);
          }
          tmem_st_wait();
        }
        // P^T row (this key) -> smem, MN-major: HC = 32 SWIZZLE_64B (16-B unit u of row r at
        // u ^ ((r >> 1) & 3)), HC = 64 SWIZZLE_128B (unit u at u ^ (r & 7)); this group
        // writes units [4 sw, 4 sw + 4)
        const uint32_t prow = sP + row * C::P_ROW;
#pragma unroll
        for (int u0 = 0; u0 < 4; ++u0) {
          const int u = 4 * sw + u0;
          const uint32_t pu = HC == 32 ? (u ^ ((row >> 1) & 3)) : (u ^ (row & 7));
          st_shared_v4(prow + (pu << 4), pk[4 * u0], pk[4 * u0 + 1], pk[4 * u0 + 2], pk[4 * u0 + 3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p_full);
        m = m_new;
      }
      // ---- epilogue: l = sum of the partial sums, O = O^T / l, LSE
      const uint32_t glast = gb + sg.n - 1;
      mbar_wait(bar_o_done, glast & 1);
      tc_fence_after();
      {
        float v[16];
        col_reduce<32, false>(lpart, v, lane);
        redl[q4 * 32 + lane] = v[0];
      }
      named_bar_sync(bar_id, 128);
      const float L = (redl[lane] + redl[32 + lane]) + (redl[64 + lane] + redl[96 + lane]);
      const float m_fin = (m == -INFINITY) ? 0.f : m;
      const float inv = (L > 0.f) ? 1.f / L : 0.f;
      const float lse2 = (L > 0.f) ? m_fin + __log2f(L) : -INFINITY;
      float iv[32];
#pragma unroll
      for (int h = 0; h < 32; ++h) iv[h] = __shfl_sync(FULL, inv, h);
      const size_t wslot = ((size_t)(hgi * p.P + part) * 2 + sg.slot);
#pragma unroll 1
      for (int mm = 0; mm < DL / 128; ++mm) {
        const int dv = mm * 128 + row;
        uint32_t ov[32];
        tmem_ld32(tmem_base + lane_off + col_o + mm * HC, ov);
        tmem_ld_wait();
        if (!sg.partial) {
          using T16 = typename std::conditional<BF16, __nv_bfloat16, __half>::type;
          T16* ob = reinterpret_cast<T16*>(p.o) + ((size_t)sg.b * p.H + h0 + hs) * DL + dv;
#pragma unroll
          for (int h = 0; h < 32; ++h) {
            if (hs + h < nvalid) {
              const float x = __uint_as_float(ov[h]) * iv[h];
              if constexpr (BF16) ob[(size_t)h * DL] = __float2bfloat16_rn(x);
              else ob[(size_t)h * DL] = __float2half_rn(x);
            }
          }
        } else {
          float* wo = p.ws_o + (wslot * HC + hs) * DL + dv;
#pragma unroll
          for (int h = 0; h < 32; ++h) wo[(size_t)h * DL] = __uint_as_float(ov[h]) * iv[h];
        }
      }
      if (q4 == 0) {
        const int hh = hs + lane;
        if (!sg.partial) {
          if (p.lse != nullptr && hh < nvalid)
            p.lse[(size_t)sg.b * p.H + h0 + hh] = lse2 * 0.69314718055994531f;
        } else {
          p.ws_lse[wslot * HC + hh] = lse2;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_o_free);
      gb += sg.n;
      ++nseg;
    }
  }

  // every MMA of this CTA has completed (softmax waited the last PV), so all its multicast
  // releases have landed in the peers; no CTA leaves while a peer may still signal it
  if (p.CL > 1) cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// cum[b] = sum_{b' < b} ceil(len_b' / BLK), cum[B] = W. One CTA, chunked block scan.
__global__ void __launch_bounds__(1024) tl_mla_meta_kernel(const int* seqlens, int B, int Skv, int* cum) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base0 = 0; base0 < B; base0 += 1024) {
    const int b = base0 + threadIdx.x;
    int n = 0;
    if (b < B) {
      int len = seqlens ? seqlens[b] : Skv;
      len = len < 0 ? 0 : (len > Skv ? Skv : len);
      n = (len + BLK - 1) / BLK;
    }
    int x = n;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int excl = carry + (wid > 0 ? warp_sums[wid - 1] : 0) + x - n;
    if (b < B) cum[b] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + n;
    __syncthreads();
  }
  if (threadIdx.x == 0) cum[B] = carry;
}

// Merge the partial (O, lse) pieces of split batches; write zeros / -inf for empty ones.
// Grid: (B, Hkv * T); 256 threads: warp w handles heads w, w+8, ... of the tile.
template <bool BF16>
__global__ void __launch_bounds__(256) tl_mla_combine_kernel(const __grid_constant__ MlaParams p) {
  const int b = blockIdx.x;
  const int hgi = blockIdx.y;
  const int kvh = hgi / p.T, t = hgi % p.T;
  const int HC = p.HC;
  const int h0 = kvh * p.g + t * HC;
  const int nvalid = min(HC, p.g - t * HC);
  const long long W = p.cum[p.B];
  const long long c0 = p.cum[b], c1 = p.cum[b + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  using T16 = typename std::conditional<BF16, __nv_bfloat16, __half>::type;
  T16* ob = reinterpret_cast<T16*>(p.o) + ((size_t)b * p.H + h0) * DL;
  if (c1 == c0) {  // no keys (seqlens[b] == 0): O = 0, LSE = -inf (reading M1 / R4)
    for (int h = warp; h < nvalid; h += 8) {
      for (int d = lane; d < DL; d += 32) {
        if constexpr (BF16) ob[(size_t)h * DL + d] = __float2bfloat16_rn(0.f);
        else ob[(size_t)h * DL + d] = __float2half_rn(0.f);
      }
      if (p.lse != nullptr && lane == 0) p.lse[(size_t)b * p.H + h0 + h] = -INFINITY;
    }
    return;
  }
  // partitions covering [c0, c1): p_lo = last with start <= c0, p_hi = last with start <= c1-1
  auto last_start_le = [&](long long x) {
    int q = (int)((x * p.P) / W);
    while (q + 1 < p.P && part_start(q + 1, W, p.P) <= x) ++q;
    while (q > 0 && part_start(q, W, p.P) > x) --q;
    return q;
  };
  const int p_lo = last_start_le(c0), p_hi = last_start_le(c1 - 1);
  if (p_lo == p_hi) return;  // one piece: the decode kernel wrote O / LSE directly
  for (int h = warp; h < nvalid; h += 8) {
    float mx = -INFINITY;
    for (int q = p_lo; q <= p_hi; ++q) {
      if (part_start(q, W, p.P) == part_start(q + 1, W, p.P)) continue;  // empty partition
      const int slot = (part_start(q, W, p.P) >= c0) ? 0 : 1;
      mx = fmaxf(mx, p.ws_lse[((size_t)(hgi * p.P + q) * 2 + slot) * HC + h]);
    }
    float acc[DL / 32];
#pragma unroll
    for (int i = 0; i < DL / 32; ++i) acc[i] = 0.f;
    float L = 0.f;
    for (int q = p_lo; q <= p_hi; ++q) {
      if (part_start(q, W, p.P) == part_start(q + 1, W, p.P)) continue;
      const int slot = (part_start(q, W, p.P) >= c0) ? 0 : 1;
      const size_t ws = (size_t)(hgi * p.P + q) * 2 + slot;
      const float w = ex2(p.ws_lse[ws * HC + h] - mx);
      L += w;
      const float* src = p.ws_o + (ws * HC + h) * DL;
#pragma unroll
      for (int i = 0; i < DL / 32; ++i) acc[i] = fmaf(w, src[i * 32 + lane], acc[i]);
    }
    const float inv = 1.f / L;
#pragma unroll
    for (int i = 0; i < DL / 32; ++i) {
      if constexpr (BF16) ob[(size_t)h * DL + i * 32 + lane] = __float2bfloat16_rn(acc[i] * inv);
      else ob[(size_t)h * DL + i * 32 + lane] = __float2half_rn(acc[i] * inv);
    }
    if (p.lse != nullptr && lane == 0)
      p.lse[(size_t)b * p.H + h0 + h] = (mx + __log2f(L)) * 0.69314718055994531f;
  }
}

}  // namespace mla
}  // namespace tlattn
