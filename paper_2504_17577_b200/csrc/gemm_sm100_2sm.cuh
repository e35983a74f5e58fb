// gemm_sm100_2sm.cuh — dense GEMM C = A · B on CTA pairs (PAPER.md
// Fig. 1 / Fig. 16 "Matmul"; shapes Table 2).
//
//   A [M][K] row-major (K contiguous), B [K][N] row-major (N contiguous), C [M][N] in the
//   input dtype, fp32 accumulation (T.gemm into C_local, then T.copy to C).
//
// B200 design (the paper's Hopper/Ampere schedules are prior art): one cluster of 2 CTAs
// per 256 x 256 output tile (M split 128/128 across the pair, B's N split 128/128), K in
// 64-element stages through a 6-deep TMA ring (A box 64 x 128, B boxes 64 x 64, SW128),
// tcgen05.mma.cta_group::2 M=256 N=256 K=16 issued by the leader, fp32 accumulators in
// TMEM double-buffered (2 x 256 columns) so the epilogue of one tile overlaps the
// main loop of the next, epilogue TMEM -> registers -> RN -> SW128 smem -> TMA store,
// persistent over tiles with cluster-launch-control work stealing.
#pragma once
#include "attn_fwd_sm100.cuh"

namespace tlattn {

struct GemmParams {
  CUtensorMap tm_a;  // A as 2-D (K, M), box (64, 128)
  CUtensorMap tm_b;  // B as 2-D (N, K), box (64, 64)
  CUtensorMap tm_c;  // C as 2-D (N, M), box (64, 128)
  int M, N, K;
  int tiles_m, tiles_n;  // ceil(M/256), ceil(N/256)
  int group_n;           // tile raster: groups of group_n tile columns (L2 reuse of B)
};

struct GCfg {
  static constexpr int BK = 64;
  static constexpr int A_STAGE = 128 * BK * 2;   // 16 KB: this CTA's 128 rows
  static constexpr int B_CHUNK = BK * 64 * 2;    // 8 KB: 64 K-rows x 64 N
  static constexpr int B_STAGE = 2 * B_CHUNK;    // this CTA's 128 N columns
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int NST = 6;
  static constexpr int C_STAGE = 128 * 64 * 2;   // 16 KB: 128 rows x 64 cols (one TMA box)
  static constexpr int OFF_RING = 0;
  static constexpr int OFF_C = OFF_RING + NST * STAGE;  // 2 C boxes (double-buffered)
  static constexpr int OFF_SCHED = OFF_C + 2 * C_STAGE;
  // full[NST], empty[NST], acc_full[2], acc_empty[2], sched_full[2], sched_empty[2]
  static constexpr int OFF_BAR = OFF_SCHED + 32;
  static constexpr int NUM_BARS = 2 * NST + 8;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16;  // base is 1024-aligned (checked)
  static_assert(SMEM_BYTES <= 232448, "shared memory budget exceeded");
  static constexpr int THREADS = 256;  // warp 0 TMA, warp 1 MMA, warps 4-7 epilogue
};

__device__ __forceinline__ void gemm_tile_coords(int tile, const GemmParams& p, int& tm, int& tn) {
  // rasterise in groups of group_n tile columns: consecutive tiles share B columns in L2
  const int per_group = p.group_n * p.tiles_m;
  const int gidx = tile / per_group;
  const int first_n = gidx * p.group_n;
  const int gw = min(p.group_n, p.tiles_n - first_n);
  const int r = tile - gidx * per_group;
  tm = r / gw;
  tn = first_n + r % gw;
}

template <bool BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GCfg::THREADS, 1)
tl_gemm_kernel_2sm(const __grid_constant__ GemmParams p) {
  using C = GCfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  if ((base & 1023u) != 0u) __trap();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const uint32_t sRing = base + C::OFF_RING;
  const uint32_t sC = base + C::OFF_C;
  const uint32_t sSched = base + C::OFF_SCHED;
  const uint32_t bar0 = base + C::OFF_BAR;
  auto bar_full = [&](int s) { return bar0 + 8u * s; };
  auto bar_empty = [&](int s) { return bar0 + 8u * (C::NST + s); };
  auto bar_acc_full = [&](int i) { return bar0 + 8u * (2 * C::NST + i); };
  auto bar_acc_empty = [&](int i) { return bar0 + 8u * (2 * C::NST + 2 + i); };
  auto bar_sched_full = [&](int i) { return bar0 + 8u * (2 * C::NST + 4 + i); };
  auto bar_sched_empty = [&](int i) { return bar0 + 8u * (2 * C::NST + 6 + i); };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem_raw + C::OFF_TMEMPTR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int kblocks = (p.K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_a);
    prefetch_tmap(&p.tm_b);
    prefetch_tmap(&p.tm_c);
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_empty(s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_acc_full(i), 1);
      mbar_init(bar_acc_empty(i), 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
      mbar_init(bar_sched_full(i), 1);
      mbar_init(bar_sched_empty(i), 1 + 8 + 1);  // MMA, epilogue warps x2 CTAs, peer producer
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm<TMEM_COLS>(smem_u32(tmem_ptr_smem));
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr_smem;

  if (warp == 0) {
    // ======================= TMA producer (both CTAs) + CLC (leader) =======================
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int tile = blockIdx.x >> 1;
      int it = 0;
      for (int k = 0;; ++k) {
        const int sl = k & 1;
        mbar_arrive_expect_tx(bar_sched_full(sl), 16);
        if (leader) {
          if (k >= 2) mbar_wait(bar_sched_empty(sl), ((k >> 1) - 1) & 1);
          clc_try_cancel_multicast(sSched + 16 * sl, bar_sched_full(sl));
        }
        int tm, tn;
        gemm_tile_coords(tile, p, tm, tn);
        const int m0 = tm * 256 + 128 * (int)rank;  // this CTA's A rows
        const int n0 = tn * 256 + 128 * (int)rank;  // this CTA's B columns
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % C::NST;
          const int use = it / C::NST;
          if (use > 0) mbar_wait(bar_empty(s), (use - 1) & 1);
          if (leader) mbar_arrive_expect_tx(bar_full(s), 2 * C::STAGE);
          const uint32_t lead_full = mapa_shared(bar_full(s), 0);
          const uint32_t dst = sRing + s * C::STAGE;
          tma_load_4d_2sm(dst, &p.tm_a, lead_full, kb * C::BK, m0, 0, 0, pol_a);
          tma_load_4d_2sm(dst + C::A_STAGE, &p.tm_b, lead_full, n0, kb * C::BK, 0, 0, pol_b);
          tma_load_4d_2sm(dst + C::A_STAGE + C::B_CHUNK, &p.tm_b, lead_full, n0 + 64, kb * C::BK, 0, 0,
                          pol_b);
        }
        mbar_wait(bar_sched_full(sl), (k >> 1) & 1);
        const int nxt = clc_query(sSched + 16 * sl);
        if (!leader) mbar_arrive_cluster(mapa_shared(bar_sched_empty(sl), 0));
        if (nxt < 0) break;
        tile = nxt >> 1;
      }
    }
    __syncwarp();
  } else if (warp == 1 && leader) {
    // ======================= MMA issuer (leader, one thread) =======================
    if (lane == 0) {
      constexpr uint32_t FMT = BF16 ? 1u : 0u;
      // M=256 (A rows split over the pair), N=256 (B columns split), A K-major, B MN-major
      constexpr uint32_t IDESC = make_idesc_f16(FMT, 256, 256, 0, 1, 0);
      int tile = blockIdx.x >> 1;
      int it = 0;
      for (int k = 0;; ++k) {
        const int ab = k & 1;  // accumulator buffer
        if (k >= 2) mbar_wait(bar_acc_empty(ab), ((k >> 1) - 1) & 1);  // epilogue drained it
        tc_fence_after();
        const uint32_t tm_acc = tmem_base + ab * 256;
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % C::NST;
          mbar_wait(bar_full(s), (it / C::NST) & 1);
          tc_fence_after();
          const uint32_t a = sRing + s * C::STAGE;
          const uint32_t b = a + C::A_STAGE;
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            // A: K-major SW128, +32 B per 16-element K step. B: MN-major SW128, 16 K-rows of
            // 128 B per step (+2 KB), LBO = 8 KB to the second 64-wide N chunk.
            mma_f16_ss_2sm(tm_acc, make_sdesc_sw128(a + kk * 32, 16, 1024),
                           make_sdesc_sw128(b + kk * 2048, C::B_CHUNK, 1024), IDESC,
                           (kb > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit_2sm(bar_empty(s));
        }
        mma_commit_2sm(bar_acc_full(ab));
        mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
        const int nxt = clc_query(sSched + 16 * (k & 1));
        mbar_arrive(bar_sched_empty(k & 1));
        if (nxt < 0) break;
        tile = nxt >> 1;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ============== epilogue (both CTAs): TMEM -> RN -> smem (SW128) -> TMA store ==============
    const int q4 = warp & 3;
    const int lr = q4 * 32 + lane;  // row within this CTA's 128 rows (TMEM lane)
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    int tile = blockIdx.x >> 1;
    int nbox = 0;  // boxes stored so far (C staging double buffer)
    for (int k = 0;; ++k) {
      const int ab = k & 1;
      int tm, tn;
      gemm_tile_coords(tile, p, tm, tn);
      mbar_wait(bar_acc_full(ab), (k >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch, ++nbox) {  // 4 boxes of 64 columns
        const int cb = nbox & 1;
        // the staging box we overwrite must have been read by its previous TMA store
        if (threadIdx.x == 128) tma_store_wait_read<1>();
        named_bar_sync(1, 128);
        const uint32_t cbase = sC + cb * C::C_STAGE;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // 2 x 32 columns
          uint32_t v[32];
          tmem_ld32(tmem_base + lane_off + ab * 256 + ch * 64 + h * 32, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = pack2<BF16>(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            const int uu = h * 4 + v4;
            st_shared_v4(cbase + lr * 128 + ((uu ^ (lr & 7)) << 4), pk[4 * v4], pk[4 * v4 + 1],
                         pk[4 * v4 + 2], pk[4 * v4 + 3]);
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == 128) {
          tma_store_4d(&p.tm_c, cbase, tn * 256 + ch * 64, tm * 256 + 128 * (int)rank, 0, 0);
          tma_store_commit();
        }
      }
      // accumulator buffer ab fully read: the MMA may reuse it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(bar_acc_empty(ab), 0));
      mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
      const int nxt = clc_query(sSched + 16 * (k & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(bar_sched_empty(k & 1), 0));
      if (nxt < 0) break;
      tile = nxt >> 1;
    }
    if (threadIdx.x == 128) tma_store_wait_all<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tlattn
