// attn_fwd_sm100_2sm.cuh — the D=128 fused attention forward on a CTA PAIR (2 SMs).
//
// Same computation as attn_fwd_sm100.cuh (include/tlattn.h; Fig. 18),
// re-tiled for Blackwell's 2-SM tensor-core mode (tcgen05 .cta_group::2):
//
//   cluster of 2 CTAs (leader rank 0, peer rank 1) on one TPC = one unit of 512 query
//   rows of one (b, h). Query tile t (t = 0, 1) is an M = 256 MMA tile: the leader
//   holds its rows [r0+256t, +128), the peer [r0+256t+128, +128), each in its own smem
//   (A operand) and TMEM (accumulators S_t, O_t for its 128 rows).
//   K_j / V_j blocks are SPLIT between the pair (B operand N-split): the leader holds
//   keys [0, 64) of K_j and D-columns [0, 64) of V_j, the peer the other halves. Each
//   SM therefore streams half of every K/V tile from L2 (half the TMA traffic, half the
//   ring slot size -> a 6-deep ring), and each operand byte read from smem serves 256
//   query rows instead of 128.
//   The leader's warps 1/2 issue tcgen05.mma.cta_group::2 (one issuer per query tile);
//   commits are multicast to both CTAs' barriers. Each CTA runs its own producer and two
//   softmax warpgroups on its own rows; their S-read / P-written signals arrive on the
//   leader's barriers (remote mbarrier arrive, cluster scope).
//
//   The two query tiles of a unit run in two independent "slots" (slot t = TMEM S_t / O_t,
//   smem Q_t / P_t, issuer warp 1+t, softmax warpgroup t). Each slot's Q tile is loaded
//   (both halves, by the peer's warp 1+t) as soon as its previous tile's last QK^T has
//   completed, and the (at most 2) key blocks only the longer tile of a causal unit needs
//   are released by that tile's issuer alone (two commits on the ring slot's "empty"
//   barrier). So the slot that finishes a unit first starts the next unit while the other
//   slot still works through its extra blocks, instead of idling until both are done;
//   the longer tile of the next unit goes to the slot that is ahead (slot_assign). When the
//   tiles differ by more (a tile past the end of Sq) the slots walk the ring in step.
#pragma once
#include "attn_fwd_sm100.cuh"

namespace tlattn {

struct KCfg2 {
  static constexpr int D = 128;
  static constexpr int Q_TILE_BYTES = BM * D * 2;       // this CTA's 128 rows of tile t
  static constexpr int K_HALF_CHUNK = 64 * 128;          // 64 keys x 64 elems (SW128 box)
  static constexpr int SLOT_BYTES = 16384;               // K half (2 x 8 KB) or V half (16 KB)
  static constexpr int NST = 6;
  static constexpr int P_TILE_BYTES = BM * BN * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + TILES * Q_TILE_BYTES;
  static constexpr int OFF_P = OFF_KV + NST * SLOT_BYTES;
  static constexpr int OFF_SCHED = OFF_P + TILES * P_TILE_BYTES;
  static constexpr int OFF_BAR = OFF_SCHED + 32;
  static constexpr int NUM_BARS = 2 + 2 * NST + 20;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_USED = OFF_TMEMPTR + 16;
  static constexpr int SMEM_BYTES = SMEM_USED + 1024;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget exceeded");
  static constexpr uint32_t TMEM_O = 2 * BN;
  static constexpr int UNIT_ROWS = 2 * TILES * BM;  // 512 query rows per CTA pair (256 in
                                                    // the short-sequence mode)
};

// K/V blocks a 256-row tile starting at r0 visits (causal tile skipping on the pair tile)
__device__ __forceinline__ int tile_nblocks_rows(int r0, int rows, const AttnParams& p) {
  if (r0 >= p.Sq) return 0;
  const int n_all = (p.Skv + BN - 1) / BN;
  if (!p.causal) return n_all;
  const int r_last = min(r0 + rows - 1, p.Sq - 1);
  const long long kmax = (long long)r_last + p.Skv - p.Sq;
  if (kmax < 0) return 0;
  return min(n_all, (int)(kmax / BN) + 1);
}

// P_t is written in NPIECE pieces of BN / NPIECE keys, each with its own "P written"
// barrier, so PV_t(j)'s first K=16 steps start while the softmax still computes the rest
// of the row. Measured on B200: 2 pieces T0 1310 -> 1405 TFLOP/s, C2
// 1248 -> 1336; 4 pieces lose (register spills, one proxy fence per piece).
// TLATTN_PSPLIT=1 (experiments only) restores the single P write.
#ifndef TLATTN_PSPLIT
#define TLATTN_PSPLIT 2
#endif
constexpr int NPIECE = TLATTN_PSPLIT;
constexpr bool P_SPLIT = NPIECE > 1;
static_assert(NPIECE == 1 || NPIECE == 2 || NPIECE == 4, "P pieces: 1, 2 or 4");

struct Unit2 {
  int b, h, hkv, r0, n0, n1;
  int tiles;  // query tiles this unit owns (2, or 1 in the short-sequence mode)
};

__device__ __forceinline__ Unit2 decode_unit2(int u, const AttnParams& p) {
  Unit2 U;
  // n_mblk = ceil(Sq / (256 * unit_tiles)) for this kernel
  const int mb_i = p.lpt ? p.fd_nbh.div(u) : p.fd_mblk.mod(u);
  const int bh = p.lpt ? p.fd_nbh.mod(u) : p.fd_mblk.div(u);
  U.b = p.fd_hq.div(bh);
  U.h = bh - U.b * p.Hq;
  const int m_blk = p.causal ? (p.n_mblk - 1 - mb_i) : mb_i;
  U.hkv = p.fd_grp.div(U.h);  // GQA grouping h / (Hq / Hkv)
  U.tiles = p.unit_tiles;
  U.r0 = m_blk * (2 * BM) * p.unit_tiles;
  U.n0 = tile_nblocks_rows(U.r0, 2 * BM, p);
  U.n1 = p.unit_tiles == 2 ? tile_nblocks_rows(U.r0 + 2 * BM, 2 * BM, p) : 0;
  return U;
}

// Which query tile of unit U slot t runs (tau = 0 / 1, or -1: none), its block count n and
// the other slot's block count n_oth (blocks j >= n_oth are this slot's alone). p0 / p1
// count the blocks each slot has been given so far (every role keeps its own copy and
// updates it identically): the slot that is ahead (fewer blocks so far, so it finishes its
// current tile first) gets the longer tile, so both slots tend to finish the unit together
// and a slot's extra causal blocks overlap the other slot's next tile. Ties give the longer
// tile to slot 1. One-tile units (short-sequence mode) always run in slot 0: a slot may run
// ahead of the other only by the <= 4 ring items of a causal unit's extra blocks (fewer than
// the NST = 6 ring slots, so a waiter is never two phases ahead of a slot's "full" barrier);
// one-tile units alternating between slots would let a slot jump a whole unit of items ahead
// and read a "full" phase of the previous revolution (parity aliasing: measured hang).
// n_skip: blocks [n, n_skip) this slot's issuer still waits for and releases (one commit
// each, the other slot's issuer commits once too): set when the other tile is longer by
// more than 2 blocks (a tile past the end of Sq), where skipping them would let this slot
// jump more than the 4-item bound ahead (see above); otherwise n_skip = n and the longer
// tile's issuer releases its extra blocks alone (j >= n_oth: two commits).
struct SlotAsg {
  int tau, n, n_oth, n_skip;
};
__device__ __forceinline__ SlotAsg slot_assign(const Unit2& U, int t, int& p0, int& p1) {
  SlotAsg a;
  if (U.tiles == 1) {
    a.tau = (t == 0) ? 0 : -1;
    a.n = (t == 0) ? U.n0 : 0;
    a.n_oth = (t == 0) ? 0 : U.n0;
    a.n_skip = a.n;
    p0 += U.n0;
  } else {
    const int ls = (p0 < p1) ? 0 : 1;
    const int tl = (U.n1 >= U.n0) ? 1 : 0;
    const int nl = max(U.n0, U.n1), ns = min(U.n0, U.n1);
    const bool lock = nl - ns > 2;
    a.tau = (t == ls) ? tl : 1 - tl;
    a.n = (t == ls) ? nl : ns;
    a.n_oth = (t == ls) ? (lock ? nl : ns) : nl;
    a.n_skip = (t == ls || !lock) ? a.n : nl;
    if (ls == 0) { p0 += nl; p1 += ns; } else { p1 += nl; p0 += ns; }
  }
  return a;
}

template <bool BF16, class PT = AttnParams>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
tl_attn_fwd_kernel_2sm(const __grid_constant__ PT p) {
  using C = KCfg2;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base = (raw_u32 + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_u32);
  const uint32_t rank = cluster_ctarank();  // 0 = leader, 1 = peer
  const bool leader = rank == 0;

  const uint32_t sQ = base + C::OFF_Q;
  const uint32_t sKV = base + C::OFF_KV;
  const uint32_t sP = base + C::OFF_P;
  const uint32_t sSched = base + C::OFF_SCHED;
  const uint32_t bar0 = base + C::OFF_BAR;
  // per-slot Q barriers: slot 0 at indices 0 / 1, slot 1 at the end of the block
  auto bar_q_full = [&](int t) { return t == 0 ? bar0 : bar0 + 8u * (2 + 2 * C::NST + 18); };
  auto bar_q_empty = [&](int t) { return t == 0 ? bar0 + 8u : bar0 + 8u * (2 + 2 * C::NST + 19); };
  auto bar_kv_full = [&](int s) { return bar0 + 8u * (2 + s); };
  auto bar_kv_empty = [&](int s) { return bar0 + 8u * (2 + C::NST + s); };
  auto bar_s_full = [&](int t) { return bar0 + 8u * (2 + 2 * C::NST + t); };
  auto bar_s_free = [&](int t) { return bar0 + 8u * (4 + 2 * C::NST + t); };
  auto bar_p_full = [&](int t) { return bar0 + 8u * (6 + 2 * C::NST + t); };
  auto bar_o_done = [&](int t) { return bar0 + 8u * (8 + 2 * C::NST + t); };
  auto bar_sched_full = [&](int i) { return bar0 + 8u * (10 + 2 * C::NST + i); };
  auto bar_sched_empty = [&](int i) { return bar0 + 8u * (12 + 2 * C::NST + i); };
  // P_SPLIT: "piece i of P_t written" (piece 0 uses bar_p_full)
  auto bar_p_piece = [&](int t, int i) { return i == 0 ? bar_p_full(t) : bar0 + 8u * (13 + 2 * C::NST + 3 * t + i); };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    TL_SPAN(0);
    prefetch_tmap(&p.tm_q);
    prefetch_tmap(&p.tm_k);
    prefetch_tmap(&p.tm_v);
    for (int t = 0; t < TILES; ++t) {
      mbar_init(bar_q_full(t), 1);   // the leader issuer's expect_tx (+ both halves' bytes)
      mbar_init(bar_q_empty(t), 1);  // commit after the tile's last QK^T
    }
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(bar_kv_full(s), 1);
      mbar_init(bar_kv_empty(s), 2);
    }
    for (int t = 0; t < TILES; ++t) {
      mbar_init(bar_s_full(t), 1);
      mbar_init(bar_s_free(t), 8);  // 4 softmax warps in each CTA (leader's copy is used)
      mbar_init(bar_p_full(t), 8);
      for (int i = 1; i < 4; ++i) mbar_init(bar_p_piece(t, i), 8);
      mbar_init(bar_o_done(t), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_sched_full(i), 1);
      mbar_init(bar_sched_empty(i), 2 + 8 + 8 + 1 + 2);  // issuers, softmax warps x2, peer producer, peer Q loaders
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2sm<TMEM_COLS>(smem_u32(tmem_ptr_smem));
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / 2-SM TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr_smem;
  // PDL: everything above (barrier init, TMEM allocation, tensor-map prefetch) may overlap
  // the previous grid's tail; global memory is touched only after this
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();

  if (warp < 4) {
    setmaxnreg_dec<REGS_SMALL>();
    if (warp == 0) {
      // =========================== TMA producer (both CTAs) + CLC (leader) =================
      if (lane == 0) {
        const uint64_t pol_kv = policy_evict_last();
        int unit = blockIdx.x >> 1;
        int it = 0;
        for (int k = 0;; ++k) {
          const int sl = k & 1;
          mbar_arrive_expect_tx(bar_sched_full(sl), 16);
          if (leader) {
            if (k >= 2) mbar_wait(bar_sched_empty(sl), ((k >> 1) - 1) & 1);
            clc_try_cancel_multicast(sSched + 16 * sl, bar_sched_full(sl));
          }
          const Unit2 U = decode_unit2(unit, p);
          const int nmax = max(U.n0, U.n1);
          // (Q tiles are loaded per slot: leader half by the slot's issuer, peer half by the
          // peer's warp 1+t, each as soon as the slot's previous tile no longer reads it)
          // ring order = MMA consumption order: K_0, K_1, V_0, K_2, V_1, ..., V_{nmax-1}
          for (int q = 0; q < 2 * nmax; ++q, ++it) {
            const bool is_k = (q == 0) || ((q & 1) && q != 2 * nmax - 1);
            const int j = (q == 0) ? 0 : (is_k ? (q + 1) >> 1 : (q == 2 * nmax - 1 ? nmax - 1 : (q - 2) >> 1));
            const int slot = it % C::NST;
            const int use = it / C::NST;
            if (use > 0) mbar_wait(bar_kv_empty(slot), (use - 1) & 1);
            if (leader) mbar_arrive_expect_tx(bar_kv_full(slot), 2 * C::SLOT_BYTES);
            const uint32_t lead_full = mapa_shared(bar_kv_full(slot), 0);
            const uint32_t dst = sKV + slot * C::SLOT_BYTES;
            if (is_k) {  // keys [j*128 + 64*rank, +64), all D (two 64-row x 64-elem boxes)
#pragma unroll
              for (int c = 0; c < D / 64; ++c)
                tma_load_4d_2sm(dst + c * C::K_HALF_CHUNK, &p.tm_k, lead_full, c * 64, U.hkv,
                                j * BN + 64 * (int)rank, U.b, pol_kv);
            } else {     // keys [j*128, +128), D-columns [64*rank, +64)
              tma_load_4d_2sm(dst, &p.tm_v, lead_full, 64 * (int)rank, U.hkv, j * BN, U.b, pol_kv);
            }
          }
          mbar_wait(bar_sched_full(sl), (k >> 1) & 1);
          const int nxt = clc_query(sSched + 16 * sl);
          if (!leader) mbar_arrive_cluster(mapa_shared(bar_sched_empty(sl), 0));
          if (nxt < 0) break;
          unit = nxt >> 1;
        }
      }
      __syncwarp();
    } else if ((warp == 1 || warp == 2) && leader) {
      // =========== MMA issuers (leader only): warp 1 -> tile 0, warp 2 -> tile 1 ===========
      // whole warp: uniform control flow, tcgen05 ops by one elected lane (elect_one():
      // descriptors stay in uniform registers, no per-MMA R2UR waterfall)
      const int t = warp - 1;
      {
        constexpr uint32_t FMT = BF16 ? 1u : 0u;
        // S = Q K^T over the pair: M=256 (rows split), N=128 keys (B split 64/64)
        const uint32_t IDESC_QK = make_idesc_f16(FMT, 2 * BM, BN, 0, 0, p.neg ? 1u : 0u);
        // O += P V: M=256, N=D=128 (V's D-columns split 64/64), V MN-major
        constexpr uint32_t IDESC_PV = make_idesc_f16(FMT, 2 * BM, D, 0, 1, 0);
        const uint32_t tm_s = tmem_base + t * BN;
        const uint32_t tm_o = tmem_base + C::TMEM_O + t * D;
        const uint32_t qa = sQ + t * C::Q_TILE_BYTES;
        const uint32_t pa = sP + t * C::P_TILE_BYTES;
        int unit = blockIdx.x >> 1;
        int it = 0;
        int p0 = 0, p1 = 0;
        uint32_t cs = 0, cpv = 0, cq = 0;
        for (int k = 0;; ++k) {
          const Unit2 U = decode_unit2(unit, p);
          const SlotAsg A = slot_assign(U, t, p0, p1);
          const int nmax = max(U.n0, U.n1);
          const int nt = A.n;
          if (lane == 0) TL_TRACE2(k, 6000 + 100 * t + 2);  // unit decoded
          const int it0 = it;
          it += 2 * nmax;
          auto kpos = [&](int j) { return it0 + (j == 0 ? 0 : 2 * j - 1); };
          auto vpos = [&](int j) { return it0 + (j == nmax - 1 ? 2 * nmax - 1 : 2 * j + 2); };
          if (nt > 0) mbar_wait(bar_q_full(t), cq & 1);  // Q_t (loaded by the peer's warp 1+t)
          if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * 15 + 7);  // Q ready (unit start)
          auto issue_s = [&](int j) {
            const int sl = kpos(j) % C::NST;
            if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * (j & 15) + 0);
            mbar_wait(bar_kv_full(sl), (kpos(j) / C::NST) & 1);
            if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * (j & 15) + 1);
#ifndef TLATTN_MMA_ONLY
            if (cs > 0) mbar_wait(bar_s_free(t), (cs - 1) & 1);  // both CTAs read S_t
#endif
            if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * (j & 15) + 2);
            tc_fence_after();
            const uint32_t kb = sKV + sl * C::SLOT_BYTES;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              if (elect_one()) mma_f16_ss_2sm(tm_s,
                             make_sdesc_sw128(qa + (kk >> 2) * CHUNK_BYTES + (kk & 3) * 32, 16, 1024),
                             make_sdesc_sw128(kb + (kk >> 2) * C::K_HALF_CHUNK + (kk & 3) * 32, 16, 1024),
                             IDESC_QK, kk > 0 ? 1u : 0u);
            }
            if (elect_one()) mma_commit_2sm(bar_s_full(t));
            if (elect_one()) mma_commit_2sm(bar_kv_empty(sl));
            if (j >= A.n_oth && elect_one()) mma_commit_2sm(bar_kv_empty(sl));  // this slot's alone
            if (lane == 0 && j < 15) TL_TRACE2(k, 4000 + 1000 * t + 8 * j + 6);  // S(j) issued (after commit)
            ++cs;
          };
          auto issue_pv = [&](int j) {
            const int sl = vpos(j) % C::NST;
            if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * (j & 15) + 3);
            mbar_wait(bar_kv_full(sl), (vpos(j) / C::NST) & 1);
            if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * (j & 15) + 4);
#ifndef TLATTN_MMA_ONLY
            mbar_wait(bar_p_full(t), cpv & 1);  // P_t written in both CTAs
#endif
            if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * (j & 15) + 5);
            tc_fence_after();
            const uint32_t vb = sKV + sl * C::SLOT_BYTES;
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
#ifndef TLATTN_MMA_ONLY
              if (P_SPLIT && kk > 0 && kk % (8 / NPIECE) == 0) {  // next piece of P_t written (both CTAs)
                mbar_wait(bar_p_piece(t, kk / (8 / NPIECE)), (cpv & 1));
                tc_fence_after();
              }
#endif
              if (elect_one()) mma_f16_ss_2sm(tm_o,
                             make_sdesc_sw128(pa + (kk >> 2) * CHUNK_BYTES + (kk & 3) * 32, 16, 1024),
                             make_sdesc_sw128(vb + kk * 2048, CHUNK_BYTES, 1024), IDESC_PV,
                             (j > 0 || kk > 0) ? 1u : 0u);
            }
            if (elect_one()) mma_commit_2sm(bar_o_done(t));
            if (elect_one()) mma_commit_2sm(bar_kv_empty(sl));
            if (j >= A.n_oth && elect_one()) mma_commit_2sm(bar_kv_empty(sl));  // this slot's alone
            if (lane == 0 && j < 15) TL_TRACE2(k, 4000 + 1000 * t + 8 * j + 7);  // PV(j) issued (after commit)
            ++cpv;
          };
          if (nt > 0) {
            issue_s(0);
            if (nt == 1 && elect_one()) mma_commit_2sm(bar_q_empty(t));
            for (int j = 0; j < nt; ++j) {
              if (j + 1 < nt) {
                issue_s(j + 1);
                if (j + 2 == nt && elect_one()) mma_commit_2sm(bar_q_empty(t));
              }
              issue_pv(j);
            }
            ++cq;
          }
          // blocks j >= nt belong to the other slot; it releases them alone unless the other
          // tile is much longer (n_skip > nt): then this slot walks them in step
          for (int j = nt; j < A.n_skip; ++j) {
            int sl = kpos(j) % C::NST;
            mbar_wait(bar_kv_full(sl), (kpos(j) / C::NST) & 1);
            if (elect_one()) mma_commit_2sm(bar_kv_empty(sl));
            sl = vpos(j) % C::NST;
            mbar_wait(bar_kv_full(sl), (vpos(j) / C::NST) & 1);
            if (elect_one()) mma_commit_2sm(bar_kv_empty(sl));
          }
          if (lane == 0) TL_TRACE2(k, 4000 + 1000 * t + 8 * 15 + 6);  // issuer done with the unit's MMAs
          mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
          if (lane == 0) TL_TRACE2(k, 6000 + 100 * t + 0);  // next unit's CLC response seen
          const int nxt = clc_query(sSched + 16 * (k & 1));
          if (elect_one()) mbar_arrive(bar_sched_empty(k & 1));
          if (lane == 0) TL_TRACE2(k, 6000 + 100 * t + 1);
          if (nxt < 0) break;
          unit = nxt >> 1;
        }
      }
      __syncwarp();
    } else if ((warp == 1 || warp == 2) && !leader) {
      // ===== Q loaders (peer warps 1, 2: slot t = warp - 1): both halves of each of the
      // slot's Q tiles, issued as soon as the slot's previous tile's last QK^T has completed
      // (q_empty, multicast commit: the peer's own copy): the peer's rows with a 2-SM load,
      // the leader's rows multicast into the leader's smem; the expected bytes are posted on
      // the leader's q_full by a remote arrive. The leader's issuer only waits q_full. =====
      const int t = warp - 1;
      if (lane == 0) {
        const uint64_t pol_q = policy_evict_first();
        const uint32_t lead_q_full = mapa_shared(bar_q_full(t), 0);
        int unit = blockIdx.x >> 1;
        int p0 = 0, p1 = 0;
        uint32_t cq = 0;
        for (int k = 0;; ++k) {
          const Unit2 U = decode_unit2(unit, p);
          const SlotAsg A = slot_assign(U, t, p0, p1);
          if (A.n > 0) {
            if (cq > 0) mbar_wait(bar_q_empty(t), (cq - 1) & 1);
            const int r = U.r0 + 256 * A.tau;
            const bool two = r + 128 < p.Sq;
            mbar_arrive_expect_tx_cluster(lead_q_full, (two ? 2 : 1) * C::Q_TILE_BYTES);
#pragma unroll
            for (int c = 0; c < D / 64; ++c)  // leader's rows [r, r + 128)
              tma_load_4d_mc(sQ + t * C::Q_TILE_BYTES + c * CHUNK_BYTES, &p.tm_q, bar_q_full(t),
                             c * 64, U.h, r, U.b, (uint16_t)1, pol_q);
            if (two) {
#pragma unroll
              for (int c = 0; c < D / 64; ++c)  // own rows [r + 128, r + 256)
                tma_load_4d_2sm(sQ + t * C::Q_TILE_BYTES + c * CHUNK_BYTES, &p.tm_q, lead_q_full,
                                c * 64, U.h, r + 128, U.b, pol_q);
            }
            ++cq;
          }
          mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
          const int nxt = clc_query(sSched + 16 * (k & 1));
          mbar_arrive_cluster(mapa_shared(bar_sched_empty(k & 1), 0));
          if (nxt < 0) break;
          unit = nxt >> 1;
        }
      }
      __syncwarp();
    }
  } else {
    setmaxnreg_inc<REGS_SOFTMAX>();
    // ============== softmax / correction / epilogue (both CTAs, own 128 rows) ==============
    const int t = (warp - SOFTMAX_WARP0) >> 2;
    const int q4 = warp & 3;
    const int lr = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tm_s = tmem_base + lane_off + t * BN;
    const uint32_t tm_o = tmem_base + lane_off + C::TMEM_O + t * D;
    const uint32_t p_row = sP + t * C::P_TILE_BYTES + lr * 128;
    const uint32_t lead_s_free = mapa_shared(bar_s_free(t), 0);
    const uint32_t lead_p_full = mapa_shared(bar_p_full(t), 0);
    uint32_t lead_p_piece[NPIECE];
#pragma unroll
    for (int i = 0; i < NPIECE; ++i) lead_p_piece[i] = mapa_shared(bar_p_piece(t, i), 0);
    const float c = p.c_log2;
    int unit = blockIdx.x >> 1;
    uint32_t g = 0;
    int p0 = 0, p1 = 0;
    for (int k = 0;; ++k) {
      const Unit2 U = decode_unit2(unit, p);
      const SlotAsg A = slot_assign(U, t, p0, p1);
#ifdef TLATTN_MMA_ONLY
      const int nt = 0;
#else
      const int nt = A.n;
#endif
      if (A.tau < 0) {  // short-sequence mode: the unit's one tile runs in the other slot
        mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
        const int nxt = clc_query(sSched + 16 * (k & 1));
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(bar_sched_empty(k & 1), 0));
        if (nxt < 0) break;
        unit = nxt >> 1;
        continue;
      }
      const int row = U.r0 + 256 * A.tau + 128 * (int)rank + lr;
      const int limit = p.causal ? min(p.Skv - 1, row + p.Skv - p.Sq) : (p.Skv - 1);
      float m = -INFINITY;
      float l = 0.f;
      for (int j = 0; j < nt; ++j, ++g) {
        mbar_wait(bar_s_full(t), g & 1);
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 0);
        if (j == 0 && k < 4 && t == 0 && lane == 0 && q4 == 0) TL_SPAN(1 + 3 * k);
        tc_fence_after();
        uint32_t sr[BN];
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc)
          tmem_ld32(tm_s + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + cc * 32));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(lead_s_free);
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 1);
        float m_new, alpha, sum;
        if constexpr (P_SPLIT) {
          float* sf = reinterpret_cast<float*>(sr);
          float m_use;
          row_max_update(sf, j * BN, limit, c, m, m_new, alpha, m_use);
          uint64_t acc[4];
#pragma unroll
          for (int a4 = 0; a4 < 4; ++a4) acc[a4] = f2pack(0.f, 0.f);
          constexpr int NC = BN / NPIECE;
          uint32_t pk[NC / 2];
          exp_cols<BF16, 0, NC, 0>(sf, c, m_use, pk, acc);
          if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 2);
          if (j > 0) {
            mbar_wait(bar_o_done(t), (g - 1) & 1);
            if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 3);
            tc_fence_after();
            if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
              for (int cc = 0; cc < D / 32; ++cc) {
                uint32_t ov[32];
                tmem_ld32(tm_o + cc * 32, ov);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
                tmem_st32(tm_o + cc * 32, ov);
              }
              tmem_st_wait();
            }
          }
          if (j == 0 && g > 0) {
            if (lr == 0) tma_store_wait_read<0>();
            named_bar_sync(1 + t, 128);
          }
          auto store_piece = [&](int i) {  // P row keys [i*NC, +NC) -> K-major SW128 smem
#pragma unroll
            for (int v = 0; v < NC / 8; ++v) {
              const int uu = ((i * NC) % 64) / 8 + v;  // 16-B unit within the 64-key chunk
              const uint32_t addr = p_row + ((i * NC) / 64) * CHUNK_BYTES + ((uu ^ (lr & 7)) << 4);
              st_shared_v4(addr, pk[v * 4], pk[v * 4 + 1], pk[v * 4 + 2], pk[v * 4 + 3]);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(lead_p_piece[i]);
          };
          store_piece(0);
          exp_cols<BF16, NC, NC, 0>(sf, c, m_use, pk, acc);
          store_piece(1);
          if constexpr (NPIECE == 4) {
            exp_cols<BF16, 2 * NC, NC, 0>(sf, c, m_use, pk, acc);
            store_piece(2);
            exp_cols<BF16, 3 * NC, NC, 0>(sf, c, m_use, pk, acc);
            store_piece(3);
          }
          if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 4);
          const uint64_t t0 = fadd2(acc[0], acc[1]);
          const uint64_t t1 = fadd2(acc[2], acc[3]);
          float a0, a1, b0, b1;
          f2unpack(t0, a0, a1);
          f2unpack(t1, b0, b1);
          sum = (a0 + b0) + (a1 + b1);
        } else {
        uint32_t pk[BN / 2];
        softmax_row_block<BF16, TLATTN_EMU_2SM>(sr, j * BN, limit, c, m, m_new, alpha, sum, pk);
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 2);
        if (j > 0) {
          mbar_wait(bar_o_done(t), (g - 1) & 1);
          if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 3);
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
            for (int cc = 0; cc < D / 32; ++cc) {
              uint32_t ov[32];
              tmem_ld32(tm_o + cc * 32, ov);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
              tmem_st32(tm_o + cc * 32, ov);
            }
            tmem_st_wait();
          }
        }
        if (j == 0 && g > 0) {
          // P_t smem held the previous unit's O tile for its TMA store: wait until the
          // bulk store has read it (one issuing thread), then release the warpgroup
          if (lr == 0) tma_store_wait_read<0>();
          named_bar_sync(1 + t, 128);
        }
#pragma unroll
        for (int ch = 0; ch < BN / 64; ++ch) {
#pragma unroll
          for (int uu = 0; uu < 8; ++uu) {
            const uint32_t addr = p_row + ch * CHUNK_BYTES + ((uu ^ (lr & 7)) << 4);
            const int w = ch * 32 + uu * 4;
            st_shared_v4(addr, pk[w], pk[w + 1], pk[w + 2], pk[w + 3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(lead_p_full);
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * j + 4);
        }
        l = l * alpha + sum;
        m = m_new;
      }
      if (nt > 0) {
        mbar_wait(bar_o_done(t), (g - 1) & 1);
        tc_fence_after();
      }
      if (lane == 0 && q4 == 0) TL_TRACE2(k, 6500 + 100 * t + 0);  // epilogue start (last PV done)
      const float inv_l = (l > 0.f) ? (1.f / l) : 0.f;
      const bool row_ok = row < p.Sq;
      if (nt == 0) {  // no PV this unit: P_t may still feed the previous unit's O store
        if (lr == 0) tma_store_wait_read<0>();
        named_bar_sync(1 + t, 128);
      }
      // O tile -> P_t smem (free: the unit's last PV is done) in the TMA SWIZZLE_128B box
      // layout, then one thread stores it with two bulk-tensor stores (coalesced; rows
      // beyond Sq are clipped by the tensor map)
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t ov[32];
        if (nt > 0) {
          tmem_ld32(tm_o + cc * 32, ov);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = 0u;
        }
        uint32_t pkd[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pkd[e] = pack2<BF16>(__uint_as_float(ov[2 * e]) * inv_l, __uint_as_float(ov[2 * e + 1]) * inv_l);
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          const int uu = (cc & 1) * 4 + v4;  // 16-B unit within the 128-B row of chunk cc/2
          const uint32_t addr = p_row + (cc >> 1) * CHUNK_BYTES + ((uu ^ (lr & 7)) << 4);
          st_shared_v4(addr, pkd[4 * v4], pkd[4 * v4 + 1], pkd[4 * v4 + 2], pkd[4 * v4 + 3]);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + t, 128);
      if (lane == 0 && q4 == 0) TL_TRACE2(k, 6500 + 100 * t + 1);  // O tile staged
      if (lr == 0) {
        const int row0 = U.r0 + 256 * A.tau + 128 * (int)rank;
        if (row0 < p.Sq) {
#pragma unroll
          for (int c2 = 0; c2 < D / 64; ++c2) {
            const uint32_t src = sP + t * C::P_TILE_BYTES + c2 * CHUNK_BYTES;
            if constexpr (PT::kRepl) {
              // replicated output: the same staged tile to every rank's full O (N2)
              for (int r = 0; r < p.n_out; ++r)
                tma_store_4d(&p.tm_out[r], src, c2 * 64, U.h + p.h_off, row0, U.b + p.b_off);
            } else {
              tma_store_4d(&p.tm_o, src, c2 * 64, U.h, row0, U.b);
            }
          }
        }
        tma_store_commit();
        if (k < 4 && t == 0) TL_SPAN(2 + 3 * k);
      }
      if (row_ok)
        store_lse(p, U.b, U.h, row, (l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY);
      tc_fence_before();
      if (lane == 0 && q4 == 0) TL_TRACE2(k, 6500 + 100 * t + 2);  // LSE stored
      mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
      const int nxt = clc_query(sSched + 16 * (k & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(bar_sched_empty(k & 1), 0));
      if (lane == 0 && q4 == 0) TL_TRACE2(k, 6500 + 100 * t + 3);  // next unit known
      if (nxt < 0) break;
      unit = nxt >> 1;
    }
  }

  if (warp >= SOFTMAX_WARP0 && ((warp - SOFTMAX_WARP0) & 3) == 0 && lane == 0)
    tma_store_wait_all<0>();  // O stores complete before the CTA's smem goes away
  if (warp == SOFTMAX_WARP0 && lane == 0) TL_SPAN(15);
  tc_fence_before();
  cluster_sync();  // both CTAs finished with TMEM / smem of the pair
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tlattn
