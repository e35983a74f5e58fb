// attn_fwd_sm100.cuh — fused attention forward for B200 (sm_100a).
//
// What it computes: see include/tlattn.h (§5.2; Fig. 18).
// How (B200-native re-design of the Fig. 18 schedule):
//
//   CTA = one "unit" = 2 query tiles of BM=128 rows of one (b, h)   [Fig. 18 tiles
//         Q_shared / acc_s / acc_o; here M=128 per tcgen05 tile]
//   warp 0        TMA producer: Q tiles once (T.copy Q), then K_j, V_j into an
//                 NST-slot mbarrier ring (T.Pipelined num_stages)
//   warps 1, 2    MMA issuers (one thread each, one per query tile t): S_t = Q_t K_j^T
//                 (T.gemm transpose_B) and O_t += P_t V_j (T.gemm) with
//                 tcgen05.mma, accumulators in TMEM; tcgen05.commit -> mbarriers
//   warps 4-7     softmax for tile 0, warps 8-11 softmax for tile 1: tcgen05.ld of the
//                 S row (one thread owns one row: TMEM lane = row), mask, running max,
//                 exp2, row sum, O rescale in TMEM, P -> smem
//                 (128B-swizzled, RN to dtype), epilogue O/l and LSE
//
// Row reductions (max, sum) are IN-THREAD, not warp shuffles: tcgen05.ld 32x32b gives each
// thread one whole TMEM lane = one S row, so there is nothing to shuffle. The shuffle-free
// alternative on this layout — two or four threads per row with a cross-warp exchange
// through SMEM — was measured at D = 128 on B200 (round 2, profiles/r02_kernel_notes.md):
// in isolation its exp/max/sum work is ~10 % cheaper (two warps per SM sub-partition feed
// MUFU), but in the kernel every schedule built around it was slower (T0 1233 / 1042 / 1010
// TFLOP/s vs 1421-1430 one-thread-per-row: lock-step warps expose the TMEM-load, barrier
// and proxy-fence latencies, and 16 softmax warps leave 96 registers per thread); at D = 64
// a 640-thread split-row variant measured C4 657 vs 664 (round 1).
//
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D, 256+2D)
// SMEM: Q0,Q1 (2 x 128 x D x 2B) | KV ring NST x (128 x D x 2B) | P0,P1 (2 x 32 KB) | mbarriers
// All operand tiles are TMA SWIZZLE_128B boxes of 128 rows x 64 elements (16 KB).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "ptx.cuh"

namespace tlattn {

constexpr int BM = 128;            // query rows per tile (tcgen05 M)
constexpr int BN = 128;            // keys per K/V block (tcgen05 N of QK^T, K of PV)
constexpr int TILES = 2;           // query tiles per CTA unit
constexpr int NUM_THREADS = 384;   // 12 warps
constexpr int SOFTMAX_WARP0 = 4;   // warps 4..11
constexpr int CHUNK_BYTES = 128 * 128;  // one 128-row x 64-element 16-bit SW128 box
constexpr uint32_t TMEM_COLS = 512;

// Division by a runtime constant without the MUFU.RCP of the generic integer divide (the
// softmax warps keep MUFU saturated, so a unit decode with five divides cost ~1200 clocks
// in the MMA issuer's unit transition, profiles/r01_trace_notes.md): for 0 <= n < 2^31,
// n / d = (umulhi(n, mul) + n) >> shr with shr = ceil(log2 d) and
// mul = floor(2^32 (2^shr - d) / d) + 1 (host-computed, make_fastdiv).
struct FastDiv {
  uint32_t d, mul, shr;
  __device__ __forceinline__ int div(int n) const {
    return static_cast<int>((__umulhi(static_cast<uint32_t>(n), mul) + static_cast<uint32_t>(n)) >> shr);
  }
  __device__ __forceinline__ int mod(int n) const { return n - div(n) * static_cast<int>(d); }
};

struct AttnParams {
  CUtensorMap tm_q;  // BSHD as 4-D (D, Hq, Sq, B), box (64, 1, 128, 1), SWIZZLE_128B
  CUtensorMap tm_k;  // (D, Hkv, Skv, B)
  CUtensorMap tm_v;
  CUtensorMap tm_o;  // output, same geometry as tm_q (TMA-store epilogue)
  void* o;           // BSHD output
  float* lse;        // [B][Hq][Sq] or nullptr
  int B, Hq, Hkv, Sq, Skv;
  int causal;
  float c_log2;      // |scale| * log2(e)
  int neg;           // scale < 0: negate A (= Q) in the QK^T instruction descriptor
  int n_mblk;        // ceil(Sq / unit rows)
  int n_units;       // B * Hq * n_mblk
  int unit_tiles;    // CTA-pair kernel: query tiles (of 256 rows) per unit, 2 or 1 (short Sq)
  FastDiv fd_mblk, fd_nbh, fd_hq, fd_grp;  // / n_mblk, / (B Hq), / Hq, / (Hq / Hkv)
  int lpt;           // unit order: 0 = (b, h)-major (K/V of a head stay in L2), 1 = query-
                     // block-major, heaviest first over ALL heads (causal, K/V fit in L2)
  unsigned long long* trace;  // debug builds (TLATTN_TRACE) only: event clocks of CTA 0
  static constexpr bool kRepl = false;
};

// Replicated output (tl_attn_fwd_replicated): the epilogue writes each O
// tile (and LSE row) of this rank's shard straight into the full [B_total][Sq][Hq_total][D]
// output of every rank (peer buffers mapped into this process), at batch / head offsets
// b_off / h_off. The all-gather of O becomes part of the kernel's store stream.
constexpr int kMaxOuts = 8;
struct AttnParamsRepl : AttnParams {
  CUtensorMap tm_out[kMaxOuts];  // full outputs, (D, Hq_total, Sq, B_total), box (64, 1, 128, 1)
  void* o_out[kMaxOuts];         // the same buffers as raw pointers (row-store epilogue)
  float* lse_out[kMaxOuts];      // full LSE [B_total][Hq_total][Sq] per output, or all NULL
  int n_out, b_off, h_off, Hq_total;
  static constexpr bool kRepl = true;
};

// Row-store epilogue helper: O row (16-byte pieces) and LSE of one query row to the
// output(s); `pieces` are 16-B chunks at byte offset `off` within the D-row.
template <class PT>
__device__ __forceinline__ uint8_t* out_row(const PT& p, int r, int b, int h, int row, int D) {
  if constexpr (PT::kRepl) {
    return reinterpret_cast<uint8_t*>(p.o_out[r]) +
           ((((size_t)(b + p.b_off) * p.Sq + row) * p.Hq_total + (h + p.h_off)) * D) * 2;
  } else {
    return reinterpret_cast<uint8_t*>(p.o) + ((((size_t)b * p.Sq + row) * p.Hq + h) * D) * 2;
  }
}
template <class PT>
__device__ __forceinline__ void store_lse(const PT& p, int b, int h, int row, float v) {
  if constexpr (PT::kRepl) {
    for (int r = 0; r < p.n_out; ++r)
      if (p.lse_out[r] != nullptr)
        p.lse_out[r][((size_t)(b + p.b_off) * p.Hq_total + (h + p.h_off)) * p.Sq + row] = v;
  } else {
    if (p.lse != nullptr) p.lse[((size_t)b * p.Hq + h) * p.Sq + row] = v;
  }
}
template <class PT>
__device__ __forceinline__ int n_outputs(const PT& p) {
  if constexpr (PT::kRepl) return p.n_out;
  else return 1;
}

// Debug-only pipeline trace (compile with -DTLATTN_TRACE): clock64 stamps of the first
// unit of CTA 0 (the pair leader), used to inspect the MMA / softmax overlap.
#ifdef TLATTN_TRACE
#define TL_TRACE(k, idx)                                                          \
  do {                                                                            \
    if (p.trace != nullptr && blockIdx.x == 0 && (k) == 0) p.trace[(idx)] = clock64(); \
  } while (0)
#define TL_TRACE2(k, idx)                                                                \
  do {                                                                                   \
    if (p.trace != nullptr && blockIdx.x < 2 && (k) < 4)                                 \
      p.trace[(idx) + 200 * (k) + 8000 * blockIdx.x] = clock64();                        \
  } while (0)
// per-CTA globaltimer spans (all CTAs): slot 0 kernel entry, 1 + 3k / 2 + 3k first S /
// O store issued of unit k < 4 (tile 0), 15 kernel end
#define TL_SPAN(idx)                                                                     \
  do {                                                                                   \
    if (p.trace != nullptr) p.trace[16000 + 16 * blockIdx.x + (idx)] = globaltimer();    \
  } while (0)
// second per-CTA area (producer events of the first unit)
#define TL_SPAN2(idx)                                                                      \
  do {                                                                                     \
    if (p.trace != nullptr) p.trace[16000 + 16 * 160 + 16 * blockIdx.x + (idx)] = globaltimer(); \
  } while (0)
#else
#define TL_SPAN2(idx) \
  do {                \
  } while (0)
#define TL_SPAN(idx) \
  do {               \
  } while (0)
#define TL_TRACE2(k, idx) \
  do {                    \
  } while (0)
#define TL_TRACE(k, idx) \
  do {                   \
  } while (0)
#endif

template <int D>
struct KCfg {
  static constexpr int Q_TILE_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  // D = 64: P lives in TMEM (columns 384..511, after S0 S1 O0 O1) and PV reads it as the
  // TMEM A operand ("TS" MMA), so no P in SMEM and a deeper K/V ring.
#ifndef TLATTN_P_SMEM64  // A/B experiments: keep P in SMEM at D = 64
  static constexpr bool P_TMEM = (D == 64);
#else
  static constexpr bool P_TMEM = false;
#endif
#ifdef TLATTN_NST_OVERRIDE  // experiments only (P smem dropped)
  static constexpr int NST = TLATTN_NST_OVERRIDE;
  static constexpr int P_TILE_BYTES = 0;
#else
#ifndef TLATTN_NST64
#define TLATTN_NST64 10
#endif
  static constexpr int NST = (D == 128) ? 3 : (P_TMEM ? TLATTN_NST64 : 6);
  static constexpr int P_TILE_BYTES = P_TMEM ? 0 : BM * BN * 2;
#endif
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + TILES * Q_TILE_BYTES;
  static constexpr int OFF_P = OFF_KV + NST * KV_BYTES;
  static constexpr int OFF_SCHED = OFF_P + TILES * P_TILE_BYTES;  // 2 x 16-B CLC responses
  static constexpr int OFF_BAR = OFF_SCHED + 32;
  // barriers: q_full, q_empty, kv_full[NST], kv_empty[NST], s_full[2], s_free[2], p_full[2],
  //           o_done[2], sched_full[2], sched_empty[2]
  static constexpr int NUM_BARS = 2 + 2 * NST + 12;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_USED = OFF_TMEMPTR + 16;
  static constexpr int SMEM_BYTES = SMEM_USED + 1024;  // slack for 1024-B alignment
  static_assert(SMEM_BYTES <= 232448, "shared memory budget exceeded");
  static constexpr uint32_t TMEM_O = 2 * BN;  // O0 column base
  static constexpr uint32_t TMEM_P = 2 * BN + 2 * D;  // P0 column base (P_TMEM): BN/2 columns per tile
};

template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  if constexpr (BF16) {
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  } else {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  }
  return r;
}

// Number of K/V blocks tile starting at row r0 must visit (causal tile skipping).
__device__ __forceinline__ int tile_nblocks(int r0, const AttnParams& p) {
  if (r0 >= p.Sq) return 0;
  const int n_all = (p.Skv + BN - 1) / BN;
  if (!p.causal) return n_all;
  const int r_last = min(r0 + BM - 1, p.Sq - 1);
  const long long kmax = (long long)r_last + p.Skv - p.Sq;  // last key the last row may see
  if (kmax < 0) return 0;
  return min(n_all, (int)(kmax / BN) + 1);
}


// Rescale O only when a row max grows by more than 2^RESCALE_LOG2:
// otherwise keep the stale max, so p = exp2(c s - m) <= 2^8 stays well inside fp16/bf16
// range and the result is unchanged up to rounding (O and l use the same m).
constexpr float RESCALE_LOG2 = 8.0f;
// The CTA is launched with 168 x 384 = 64512 registers (__launch_bounds__(384, 1)); the
// split must fit that pool (216 for the softmax warpgroups would need 65536 and blocks
// setmaxnreg.inc forever — measured: the watchdog traps).
#ifndef TLATTN_REGS_SMALL  // experiments may override the split (must fit 64512)
#define TLATTN_REGS_SMALL 88
#define TLATTN_REGS_SOFTMAX 208
#endif
constexpr uint32_t REGS_SMALL = TLATTN_REGS_SMALL;      // warpgroup 0: 128 x 88
constexpr uint32_t REGS_SOFTMAX = TLATTN_REGS_SOFTMAX;  // warpgroups 1-2: 256 x 208 (total 64512)
static_assert(128 * REGS_SMALL + 256 * REGS_SOFTMAX <= 64512, "register split exceeds the launch pool");

// exp2 on the FMA pipe for a pair of values: round-to-nearest
// range reduction with the 1.5*2^23 magic add, 2^f on f in [-0.5, 0.5] by a degree-3
// polynomial with p(0) = 1 (max relative error 1.0e-4, fitted in tools/fit_exp2_poly.py),
// and the integer part added to the exponent field with one integer multiply-add.
// Inputs are clamped to >= -125 so the exponent never underflows (2^-125 contributes
// nothing visible next to the row max's p >= 1).
struct Exp2Poly {
  uint64_t magic, neg_magic, neg_one, c3, c2, c1, one;
  __device__ __forceinline__ Exp2Poly()
      : magic(f2pack(12582912.f, 12582912.f)),
        neg_magic(f2pack(-12582912.f, -12582912.f)),
        neg_one(f2pack(-1.f, -1.f)),
        c3(f2pack(0.055008258670568466f, 0.055008258670568466f)),
        c2(f2pack(0.24220958352088928f, 0.24220958352088928f)),
        c1(f2pack(0.6932828426361084f, 0.6932828426361084f)),
        one(f2pack(1.f, 1.f)) {}
  __device__ __forceinline__ void operator()(uint64_t x2, float& y0, float& y1) const {
    float x0, x1;
    f2unpack(x2, x0, x1);
    x2 = f2pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
    const uint64_t t = fadd2(x2, magic);          // RN(x) in the low mantissa bits
    const uint64_t f = ffma2(fadd2(t, neg_magic), neg_one, x2);  // x - RN(x) in [-0.5, 0.5]
    const uint64_t pp = ffma2(ffma2(ffma2(c3, f, c2), f, c1), f, one);
    float t0, t1, p0, p1;
    f2unpack(t, t0, t1);
    f2unpack(pp, p0, p1);
    // 2^RN(x) * p: add RN(x) to the exponent field (t's low bits hold RN(x) mod 2^9)
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
  }
};

// Column pairs (of 64 per row) whose exp2 runs on the FMA pipe instead of MUFU: EMU of
// every 8. Measured on B200: D=64 gains from EMU=2 (the softmax
// bounds that shape; TLATTN_EMU64), D=128 is fastest with EMU=0 (the extra issue slots cost more than
// the MUFU time saved).
// TLATTN_EXP_VARIANT (experiments only): 0 = per-kernel EMU, 1 = none, 2 = all,
// 3 = no exp at all (timing of everything else; WRONG results).
#ifndef TLATTN_EXP_VARIANT
#define TLATTN_EXP_VARIANT 0
#endif
#ifdef TLATTN_EMU_OVERRIDE  // experiments only
#define TLATTN_EMU_2SM TLATTN_EMU_OVERRIDE
#else
#define TLATTN_EMU_2SM 0
#endif
// exp2 offload of the D = 64 kernel: EMU of every 8 column pairs on the FMA pipe. Measured
// with P in TMEM and the LPT order (B200, same box): EMU 1/2/3 -> C4 779 / 811 / 763,
// D=64 non-causal 760 / 805 / 740 TFLOP/s, so 2.
#ifndef TLATTN_EMU64
#define TLATTN_EMU64 2
#endif
template <int EMU>
__host__ __device__ constexpr bool emu_pair(int q) {
  return TLATTN_EXP_VARIANT == 2 ? true
       : TLATTN_EXP_VARIANT == 1 ? false
       : EMU == 3 ? ((q & 7) == 2 || (q & 7) == 5 || (q & 7) == 7)
       : EMU == 2 ? ((q & 7) == 3 || (q & 7) == 7)
       : EMU == 1 ? ((q & 7) == 7)
       : false;
}


// p = exp2(s*c - m) for one 128-column row with paired FFMA2, FADD2 row sums (two
// accumulators), P packed RN to the dtype; emu_pair<EMU>() column pairs use Exp2Poly.
template <bool BF16, int EMU>
__device__ __forceinline__ void exp_row(float* s, float c, float m_use, uint32_t (&pk)[BN / 2],
                                        float& sum0, float& sum1) {
  const uint64_t c2 = f2pack(c, c);
  const uint64_t nm2 = f2pack(-m_use, -m_use);
  // Phases, 32 columns at a time (independent work back to back so one warp keeps MUFU
  // fed): x = s*c - m (FFMA2), then p = exp2(x) (MUFU or Exp2Poly), then row sums (FADD2,
  // 4 accumulators) and RN packing.
  uint64_t acc[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) acc[a] = f2pack(0.f, 0.f);
#pragma unroll
  for (int h = 0; h < BN; h += 32) {
    float x[32];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const uint64_t x2 = ffma2(f2pack(s[h + 2 * q], s[h + 2 * q + 1]), c2, nm2);
      f2unpack(x2, x[2 * q], x[2 * q + 1]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int qq = h / 2 + q;
      if (TLATTN_EXP_VARIANT == 3) {
      } else if (emu_pair<EMU>(qq)) {
        const Exp2Poly poly;
        poly(f2pack(x[2 * q], x[2 * q + 1]), x[2 * q], x[2 * q + 1]);
      } else {
        x[2 * q] = ex2(x[2 * q]);
        x[2 * q + 1] = ex2(x[2 * q + 1]);
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      acc[q & 3] = fadd2(acc[q & 3], f2pack(x[2 * q], x[2 * q + 1]));
      pk[h / 2 + q] = pack2<BF16>(x[2 * q], x[2 * q + 1]);  // P rounded RN (R8)
    }
  }
  const uint64_t t0 = fadd2(acc[0], acc[1]);
  const uint64_t t1 = fadd2(acc[2], acc[3]);
  float a0, a1, b0, b1;
  f2unpack(t0, a0, a1);
  f2unpack(t1, b0, b1);
  sum0 = a0 + b0;
  sum1 = a1 + b1;
}

// Mask columns [C0, C0+NC) of a diagonal / tail block (k0 + col > limit -> -inf) and
// return their max (T.reduce_max: in-thread, each thread owns one whole S row).
// The 32 rows of a warp are consecutive, so their limits span at most 32 keys: a 32-column
// chunk that every lane sees whole is skipped with one warp-uniform test, and the compare
// of the other chunks is against a per-chunk bound (ISETP with an immediate + SEL per
// element). The naive form (VIADD + ISETP + SEL on all 128 columns, ALU pipe at half rate)
// measured ~900 extra SM clocks per diagonal block on C5 (profiles/r02_kernel_notes.md).
// Variants that also skipped fully masked chunks in the exp pass measured slower on every
// config (larger code on the unmasked path, or register spills: r02 notes).
template <int C0, int NC>
__device__ __forceinline__ float mask_max_cols(float* s, int k0, int limit, bool masked) {
#ifdef TLATTN_NO_MASK  // timing experiment only (WRONG results): no causal / tail mask
  masked = false;
#endif
  if (masked) {
    const int lim_lo = __shfl_sync(0xffffffffu, limit, 0);  // rows ascend with the lane
#pragma unroll
    for (int q = 0; q < NC / 32; ++q) {
      const int c0 = k0 + C0 + 32 * q;
      if (c0 + 31 > lim_lo) {       // not every lane sees the whole chunk
        const int nv = limit - c0;  // this lane sees columns e <= nv of the chunk
#pragma unroll
        for (int e = 0; e < 32; ++e) s[C0 + 32 * q + e] = e > nv ? -INFINITY : s[C0 + 32 * q + e];
      }
    }
  }
  constexpr int R = NC / 32;
  float mq[R];
#pragma unroll
  for (int r = 0; r < R; ++r) mq[r] = fmax3(s[C0 + r * 32], s[C0 + r * 32 + 1], s[C0 + r * 32 + 2]);
#pragma unroll
  for (int cc = 3; cc + 1 < 32; cc += 2)
#pragma unroll
    for (int r = 0; r < R; ++r) mq[r] = fmax3(mq[r], s[C0 + r * 32 + cc], s[C0 + r * 32 + cc + 1]);
#pragma unroll
  for (int r = 0; r < R; ++r) mq[r] = fmaxf(mq[r], s[C0 + r * 32 + 31]);
  float mx = mq[0];
#pragma unroll
  for (int r = 1; r < R; ++r) mx = fmaxf(mx, mq[r]);
  return mx;
}

// Conditional running-max update from the block's row max mx (raw score units).
__device__ __forceinline__ void row_max_finish(float mx, float c, float m, float& m_new_out,
                                               float& alpha_out, float& m_use_out) {
  const float mxs = (mx == -INFINITY) ? -INFINITY : mx * c;
  const float m_new = (mxs > m + RESCALE_LOG2) ? mxs : m;  // conditional rescale
  const float m_use = (m_new == -INFINITY) ? 0.f : m_new;  // -inf guard
  alpha_out = ex2(m - m_use);                              // scores_scale
  m_new_out = m_new;
  m_use_out = m_use;
}

// Mask (diagonal / tail blocks only), row max and the conditional running-max update of
// one K/V block. Returns whether the block was masked; m_use is the max the exps
// subtract (-inf guard).
__device__ __forceinline__ bool row_max_update(float* s, int k0, int limit, float c, float m,
                                               float& m_new_out, float& alpha_out, float& m_use_out) {
  // any column beyond this row's last key? (diagonal / tail blocks only)
  const bool masked = __any_sync(0xffffffffu, k0 + BN - 1 > limit);
  const float mx = mask_max_cols<0, BN>(s, k0, limit, masked);
  row_max_finish(mx, c, m, m_new_out, alpha_out, m_use_out);
  return masked;
}

// One K/V block of the online softmax for the row this thread owns (Fig. 18
// P:L660-679): mask, row max, conditional running-max update (row_max_update), p =
// exp2(s*c - m) with part of the exp2s on the FMA pipe, fp32 row sum of the unrounded p,
// and P packed (RN) to the input dtype. sr[] holds the raw fp32 S row.
template <bool BF16, int EMU>
__device__ __forceinline__ void softmax_row_block(uint32_t (&sr)[BN], int k0, int limit, float c,
                                                  float m, float& m_new_out, float& alpha_out,
                                                  float& sum_out, uint32_t (&pk)[BN / 2]) {
  float* s = reinterpret_cast<float*>(sr);
  float m_use;
  const bool masked = row_max_update(s, k0, limit, c, m, m_new_out, alpha_out, m_use);
  // p = exp2(s*c - m); row sum over the unrounded fp32 p (R8).
  // c > 0 always (scale = 0 arrives as a tiny positive c, host side), so a masked
  // s = -inf gives exp2(-inf) = 0 exactly and masked blocks use the same paired loop
  // (MUFU only); unmasked blocks offload emu_pair<EMU>() columns to the FMA pipe.
  float sum0, sum1;
  if (masked) exp_row<BF16, 0>(s, c, m_use, pk, sum0, sum1);  // diagonal / tail: MUFU only
  else exp_row<BF16, EMU>(s, c, m_use, pk, sum0, sum1);
  sum_out = sum0 + sum1;
}

// p = exp2(s*c - m) for columns [C0, C0+NC) of the row (MUFU, or Exp2Poly for the
// emu_pair<EMU>() column pairs), packed RN into pk[0..NC/2), fp32 row sums accumulated
// into acc (paired FADD2). The P-in-pieces softmax paths use it per piece.
template <bool BF16, int C0, int NC, int EMU>
__device__ __forceinline__ void exp_cols(const float* s, float c, float m_use, uint32_t (&pk)[NC / 2],
                                         uint64_t (&acc)[4]) {
  const uint64_t c2 = f2pack(c, c);
  const uint64_t nm2 = f2pack(-m_use, -m_use);
#pragma unroll
  for (int h = 0; h < NC; h += 32) {
    float x[32];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const uint64_t x2 = ffma2(f2pack(s[C0 + h + 2 * q], s[C0 + h + 2 * q + 1]), c2, nm2);
      f2unpack(x2, x[2 * q], x[2 * q + 1]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (emu_pair<EMU>((C0 + h) / 2 + q)) {
        const Exp2Poly poly;
        poly(f2pack(x[2 * q], x[2 * q + 1]), x[2 * q], x[2 * q + 1]);
      } else {
        x[2 * q] = ex2(x[2 * q]);
        x[2 * q + 1] = ex2(x[2 * q + 1]);
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      acc[q & 3] = fadd2(acc[q & 3], f2pack(x[2 * q], x[2 * q + 1]));
      pk[h / 2 + q] = pack2<BF16>(x[2 * q], x[2 * q + 1]);
    }
  }
}

struct Unit {
  int b, h, hkv, m_blk, n0, n1;
};

// Unit order: (b, h) major, 256-row query block minor; causal: heaviest block first.
// Units of one (b, kv-head) group are adjacent in launch (= CLC steal) order, so their
// K/V stay L2-resident (the T.use_swizzle idea).
__device__ __forceinline__ Unit decode_unit(int u, const AttnParams& p) {
  Unit U;
  const int mb_i = p.lpt ? p.fd_nbh.div(u) : p.fd_mblk.mod(u);
  const int bh = p.lpt ? p.fd_nbh.mod(u) : p.fd_mblk.div(u);
  U.b = p.fd_hq.div(bh);
  U.h = bh - U.b * p.Hq;
  U.m_blk = p.causal ? (p.n_mblk - 1 - mb_i) : mb_i;
  U.hkv = p.fd_grp.div(U.h);  // GQA grouping h / (Hq / Hkv)
  U.n0 = tile_nblocks(U.m_blk * (TILES * BM), p);
  U.n1 = tile_nblocks(U.m_blk * (TILES * BM) + BM, p);
  return U;
}

template <int D, bool BF16, class PT = AttnParams>
__global__ void __launch_bounds__(NUM_THREADS, 1)
tl_attn_fwd_kernel(const __grid_constant__ PT p) {
  using C = KCfg<D>;
  // K/V load order: K_{j+1} ahead of V_j (MMA consumption order; measured faster with the
  // D=128 3-slot ring, and +1 % at D=64 with the 10-slot ring: C4 810 -> 818 TFLOP/s).
  constexpr bool K_AHEAD = true;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base = (raw_u32 + 1023u) & ~1023u;  // 1024-B aligned (SWIZZLE_128B atoms)
  uint8_t* smem = smem_raw + (base - raw_u32);

  const uint32_t sQ = base + C::OFF_Q;
  const uint32_t sKV = base + C::OFF_KV;
  const uint32_t sP = base + C::OFF_P;
  const uint32_t sSched = base + C::OFF_SCHED;
  const uint32_t bar0 = base + C::OFF_BAR;
  const uint32_t bar_q_full = bar0;
  const uint32_t bar_q_empty = bar0 + 8u;
  auto bar_kv_full = [&](int s) { return bar0 + 8u * (2 + s); };
  auto bar_kv_empty = [&](int s) { return bar0 + 8u * (2 + C::NST + s); };
  auto bar_s_full = [&](int t) { return bar0 + 8u * (2 + 2 * C::NST + t); };
  auto bar_s_free = [&](int t) { return bar0 + 8u * (4 + 2 * C::NST + t); };
  auto bar_p_full = [&](int t) { return bar0 + 8u * (6 + 2 * C::NST + t); };
  auto bar_o_done = [&](int t) { return bar0 + 8u * (8 + 2 * C::NST + t); };
  auto bar_sched_full = [&](int i) { return bar0 + 8u * (10 + 2 * C::NST + i); };
  auto bar_sched_empty = [&](int i) { return bar0 + 8u * (12 + 2 * C::NST + i); };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- setup (once per persistent CTA)
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tm_q);
    prefetch_tmap(&p.tm_k);
    prefetch_tmap(&p.tm_v);
    mbar_init(bar_q_full, 1);
    mbar_init(bar_q_empty, 2);  // one release per MMA issuer
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(bar_kv_full(s), 1);
      mbar_init(bar_kv_empty(s), 2);  // one release per MMA issuer
    }
    for (int t = 0; t < TILES; ++t) {
      mbar_init(bar_s_full(t), 1);
      mbar_init(bar_s_free(t), 4);
      mbar_init(bar_p_full(t), 4);
      mbar_init(bar_o_done(t), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_sched_full(i), 1);
      mbar_init(bar_sched_empty(i), 2 + 8);  // 2 MMA issuers + 8 softmax warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(smem_u32(tmem_ptr_smem));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr_smem;
  griddep_wait();  // PDL (see attn_fwd_sm100_2sm.cuh)
  if (threadIdx.x == 0) griddep_launch_dependents();

  // Register rebalancing: warpgroup 0 (load / MMA / spare warps) gives registers to the
  // two softmax warpgroups, which hold a 128-column fp32 S row per thread.
  if (warp < 4) {
  setmaxnreg_dec<REGS_SMALL>();
  if (warp == 0) {
    // =========================== TMA producer + CLC scheduler ===========================
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      int unit = blockIdx.x;
      int it = 0;  // K/V ring position (K_j, V_j alternate)
      for (int k = 0;; ++k) {
        // ask for the next unit now; the answer is needed only at the end of this one
        const int sl = k & 1;
        if (k >= 2) mbar_wait(bar_sched_empty(sl), ((k >> 1) - 1) & 1);
        mbar_arrive_expect_tx(bar_sched_full(sl), 16);
        clc_try_cancel(sSched + 16 * sl, bar_sched_full(sl));

        const Unit U = decode_unit(unit, p);
        const int nmax = max(U.n0, U.n1);
        const int r00 = U.m_blk * (TILES * BM);
        if (k >= 1) mbar_wait(bar_q_empty, (k - 1) & 1);  // previous unit's QK^T done
        uint32_t qbytes = 0;
#pragma unroll
        for (int t = 0; t < TILES; ++t)
          if (r00 + t * BM < p.Sq) qbytes += C::Q_TILE_BYTES;
        mbar_arrive_expect_tx(bar_q_full, qbytes);
#pragma unroll
        for (int t = 0; t < TILES; ++t) {
          if (r00 + t * BM < p.Sq) {
#pragma unroll
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(sQ + t * C::Q_TILE_BYTES + c * CHUNK_BYTES, &p.tm_q, bar_q_full, c * 64,
                          U.h, r00 + t * BM, U.b, pol_q);
          }
        }
        // Load order = MMA consumption order: K_0, then K_{j+1} before V_j, so the next
        // QK^T's operand is never queued behind a V tile that waits for softmax(j).
        for (int q = 0; q < 2 * nmax; ++q, ++it) {
          bool is_k;
          int j;
          if (K_AHEAD) {
            is_k = (q == 0) || ((q & 1) && q != 2 * nmax - 1);
            j = (q == 0) ? 0 : (is_k ? (q + 1) >> 1 : (q == 2 * nmax - 1 ? nmax - 1 : (q - 2) >> 1));
          } else {
            is_k = (q & 1) == 0;
            j = q >> 1;
          }
          const int slot = it % C::NST;
          const int use = it / C::NST;
          if (use > 0) mbar_wait(bar_kv_empty(slot), (use - 1) & 1);
          mbar_arrive_expect_tx(bar_kv_full(slot), C::KV_BYTES);
#pragma unroll
          for (int c = 0; c < D / 64; ++c)
            tma_load_4d(sKV + slot * C::KV_BYTES + c * CHUNK_BYTES, is_k ? &p.tm_k : &p.tm_v,
                        bar_kv_full(slot), c * 64, U.hkv, j * BN, U.b, pol_kv);
        }
        mbar_wait(bar_sched_full(sl), (k >> 1) & 1);
        const int nxt = clc_query(sSched + 16 * sl);
        if (nxt < 0) break;
        unit = nxt;
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == 2) {
    // ==================== MMA issuers: warp 1 -> tile 0, warp 2 -> tile 1 ====================
    // One issuing thread per query tile, each with blocking waits in its tile's natural
    // event order: S_t(j+1) as soon as softmax t has read S_t(j) (P lives in smem, so the
    // S buffer frees early), then PV_t(j) once P_t(j) is written. The tensor pipe
    // interleaves the two streams. K/V slots, the Q buffer and the scheduler slot are
    // released by BOTH issuers (barrier counts 2).
    // Whole warp: uniform control flow, tcgen05 ops by one elected lane (elect_one(): the
    // descriptors stay in uniform registers, no per-MMA R2UR loop).
    const int t = warp - 1;
    {
      constexpr uint32_t FMT = BF16 ? 1u : 0u;
      // S = Q K^T: A = Q (K-major), B = K (K-major), M=128, N=128; a_negate if scale < 0
      const uint32_t IDESC_QK = make_idesc_f16(FMT, BM, BN, 0, 0, p.neg ? 1u : 0u);
      // O += P V: A = P (K-major), B = V (MN-major: D contiguous), M=128, N=D
      constexpr uint32_t IDESC_PV = make_idesc_f16(FMT, BM, D, 0, 1, 0);
      const uint32_t tm_s = tmem_base + t * BN;
      const uint32_t tm_o = tmem_base + C::TMEM_O + t * D;
      const uint32_t qa = sQ + t * C::Q_TILE_BYTES;
      const uint32_t pa = sP + t * C::P_TILE_BYTES;
      const uint32_t tm_p = tmem_base + C::TMEM_P + t * (BN / 2);
      int unit = blockIdx.x;
      int it = 0;        // K/V ring position (same sequence as the producer)
      uint32_t cs = 0;   // S MMAs issued by this tile (cumulative: barrier phases)
      uint32_t cpv = 0;  // PV MMAs issued by this tile
      for (int k = 0;; ++k) {
        const Unit U = decode_unit(unit, p);
        const int nmax = max(U.n0, U.n1);
        const int nt = t ? U.n1 : U.n0;
        const int it0 = it;
        it += 2 * nmax;
        // ring positions (producer order K_0, K_1, V_0, K_2, V_1, ..., V_{nmax-1})
        auto kpos = [&](int j) { return it0 + (K_AHEAD ? (j == 0 ? 0 : 2 * j - 1) : 2 * j); };
        auto vpos = [&](int j) {
          return it0 + (K_AHEAD ? (j == nmax - 1 ? 2 * nmax - 1 : 2 * j + 2) : 2 * j + 1);
        };
        auto kslot = [&](int j) { return kpos(j) % C::NST; };
        auto kpar = [&](int j) { return (kpos(j) / C::NST) & 1; };
        auto vslot = [&](int j) { return vpos(j) % C::NST; };
        auto vpar = [&](int j) { return (vpos(j) / C::NST) & 1; };
        mbar_wait(bar_q_full, k & 1);
        // S_t(j) = Q_t K_j^T
        auto issue_s = [&](int j) {
          mbar_wait(bar_kv_full(kslot(j)), kpar(j));
#ifndef TLATTN_MMA_ONLY
          if (cs > 0) mbar_wait(bar_s_free(t), (cs - 1) & 1);  // softmax t has read S_t
#endif
          tc_fence_after();
          const uint32_t kb = sKV + kslot(j) * C::KV_BYTES;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
#ifdef TLATTN_SKIP_S
            break;
#endif
            // K-major SW128: a 16-element K step is +32 B inside the 128-B swizzle row;
            // every 64 elements the next 16 KB TMA box
            const uint32_t off = (kk >> 2) * CHUNK_BYTES + (kk & 3) * 32;
            if (elect_one())
              mma_f16_ss(tm_s, make_sdesc_sw128(qa + off, 16, 1024),
                         make_sdesc_sw128(kb + off, 16, 1024), IDESC_QK, kk > 0 ? 1u : 0u);
          }
          if (elect_one()) mma_commit(bar_s_full(t));
          if (elect_one()) mma_commit(bar_kv_empty(kslot(j)));  // this tile is done with K_j
          ++cs;
        };
        // O_t += P_t V_j
        auto issue_pv = [&](int j) {
          mbar_wait(bar_kv_full(vslot(j)), vpar(j));
#ifndef TLATTN_MMA_ONLY
          mbar_wait(bar_p_full(t), cpv & 1);
#endif
          tc_fence_after();
          const uint32_t vb = sKV + vslot(j) * C::KV_BYTES;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
#ifdef TLATTN_SKIP_PV
            break;
#endif
            // B = V MN-major SW128: 16 keys = 16 rows of 128 B (+2 KB); LBO = 16 KB to the
            // next 64-wide D chunk
            const uint64_t bd = make_sdesc_sw128(vb + kk * 2048, CHUNK_BYTES, 1024);
            if constexpr (C::P_TMEM) {
              // A = P_t in TMEM: 16 keys = 8 columns of packed 16-bit pairs
              if (elect_one())
                mma_f16_ts(tm_o, tm_p + kk * 8, bd, IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
            } else {
              // A = P (K-major SW128, 2 x 16 KB key chunks)
              const uint64_t ad = make_sdesc_sw128(pa + (kk >> 2) * CHUNK_BYTES + (kk & 3) * 32, 16, 1024);
              if (elect_one())
                mma_f16_ss(tm_o, ad, bd, IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
            }
          }
          if (elect_one()) mma_commit(bar_o_done(t));
          if (elect_one()) mma_commit(bar_kv_empty(vslot(j)));  // this tile is done with V_j
          ++cpv;
        };
        if (nt > 0) {
          issue_s(0);
          if ((nt == 1) && elect_one()) mma_commit(bar_q_empty);
          for (int j = 0; j < nt; ++j) {
            if (j + 1 < nt) {
              issue_s(j + 1);
              // last QK^T of this tile issued
              if ((j + 2 == nt) && elect_one()) mma_commit(bar_q_empty);
            }
            issue_pv(j);
          }
        } else {
          if (elect_one()) mbar_arrive(bar_q_empty);
        }
        // blocks this tile skips (causal): release its share of their K/V slots, after the
        // slot holds that block (so the arrival counts toward the right phase)
        for (int j = nt; j < nmax; ++j) {
          mbar_wait(bar_kv_full(kslot(j)), kpar(j));
          if (elect_one()) mbar_arrive(bar_kv_empty(kslot(j)));
          mbar_wait(bar_kv_full(vslot(j)), vpar(j));
          if (elect_one()) mbar_arrive(bar_kv_empty(vslot(j)));
        }
        mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
        const int nxt = clc_query(sSched + 16 * (k & 1));
        if (elect_one()) mbar_arrive(bar_sched_empty(k & 1));
        if (nxt < 0) break;
        unit = nxt;
      }
    }
    __syncwarp();
  }
  } else {
    setmaxnreg_inc<REGS_SOFTMAX>();
    // =========================== softmax / correction / epilogue ===========================
    const int t = (warp - SOFTMAX_WARP0) >> 2;     // query tile of the unit
    const int q4 = warp & 3;                        // TMEM lane quarter this warp may access
    const int lr = q4 * 32 + lane;                  // row within tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tm_s = tmem_base + lane_off + t * BN;
    const uint32_t tm_o = tmem_base + lane_off + C::TMEM_O + t * D;
    const uint32_t p_row = sP + t * C::P_TILE_BYTES + lr * 128;
    const uint32_t tm_p_row = tmem_base + lane_off + C::TMEM_P + t * (BN / 2);
    const float c = p.c_log2;
    int unit = blockIdx.x;
    uint32_t g = 0;  // blocks processed by this tile's warpgroup (cumulative, barrier phases)
    for (int k = 0;; ++k) {
      const Unit U = decode_unit(unit, p);
#ifdef TLATTN_MMA_ONLY
      const int nt = 0;  // experiment: tensor/TMA data path alone
#else
      const int nt = t ? U.n1 : U.n0;
#endif
      const int row = U.m_blk * (TILES * BM) + t * BM + lr;  // global query index
      // last key index this row may attend to (inclusive); bottom-right causal (R3)
      const int limit = p.causal ? min(p.Skv - 1, row + p.Skv - p.Sq) : (p.Skv - 1);
      float m = -INFINITY;  // running max of c*s (scores_max; reading R2)
      float l = 0.f;        // running sum        (logsum)

      for (int j = 0; j < nt; ++j, ++g) {
        mbar_wait(bar_s_full(t), g & 1);
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * (j & 15) + 0);
        tc_fence_after();
        uint32_t sr[BN];
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc)
          tmem_ld32(tm_s + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + cc * 32));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s_free(t));  // S_t may be overwritten by QK^T(j+1)
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * (j & 15) + 1);

        float m_new, alpha, sum;
        uint32_t pk[BN / 2];
        softmax_row_block<BF16, (D == 64 ? TLATTN_EMU64 : 0)>(sr, j * BN, limit, c, m, m_new, alpha, sum, pk);
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * (j & 15) + 2);
        if (j > 0) {
          // O_t must hold PV_t(j-1) before it is rescaled and before P_t smem is reused
          mbar_wait(bar_o_done(t), (g - 1) & 1);
          if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * (j & 15) + 3);
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {  // acc_o *= scores_scale
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
        if constexpr (C::P_TMEM) {
          // P row -> TMEM (this thread's lane, 64 columns of packed 16-bit pairs): the TS
          // MMA's A operand; no SMEM traffic, no proxy fence
          tmem_st32(tm_p_row, *reinterpret_cast<const uint32_t(*)[32]>(pk));
          tmem_st32(tm_p_row + 32, *reinterpret_cast<const uint32_t(*)[32]>(pk + 32));
          tmem_st_wait();
        } else {
        // P row -> smem, K-major SWIZZLE_128B: 16-B unit u of a 64-key chunk -> u ^ (row & 7)
#pragma unroll
        for (int ch = 0; ch < BN / 64; ++ch) {
#pragma unroll
          for (int uu = 0; uu < 8; ++uu) {
#ifdef TLATTN_NO_PSTORE
            if (uu != 0) continue;
#endif
            const uint32_t addr = p_row + ch * CHUNK_BYTES + ((uu ^ (lr & 7)) << 4);
            const int w = ch * 32 + uu * 4;
            st_shared_v4(addr, pk[w], pk[w + 1], pk[w + 2], pk[w + 3]);
          }
        }
        fence_proxy_async_smem();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p_full(t));
        if (lane == 0 && q4 == 0) TL_TRACE2(k, 1000 * t + 8 * (j & 15) + 4);
        l = l * alpha + sum;  // logsum = logsum * scores_scale + scores_sum
        m = m_new;
      }

      // ---- epilogue: O / l, LSE, store
      if (nt > 0) {
        mbar_wait(bar_o_done(t), (g - 1) & 1);
        tc_fence_after();
      }
      const float inv_l = (l > 0.f) ? (1.f / l) : 0.f;
      const bool row_ok = row < p.Sq;
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
        if (row_ok) {
          for (int r = 0; r < n_outputs(p); ++r) {
            uint8_t* orow = out_row(p, r, U.b, U.h, row, D);
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4)
              st_global_v4(orow + cc * 64 + v4 * 16, pkd[4 * v4], pkd[4 * v4 + 1], pkd[4 * v4 + 2],
                           pkd[4 * v4 + 3]);
          }
        }
      }
      if (row_ok) {
        // lse = ln sum exp(scale*s) = (m + log2 l) ln 2, m in log2 units (reading R5)
        store_lse(p, U.b, U.h, row, (l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY);
      }
      tc_fence_before();  // O_t reads complete before the next unit's first PV_t overwrites

      mbar_wait(bar_sched_full(k & 1), (k >> 1) & 1);
      const int nxt = clc_query(sSched + 16 * (k & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_sched_empty(k & 1));
      if (nxt < 0) break;
      unit = nxt;
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace tlattn
