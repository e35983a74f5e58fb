/*
 * tlattn.h — C ABI of libtlattn, the B200 (sm_100a) fused attention forward.
 *
 * Operation (§5.2 P:L362 / Fig. 12: the FlashAttention forward; Fig. 18
 * P:L573-696 gives the tiled online-softmax algorithm; "exact attention", ref [12]
 * P:L424):
 *
 *   o[b,i,h,:] = sum_{j in J_i} softmax_j( scale * q[b,i,h,:] . k[b,j,g,:] ) * v[b,j,g,:]
 *   g   = h / (Hq / Hkv)                 GQA grouping, cur_kv_head
 *   J_i = { 0 <= j < Skv : !causal || j <= i + Skv - Sq }   (bottom-right causal)
 *   lse[b,h,i] = ln sum_{j in J_i} exp(scale * q.k_j)        (natural log)
 *   J_i empty (only causal with Sq > Skv): o = 0, lse = -inf
 *
 * Precision (P:L592, P:L602-614 dtype / accum_dtype): q, k, v, o are fp16 or bf16;
 * S = QK^T and O = PV accumulate in fp32 (tensor-core TMEM accumulators); the
 * running max and row sum are fp32, the row sum is taken over the unrounded fp32
 * probabilities; P is rounded to the input dtype (round-to-nearest-even) before
 * the PV product; O is rounded RN on output.
 *
 * Layout (KV[batch, seqlen_kv, kv_head_num, dim]): contiguous BSHD,
 *   q[B][Sq][Hq][D], k[B][Skv][Hkv][D], v[B][Skv][Hkv][D], o[B][Sq][Hq][D],
 *   lse[B][Hq][Sq] fp32.
 *
 * Ownership: the caller owns every buffer. The library allocates no device memory
 * and keeps no pointer after a call returns; it caches only immutable per-device
 * attributes (SM count, compute capability), initialised thread-safely.
 * o / lse must not alias q / k / v.
 *
 * Synchronisation: tl_attn_fwd is stream-ordered and asynchronous (no host sync, no
 * allocation: CUDA-graph capturable). Device faults surface at the caller's next
 * synchronisation, as usual for CUDA.
 *
 * Errors: argument errors are returned synchronously BEFORE any CUDA call and
 * nothing is launched. There is no CPU fallback: a device that is not sm_100
 * returns TL_ERR_UNSUPPORTED.
 */
#ifndef TLATTN_H
#define TLATTN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLATTN_VERSION 0x000300 /* 0.3.0: bounded tl_peer_barrier (+ _set_timeout_ns, _check); tl_attn_set/get_option; tl_ssd_chunk_state / _scan */

enum tl_dtype { TL_DTYPE_F16 = 0, TL_DTYPE_BF16 = 1 };

enum tl_status {
  TL_OK = 0,
  /* NULL q/k/v/o; B, Hq, Hkv, Sq, Skv or D < 1; causal not 0/1; scale not finite;
     unknown dtype; nbytes/workspace too small (tl_attn_fwd_host) */
  TL_ERR_INVALID_VALUE = 1,
  /* D not in {64, 128}; Hq % Hkv != 0; q/k/v/o not 16-byte aligned or lse not 4-byte
     aligned; a tensor too large for 32-bit TMA coordinates; device not sm_100 */
  TL_ERR_UNSUPPORTED = 2,
  /* a CUDA runtime / driver call failed (no device, tensor-map encode, launch) */
  TL_ERR_CUDA = 3,
  /* tl_peer_barrier: a peer did not arrive within the barrier's timeout (reported by
     tl_peer_barrier_check after the barrier kernel ran) */
  TL_ERR_TIMEOUT = 4
};

/*
 * tl_attn_fwd — fused attention forward on the current CUDA device.
 *
 *   q, k, v  device pointers, contiguous BSHD (see above), 16-byte aligned
 *   o        device pointer, contiguous BSHD [B][Sq][Hq][D], written in full
 *   lse      device pointer to fp32 [B][Hq][Sq], 4-byte aligned, or NULL (not written)
 *   B, Hq, Hkv, Sq, Skv, D    sizes; Hq % Hkv == 0; D in {64, 128}; all >= 1
 *   causal   0 = full attention, 1 = bottom-right causal mask (j <= i + Skv - Sq)
 *   scale    natural-exp score scale, used literally (callers normally pass 1/sqrt(D));
 *            0 and negative values are legal
 *   dtype    TL_DTYPE_F16 or TL_DTYPE_BF16 (q, k, v and o share it)
 *   stream   cudaStream_t (as void*) to launch on; NULL = legacy default stream
 *
 * Returns TL_OK or a tl_status code (see tl_attn_strerror).
 */
int tl_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                int B, int Hq, int Hkv, int Sq, int Skv, int D,
                int causal, float scale, int dtype, void* stream);

/*
 * tl_attn_fwd_host — the same operation on HOST buffers (the end-to-end entry point).
 *
 * q_h, k_h, v_h, o_h, lse_h are host pointers (pinned memory gives full PCIe speed;
 * lse_h may be NULL). The library stages them through the caller-provided DEVICE
 * workspace `ws` of `ws_bytes` bytes (>= tl_attn_host_workspace_bytes(...)),
 * copying inputs host->device, running tl_attn_fwd and copying o (and lse)
 * device->host on `stream`. Batches are processed in chunks so that the copies of
 * one chunk overlap the attention of another (two internal chunk slots in `ws`).
 * Stream-ordered; the host buffers must stay valid until the stream reaches this
 * point. Returns TL_OK or a tl_status code.
 */
int tl_attn_fwd_host(const void* q_h, const void* k_h, const void* v_h, void* o_h, float* lse_h,
                     int B, int Hq, int Hkv, int Sq, int Skv, int D,
                     int causal, float scale, int dtype,
                     void* ws, uint64_t ws_bytes, void* stream);

/* Device workspace bytes tl_attn_fwd_host needs for this problem (0 on bad arguments). */
uint64_t tl_attn_host_workspace_bytes(int B, int Hq, int Hkv, int Sq, int Skv, int D,
                                      int with_lse);

/*
 * tl_gemm — dense GEMM C = A · B (Fig. 1 / Fig. 16 "Matmul",
 * P:L58-157; benchmark shapes Table 2), on the current device.
 *
 *   a      device pointer, A [M][K] row-major (K contiguous), fp16 or bf16
 *   b      device pointer, B [K][N] row-major (N contiguous), same dtype
 *   c      device pointer, C [M][N] row-major, same dtype, written in full
 *   M,N,K  sizes >= 1; N and K multiples of 8 (16-byte TMA row strides)
 *   dtype  TL_DTYPE_F16 or TL_DTYPE_BF16; accumulation is fp32, C is rounded RN
 *   stream cudaStream_t as void*
 *
 * M = 1 (the GEMV rows of Table 2) runs an HBM-bound kernel instead of the tensor-core
 * tiles: clusters of 8 CTAs split K and reduce through distributed shared memory in a
 * fixed order (deterministic). Both paths are one kernel launch.
 *
 * Ownership / synchronisation as tl_attn_fwd (caller-owned buffers, stream-ordered, no
 * allocation, graph-capturable). c must not alias a or b.
 * Errors: TL_ERR_INVALID_VALUE (NULL pointer, size < 1, bad dtype), TL_ERR_UNSUPPORTED
 * (N or K not a multiple of 8, pointer not 16-byte aligned, too many tiles, device not
 * sm_100), TL_ERR_CUDA. Argument errors are returned before any CUDA call.
 */
int tl_gemm(const void* a, const void* b, void* c, int M, int N, int K, int dtype, void* stream);

/*
 * tl_mla_decode — Multi-Head Latent Attention decode (PAPER.md Appendix
 * B.3, Fig. 18 "FlashMLA"; benchmarked in Fig. 14), on the current
 * device. One query token per (batch, head) attends to a latent KV cache:
 *
 *   n_b   = seqlens ? clamp(seqlens[b], 0, Skv) : Skv          (reading M1)
 *   g     = h / (H / Hkv)                                         (cur_kv_head)
 *   s_j   = scale * ( q[b,h,:] . kv[b,j,g,:] + q_pe[b,h,:] . k_pe[b,j,g,:] ),  j < n_b
 *                                                 (two T.gemm into acc_s)
 *   o[b,h,:]  = sum_j softmax_j(s) * kv[b,j,g,:]  (the value operand is KV itself)
 *   lse[b,h]  = ln sum_j exp(s_j);   n_b = 0: o = 0, lse = -inf
 *
 *   q        device, [B][H][Dl]          contiguous, 16-byte aligned
 *   q_pe     device, [B][H][Dr]
 *   kv       device, [B][Skv][Hkv][Dl]   (Fig. 18 KV[batch, seqlen_kv, kv_head_num, dim])
 *   k_pe     device, [B][Skv][Hkv][Dr]
 *   o        device, [B][H][Dl], written in full
 *   lse      device fp32 [B][H] (natural log), 4-byte aligned, or NULL
 *   seqlens  device int32 [B] (per-batch cache lengths, clamped to [0, Skv] on the
 *            device), or NULL (every batch has Skv keys)
 *   Dl, Dr   must be 512 and 64 (the DeepSeek latent / rope dims of Fig. 18)
 *   scale    natural-exp scale (callers normally pass 1/sqrt(Dl + Dr)); 0 / negative legal
 *   dtype    TL_DTYPE_F16 or TL_DTYPE_BF16 for q, q_pe, kv, k_pe and o
 *   ws       device workspace of ws_bytes >= tl_mla_decode_workspace_bytes(B, H, Hkv),
 *            256-byte aligned; holds the split-KV partial results (contents scratch)
 *   stream   cudaStream_t as void*
 *
 * Precision as tl_attn_fwd: fp32 scores and accumulators, fp32 l over unrounded p,
 * P rounded RN to dtype before the PV product, O rounded RN. Split-KV pieces are merged in
 * fp32. Three kernels per call (key-block prefix sums, decode, merge); stream-ordered, no
 * allocation, graph-capturable. Ownership as tl_attn_fwd.
 * Errors: TL_ERR_INVALID_VALUE (NULL q/q_pe/kv/k_pe/o/ws, size < 1, non-finite scale, bad
 * dtype, workspace too small); TL_ERR_UNSUPPORTED (Dl != 512 or Dr != 64, H % Hkv != 0,
 * misaligned pointer, sizes beyond 32-bit TMA coordinates, device not sm_100);
 * TL_ERR_CUDA. Argument errors are returned before any CUDA call.
 */
int tl_mla_decode(const void* q, const void* q_pe, const void* kv, const void* k_pe, void* o,
                  float* lse, const int* seqlens, int B, int H, int Hkv, int Skv, int Dl, int Dr,
                  float scale, int dtype, void* ws, uint64_t ws_bytes, void* stream);

/* Device workspace bytes tl_mla_decode needs on the CURRENT device (it depends on the SM
 * count); 0 on bad arguments or when no device is available. */
uint64_t tl_mla_decode_workspace_bytes(int B, int H, int Hkv);

/*
 * tl_attn_fwd_replicated — tl_attn_fwd on this rank's shard with the output REPLICATED
 * into several full-size buffers by the kernel itself (the replicated
 * output of §8(e) fused into the epilogue; the paper lists tile-level communication
 * primitives as future work). Each O tile leaves shared memory once per output
 * buffer (TMA bulk-tensor stores; over NVLink when the buffer is a peer GPU's memory), so
 * the all-gather overlaps the attention of the remaining tiles instead of following it.
 *
 *   q, k, v      this rank's shard, device pointers, contiguous BSHD: q [B][Sq][Hq][D],
 *                k, v [B][Skv][Hkv][D] (as tl_attn_fwd)
 *   o_outs       HOST array of n_outs device pointers (1 <= n_outs <= 8), each a full
 *                output [B_total][Sq][Hq_total][D] valid in this process (own buffer, or a
 *                peer's opened with tl_ipc_open_handle); 16-byte aligned
 *   lse_outs     NULL, or HOST array of n_outs device pointers (entries may be NULL) to full
 *                fp32 LSE [B_total][Hq_total][Sq]; 4-byte aligned
 *   B_total, b_off, Hq_total, h_off
 *                full sizes and this shard's offsets: local (b, h) is written to
 *                (b + b_off, h + h_off); b_off + B <= B_total, h_off + Hq <= Hq_total
 *                (head shard: b_off = 0, h_off = rank * Hq; batch shard: h_off = 0)
 *   other arguments as tl_attn_fwd
 *
 * Only this shard's rows of each output are written. One kernel launch, stream-ordered, no
 * allocation, graph-capturable. Writes into peer memory are complete when the kernel is;
 * readers on other ranks must order after it (tl_peer_barrier). Ownership: the caller owns
 * every buffer (and the IPC mappings). Errors as tl_attn_fwd, plus TL_ERR_INVALID_VALUE for
 * NULL o_outs / entries, n_outs outside [1, 8] or offsets outside the full sizes.
 */
int tl_attn_fwd_replicated(const void* q, const void* k, const void* v,
                           void* const* o_outs, float* const* lse_outs, int n_outs,
                           int B_total, int b_off, int Hq_total, int h_off,
                           int B, int Hq, int Hkv, int Sq, int Skv, int D,
                           int causal, float scale, int dtype, void* stream);

/*
 * tl_peer_barrier — stream-ordered device-side barrier among `world` ranks (one kernel).
 *
 *   flags   HOST array of `world` device pointers (world <= 8): flags[r] = rank r's array
 *           of TL_PEER_FLAG_WORDS uint32 as mapped in THIS process (flags[rank] = own array;
 *           peers' opened with tl_ipc_open_handle); zero-initialised once by their owners.
 *           Words [0, world) are the epoch counters, word TL_PEER_STATUS_WORD the status.
 *   rank    this rank; epoch: a value that increases by 1 on every use (wraps mod 2^32)
 *
 * Rank `rank` stores `epoch` into flags[r][rank] for every r (system-scope release, after
 * this stream's earlier work) and waits until flags[rank][r] >= epoch for every r
 * (acquire). After it, this stream sees every rank's writes issued before that rank's
 * barrier (e.g. tl_attn_fwd_replicated into this rank's output). All ranks must call it
 * with the same epoch sequence.
 * The wait is BOUNDED: a peer that has not arrived after the timeout (default 10 s,
 * tl_peer_barrier_set_timeout_ns) makes the kernel store TL_ERR_TIMEOUT into
 * flags[rank][TL_PEER_STATUS_WORD] and return instead of hanging the stream; read it with
 * tl_peer_barrier_check. The status word is sticky until the owner rewrites it.
 * Errors (synchronous): TL_ERR_INVALID_VALUE (NULL / misaligned flags, bad world / rank),
 * TL_ERR_CUDA.
 */
#define TL_PEER_FLAG_WORDS 16
#define TL_PEER_STATUS_WORD 15
int tl_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, void* stream);
/* Timeout of later tl_peer_barrier calls on this host thread, in nanoseconds (> 0). */
int tl_peer_barrier_set_timeout_ns(uint64_t ns);
/* Synchronises the current device, then reads own_flags[TL_PEER_STATUS_WORD]: TL_OK, or
 * TL_ERR_TIMEOUT if a barrier on this rank's flags timed out; TL_ERR_CUDA / _INVALID_VALUE. */
int tl_peer_barrier_check(const uint32_t* own_flags);

/* CUDA IPC helpers for the peer buffers above (wrappers over cudaIpc*MemHandle): a handle
 * is tl_ipc_handle_bytes() opaque bytes the caller ships to other processes (e.g. with
 * torch.distributed.all_gather_object). tl_ipc_get_handle: dev_ptr must be the base of a
 * cudaMalloc allocation. tl_ipc_open_handle maps another process's allocation into this
 * one (same or peer GPU); close with tl_ipc_close_handle. Return TL_OK, TL_ERR_INVALID_VALUE
 * (NULL arguments) or TL_ERR_CUDA. */
int tl_ipc_handle_bytes(void);
int tl_ipc_get_handle(const void* dev_ptr, void* handle_out);
int tl_ipc_open_handle(const void* handle, void** dev_ptr_out);
int tl_ipc_close_handle(void* dev_ptr);

/*
 * Mamba-2 SSD chunk kernels ("linear attention"): the chunk-state and
 * chunk-scan functions of Mamba-2 the paper benchmarks (§5.2, Table 4
 * P:L464-478). The paper prints no formula; the definitions below are the Mamba-2 SSD
 * chunked algorithm for the scalar-decay SSM h_t = exp(dt_t A_h) h_{t-1} + dt_t B_t x_t^T,
 * y_t = C_t^T h_t + D_h x_t (readings L1-L8). Chunk c covers positions
 * [cQ, cQ + len_c), len_c = min(Q, seqlen - cQ); nchunks = ceil(seqlen / Q); head h uses
 * group g = h / (nheads / ngroups).
 *
 * tl_ssd_chunk_state:
 *   states[b,c,h,p,n] = sum_{i < len_c} x[b,cQ+i,h,p] Bm[b,cQ+i,g,n]
 *                        * exp(dA[b,h,c,len_c-1] - dA[b,h,c,i]) * dt[b,h,c,i]
 * tl_ssd_chunk_scan:
 *   out[b,cQ+i,h,p] = exp(dA[b,h,c,i]) sum_n C[b,cQ+i,g,n] prev[b,c,h,p,n]
 *                    + sum_{j <= i} cb[b,c,g,i,j] exp(dA[b,h,c,i] - dA[b,h,c,j]) dt[b,h,c,j] x[b,cQ+j,h,p]
 *                    + D[h] x[b,cQ+i,h,p]
 *
 *   x       [batch][seqlen][nheads][headdim]            16-bit (dtype), 16-byte aligned
 *   Bm, C   [batch][seqlen][ngroups][dstate]            16-bit
 *   dt, dA  [batch][nheads][nchunks][chunk_size] fp32 (dt > 0: the step sizes; dA: the
 *           inclusive cumulative sum of dt * A_h inside each chunk); entries i >= len_c of
 *           the last chunk are ignored
 *   cb      [batch][nchunks][ngroups][chunk_size][chunk_size] 16-bit (C B^T per chunk)
 *   prev_states / states [batch][nchunks][nheads][headdim][dstate] 16-bit
 *   D       [nheads] fp32, or NULL (no skip term)
 *   out     [batch][seqlen][nheads][headdim] 16-bit
 * fp32 accumulation; chunk_state rounds each state RN to dtype, chunk_scan each output.
 * Supported: headdim = 64, dstate = 128, chunk_size = 256 (Table 4 / reading L2), fp16 or
 * bf16, nheads % ngroups == 0; chunk_state also needs nheads / ngroups even (the two
 * heads of a CTA's head pair share one group's Bm tile).
 * One kernel launch each, stream-ordered, no allocation, graph-capturable; the caller owns
 * every buffer. Errors: TL_ERR_INVALID_VALUE (NULL pointers, sizes < 1, nheads % ngroups,
 * bad dtype), TL_ERR_UNSUPPORTED (headdim / dstate / chunk_size / odd nheads / ngroups, misaligned
 * pointers, sizes beyond 32-bit TMA coordinates, device not sm_100), TL_ERR_CUDA.
 */
int tl_ssd_chunk_state(const void* x, const void* Bm, const float* dt, const float* dA,
                       void* states, int batch, int seqlen, int nheads, int ngroups, int headdim,
                       int dstate, int chunk_size, int dtype, void* stream);
int tl_ssd_chunk_scan(const void* cb, const void* x, const float* dt, const float* dA,
                      const void* C, const void* prev_states, const float* D, void* out,
                      int batch, int seqlen, int nheads, int ngroups, int headdim, int dstate,
                      int chunk_size, int dtype, void* stream);

/* Static, NUL-terminated description of a tl_status code. Never NULL. */
const char* tl_attn_strerror(int status);

/* TLATTN_VERSION of the loaded library. */
int tl_attn_version(void);

/*
 * Experiment / test options (process-wide; NOT needed for normal use). Each defaults to
 * -1 = automatic (the launcher's measured choice); the tools/ A/B scripts seed them once
 * from the environment (TLATTN_KERNEL=1cta, TLATTN_UNIT_TILES, TLATTN_LPT, TLATTN_GEMV_TC,
 * TLATTN_MLA_HC, TLATTN_MLA_CL) on first use. Values outside an option's set are ignored
 * by the launcher (automatic). tl_attn_set_option returns TL_OK or TL_ERR_INVALID_VALUE
 * (unknown option); tl_attn_get_option returns the current value (-2: unknown option).
 *   TL_OPT_FORCE_1CTA  1: D = 128 on the single-CTA kernel instead of CTA pairs
 *   TL_OPT_UNIT_TILES  1 or 2 query tiles of 256 rows per CTA-pair unit
 *   TL_OPT_LPT         0: (b, h)-major unit order; 1: heaviest query block first (LPT)
 *   TL_OPT_GEMV_TC     GEMV (M = 1) column tile: 32, 64, 128 or 256
 *   TL_OPT_MLA_HC      MLA heads per CTA tile: 32 or 64
 *   TL_OPT_MLA_CL      MLA K/V multicast cluster size: 1, 2 or 4
 */
enum tl_option {
  TL_OPT_FORCE_1CTA = 0,
  TL_OPT_UNIT_TILES = 1,
  TL_OPT_LPT = 2,
  TL_OPT_GEMV_TC = 3,
  TL_OPT_MLA_HC = 4,
  TL_OPT_MLA_CL = 5,
  TL_OPT_COUNT = 6
};
int tl_attn_set_option(int option, int value);
int tl_attn_get_option(int option);

/* Number of kernel launches the most recent successful tl_attn_fwd / tl_attn_fwd_host /
 * tl_attn_fwd_replicated / tl_peer_barrier / tl_gemm / tl_mla_decode call on this host
 * thread issued (tl_attn_fwd: 1, tl_mla_decode: 3). For accounting in benchmarks. */
int tl_attn_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TLATTN_H */
