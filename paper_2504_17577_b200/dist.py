"""Multi-GPU partitioning of the attention forward.

The forward shards with no exchange: every (b, kv-head group) is independent
(Fig. 18: the grid is (batch, heads)). Two partitions:

  head shard (default)  rank r owns kv-heads [r*Hkv/w, (r+1)*Hkv/w) and their query heads
                        [r*Hq/w, (r+1)*Hq/w) for all batches -> local q/o [B, S, Hq/w, D],
                        k/v [B, S, Hkv/w, D]; each GQA group stays on one rank.
  batch shard           rank r owns batches [r*B/w, (r+1)*B/w).

Each rank calls tl_attn_fwd on its local shard (kernel unchanged). The only collective
is the optional all-gather that replicates O (and LSE) when the caller asks for it;
NCCL over NVLink in production, gloo in the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    mode: str
    rank: int
    world: int
    b: slice
    hq: slice
    hkv: slice

    def local_dims(self, B, Hq, Hkv):
        return (self.b.stop - self.b.start, self.hq.stop - self.hq.start,
                self.hkv.stop - self.hkv.start)


def make_shard(mode: str, rank: int, world: int, B: int, Hq: int, Hkv: int) -> Shard:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if mode == "head":
        if Hkv % world != 0:
            raise ValueError(f"head shard needs world | Hkv (Hkv={Hkv}, world={world})")
        gk = Hkv // world
        gq = Hq // world
        return Shard(mode, rank, world, slice(0, B), slice(rank * gq, (rank + 1) * gq),
                     slice(rank * gk, (rank + 1) * gk))
    if mode == "batch":
        if B % world != 0:
            raise ValueError(f"batch shard needs world | B (B={B}, world={world})")
        gb = B // world
        return Shard(mode, rank, world, slice(rank * gb, (rank + 1) * gb), slice(0, Hq),
                     slice(0, Hkv))
    raise ValueError(f"unknown shard mode {mode!r}")


def gather_output(o_local: torch.Tensor, lse_local: torch.Tensor | None, shard: Shard,
                  group=None):
    """Replicate the full O[B, S, Hq, D] (and LSE[B, Hq, S]) on every rank.

    Batch shards concatenate directly along B. Head shards gather into
    [w, B, S, Hq/w, D] and are permuted into BSHD (LSE: [w, B, Hq/w, S] -> [B, Hq, S]).
    """
    w = shard.world
    o_local = o_local.contiguous()
    buf = torch.empty((w * o_local.numel(),), dtype=o_local.dtype, device=o_local.device)
    dist.all_gather_into_tensor(buf, o_local.view(-1), group=group)
    Bl, S, Hl, D = o_local.shape
    if shard.mode == "batch":
        o_full = buf.view(w * Bl, S, Hl, D)
    else:
        o_full = buf.view(w, Bl, S, Hl, D).permute(1, 2, 0, 3, 4).reshape(Bl, S, w * Hl, D)
    lse_full = None
    if lse_local is not None:
        lse_local = lse_local.contiguous()
        lbuf = torch.empty((w * lse_local.numel(),), dtype=lse_local.dtype, device=lse_local.device)
        dist.all_gather_into_tensor(lbuf, lse_local.view(-1), group=group)
        Bl2, Hl2, S2 = lse_local.shape
        if shard.mode == "batch":
            lse_full = lbuf.view(w * Bl2, Hl2, S2)
        else:
            lse_full = lbuf.view(w, Bl2, Hl2, S2).permute(1, 0, 2, 3).reshape(Bl2, w * Hl2, S2)
    return o_full, lse_full


def replica_layout(shard: Shard, B: int, Hq: int):
    """(B_total, b_off, Hq_total, h_off) of this rank's shard inside the full output."""
    return B, shard.b.start, Hq, shard.hq.start


def _al(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


class ReplicatedOutput:
    """Full O[B, Sq, Hq, D] (and LSE[B, Hq, Sq]) on every rank, written by the attention
    kernel itself (include/tlattn.h tl_attn_fwd_replicated).

    Each rank owns one device allocation [O | LSE | flags], maps every peer's allocation
    into its address space once (CUDA IPC handles exchanged with all_gather_object), and
    on every call runs its shard with the epilogue storing each O tile into all ranks'
    buffers (NVLink P2P stores for peer GPUs), followed by a device-side flag barrier
    (tl_peer_barrier) so each rank's stream sees every shard. A barrier also precedes the
    kernel (pre_barrier) so no rank overwrites a buffer a peer may still be reading.
    world <= 8. Host logic only: every byte of O moves inside the kernels.
    """

    def __init__(self, shard: Shard, B: int, Sq: int, Hq: int, D: int, dtype, with_lse=True,
                 device=None, group=None):
        from . import tlattn as T
        if shard.world > 8:
            raise ValueError("replicated output supports up to 8 ranks")
        self.shard, self.B, self.Sq, self.Hq, self.D = shard, B, Sq, Hq, D
        self.dtype, self.with_lse = dtype, with_lse
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        esz = torch.empty((), dtype=dtype).element_size()
        o_bytes = B * Sq * Hq * D * esz
        lse_bytes = B * Hq * Sq * 4 if with_lse else 0
        self.off_lse = _al(o_bytes)
        self.off_flags = self.off_lse + _al(lse_bytes)
        total = self.off_flags + _al(4 * T.TL_PEER_FLAG_WORDS)
        self.buf = torch.zeros(total, dtype=torch.uint8, device=dev)
        self.o = self.buf[:o_bytes].view(dtype).view(B, Sq, Hq, D)
        self.lse = (self.buf[self.off_lse:self.off_lse + lse_bytes].view(torch.float32)
                    .view(B, Hq, Sq) if with_lse else None)
        torch.cuda.synchronize(dev)
        handle = T.tl_ipc_get_handle(self.buf)
        handles = [None] * shard.world
        dist.all_gather_object(handles, handle, group=group)
        self.bases, self._opened = [], []
        for r, h in enumerate(handles):
            if r == shard.rank:
                self.bases.append(self.buf.data_ptr())
            else:
                p = T.tl_ipc_open_handle(h)
                self._opened.append(p)
                self.bases.append(p)
        self.o_ptrs = list(self.bases)
        self.lse_ptrs = [b + self.off_lse for b in self.bases] if with_lse else None
        self.flag_ptrs = [b + self.off_flags for b in self.bases]
        self.epoch = 0
        self.group = group
        dist.barrier(group=group)  # every rank's flags are zeroed and mapped before first use

    def barrier(self, stream=None):
        from . import tlattn as T
        self.epoch += 1
        T.tl_peer_barrier(self.flag_ptrs, self.shard.rank, self.epoch, stream)

    def check(self):
        """Synchronise and raise TlAttnError(TL_ERR_TIMEOUT) if one of this rank's device
        barriers gave up waiting for a peer (a dead rank no longer hangs the others)."""
        from . import tlattn as T
        T.tl_peer_barrier_check(self.flag_ptrs[self.shard.rank])

    def __call__(self, q, k, v, causal=False, scale=None, stream=None, pre_barrier=True):
        """Run this rank's shard (local q [B_l, Sq, Hq_l, D], k/v [B_l, Skv, Hkv_l, D]) and
        return the full (O, LSE) views of this rank's buffer, complete on `stream`."""
        import math

        from . import tlattn as T
        if q.dim() != 4 or k.dim() != 4 or v.dim() != 4 or k.shape != v.shape:
            raise ValueError("expected BSHD q[B_l,Sq,Hq_l,D], k/v[B_l,Skv,Hkv_l,D]")
        Bl, Sq, Hl, D = q.shape
        Skv, Hkvl = k.shape[1], k.shape[2]
        # the kernel builds every output tensor map from the CALL's sizes: a call that does
        # not match the buffers allocated here (or this rank's shard) would write past O into
        # the LSE / flag region of every peer, so refuse it before any launch
        if Sq != self.Sq or D != self.D or q.dtype != self.dtype or k.dtype != self.dtype or \
                v.dtype != self.dtype:
            raise ValueError(f"ReplicatedOutput was built for Sq={self.Sq}, D={self.D}, "
                             f"{self.dtype}; got Sq={Sq}, D={D}, {q.dtype}/{k.dtype}/{v.dtype}")
        sh = self.shard
        b_len = len(range(*sh.b.indices(self.B)))
        hq_len = len(range(*sh.hq.indices(self.Hq)))
        if Bl != b_len or Hl != hq_len or k.shape[0] != Bl:
            raise ValueError(f"this rank's shard is B_l={b_len}, Hq_l={hq_len}; got q with "
                             f"B_l={Bl}, Hq_l={Hl} and k/v with B_l={k.shape[0]}")
        if Hl % Hkvl != 0:
            raise ValueError("Hq_l must be a multiple of Hkv_l")
        scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
        B_total, b_off, Hq_total, h_off = replica_layout(self.shard, self.B, self.Hq)
        if pre_barrier:
            self.barrier(stream)
        T.tl_attn_fwd_replicated(q, k, v, self.o_ptrs, self.lse_ptrs, B_total, b_off, Hq_total,
                                 h_off, Bl, Hl, Hkvl, Sq, Skv, D, int(bool(causal)), scale,
                                 T.dtype_code(q.dtype), stream)
        self.barrier(stream)
        return self.o, self.lse

    def close(self):
        from . import tlattn as T
        for p in self._opened:
            T.tl_ipc_close_handle(p)
        self._opened = []
