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
