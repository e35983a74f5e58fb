"""Multi-GPU partitioning logic on CPU (gloo, world size 2 and 4).

The forward shards with no exchange (each (b, kv-head group) is independent, PAPER.md
Fig. 18 grid (batch, heads)). Each rank generates ITS shard of the seeded
inputs from global indices, computes it, and the optional all-gather reassembles O and
LSE. Here the per-rank compute is the fp64 oracle (test-only stand-in for the kernel on
a CPU box); the partition, the shard-local input generation and the reassembly are the
production code of paper_2504_17577_b200.dist / .inputs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_17577_b200.dist import gather_output, make_shard
from paper_2504_17577_b200.inputs import gen_qkv, to_bits

B, HQ, HKV, S, D = 4, 8, 4, 12, 8
SEED = 4242


def test_head_shard_partition_covers_every_head_once():
    for w in (1, 2, 4):
        seen_q, seen_kv = [], []
        for r in range(w):
            sh = make_shard("head", r, w, B, HQ, HKV)
            seen_q += list(range(sh.hq.start, sh.hq.stop))
            seen_kv += list(range(sh.hkv.start, sh.hkv.stop))
            # every query head of the shard maps (h / (Hq/Hkv)) into the shard's kv heads
            for h in range(sh.hq.start, sh.hq.stop):
                assert sh.hkv.start <= h // (HQ // HKV) < sh.hkv.stop
        assert sorted(seen_q) == list(range(HQ)) and sorted(seen_kv) == list(range(HKV))


def test_batch_shard_partition_and_errors():
    for w in (1, 2, 4):
        got = []
        for r in range(w):
            sh = make_shard("batch", r, w, B, HQ, HKV)
            got += list(range(sh.b.start, sh.b.stop))
        assert got == list(range(B))
    with pytest.raises(ValueError):
        make_shard("head", 0, 3, B, HQ, HKV)      # 3 does not divide Hkv
    with pytest.raises(ValueError):
        make_shard("batch", 0, 3, B, HQ, HKV)     # 3 does not divide B
    with pytest.raises(ValueError):
        make_shard("ring", 0, 2, B, HQ, HKV)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, mode, causal, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = make_shard(mode, rank, world, B, HQ, HKV)
        ql, kl, vl = gen_qkv(B, HQ, HKV, S, S, D, torch.bfloat16, SEED, "cpu",
                             b_slice=sh.b, hq_slice=sh.hq, hkv_slice=sh.hkv)
        o, lse = oracle.attn_full(to_bits(ql), to_bits(kl), to_bits(vl), oracle.ORACLE_BF16,
                                  int(causal), 0.35)
        o_full, lse_full = gather_output(torch.from_numpy(o), torch.from_numpy(lse), sh)
        if rank == 0:
            q.put((o_full.numpy(), lse_full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["head", "batch"])
@pytest.mark.parametrize("causal", [False, True])
def test_sharded_forward_reassembles_bitwise(world, mode, causal):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, mode, causal, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    o_got, lse_got = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    qf, kf, vf = gen_qkv(B, HQ, HKV, S, S, D, torch.bfloat16, SEED, "cpu")
    o_ref, lse_ref = oracle.attn_full(to_bits(qf), to_bits(kf), to_bits(vf), oracle.ORACLE_BF16,
                                      int(causal), 0.35)
    assert o_got.shape == o_ref.shape and lse_got.shape == lse_ref.shape
    assert np.array_equal(o_got, o_ref)
    assert np.array_equal(lse_got, lse_ref)


@pytest.mark.parametrize("mode", ["head", "batch"])
@pytest.mark.parametrize("w", [1, 2, 4])
def test_replica_layout_covers_full_output_once(mode, w):
    """The fused replicated epilogue (tl_attn_fwd_replicated) writes local (b, h) of rank r
    to (b + b_off, h + h_off) of every output: over all ranks each (b, h) of the full
    output is written exactly once, and each local GQA group keeps its kv heads."""
    from paper_2504_17577_b200.dist import replica_layout
    hits = np.zeros((B, HQ), dtype=int)
    for r in range(w):
        sh = make_shard(mode, r, w, B, HQ, HKV)
        Bt, b_off, Ht, h_off = replica_layout(sh, B, HQ)
        assert (Bt, Ht) == (B, HQ)
        Bl, Hl, Hkvl = sh.local_dims(B, HQ, HKV)
        assert b_off == sh.b.start and h_off == sh.hq.start
        hits[b_off:b_off + Bl, h_off:h_off + Hl] += 1
        # the kernel maps local query head h to local kv head h // (Hl / Hkvl); globally
        # that must be the same kv head as h_off + h -> (h_off + h) // (HQ / HKV)
        for h in range(Hl):
            assert sh.hkv.start + h // (Hl // Hkvl) == (h_off + h) // (HQ // HKV)
    assert (hits == 1).all()
