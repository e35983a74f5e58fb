"""Fused replicated output (include/tlattn.h tl_attn_fwd_replicated,
tl_peer_barrier, tl_ipc_*) on one B200: two processes on the same GPU stand in for two
ranks. Each process maps the other's output buffer through CUDA IPC, runs its head (or
batch) shard with the epilogue storing into BOTH buffers, and after the device-side flag
barrier both processes must hold the full O and LSE, bitwise equal to the unsharded
tl_attn_fwd result (the kernel is deterministic and shard-invariant), AND every rank's full
O and LSE must match the fp64 oracle (rows 0-63, the tile / unit boundaries and the last 16
rows of every (b, h); north_star tolerances). The peer stores here stay on one device; on a
multi-GPU box the same code stores over NVLink."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [
    # B, Hq, Hkv, S, D, dtype, causal, mode
    (2, 4, 2, 384, 128, torch.bfloat16, True, "head"),
    (2, 4, 4, 300, 64, torch.float16, False, "head"),
    (4, 2, 1, 256, 128, torch.bfloat16, False, "batch"),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2504_17577_b200 import attention
    from paper_2504_17577_b200.dist import ReplicatedOutput, make_shard
    from paper_2504_17577_b200.inputs import gen_qkv
    B, Hq, Hkv, S, D, dt, causal, mode = case
    q, k, v = gen_qkv(B, Hq, Hkv, S, S, D, dt, 77, "cuda")
    o_ref, lse_ref = attention(q, k, v, causal=causal)
    sh = make_shard(mode, rank, world, B, Hq, Hkv)
    ql = q[sh.b, :, sh.hq].contiguous()
    kl = k[sh.b, :, sh.hkv].contiguous()
    vl = v[sh.b, :, sh.hkv].contiguous()
    rep = ReplicatedOutput(sh, B, S, Hq, D, dt)
    ok = True
    stats = None
    for it in range(3):  # repeated calls: epochs advance, buffers rewritten in place
        rep.o.fill_(float("nan"))
        rep.lse.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        o, lse = rep(ql, kl, vl, causal=causal)
        torch.cuda.synchronize()
        ok &= torch.equal(o.view(torch.int16), o_ref.view(torch.int16))
        ok &= torch.equal(lse, lse_ref)
        if it == 2:
            # this rank's full replicated O / LSE (its own shard + the peer's epilogue stores)
            # against the fp64 oracle, not only against the CUDA path itself
            from _parity import compare_outputs_with_oracle, sample_rows
            import numpy as np
            rows = sample_rows(S, np.random.default_rng(rank))
            stats = compare_outputs_with_oracle(q, k, v, o, lse, causal, D ** -0.5, rows,
                                                label=f"rank {rank}")
    dist.barrier()
    rep.close()
    results[rank] = (bool(ok), stats)
    dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[7]}-D{c[4]}-{'causal' if c[6] else 'full'}")
def test_two_ranks_one_gpu_replicated_output_bitwise(case):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = dict(results)
    assert sorted(res) == [0, 1]
    for r in (0, 1):
        bitwise, stats = res[r]
        assert bitwise, f"rank {r}: replicated output differs from tl_attn_fwd"
        assert stats is not None and stats["rows_checked"] > 0, stats  # oracle checked


def test_single_rank_replicated_equals_tl_attn_fwd():
    """n_outs = 2 buffers in one process (no IPC): both hold the unsharded result."""
    from paper_2504_17577_b200 import attention, tl_attn_fwd_replicated
    from paper_2504_17577_b200.inputs import gen_qkv
    from paper_2504_17577_b200.tlattn import dtype_code
    B, Hq, Hkv, S, D = 2, 4, 2, 520, 128
    q, k, v = gen_qkv(B, Hq, Hkv, S, S, D, torch.bfloat16, 5, "cuda")
    o_ref, lse_ref = attention(q, k, v, causal=True)
    outs = [torch.full_like(o_ref, float("nan")) for _ in range(2)]
    lses = [torch.full_like(lse_ref, float("nan")) for _ in range(2)]
    tl_attn_fwd_replicated(q, k, v, outs, lses, B, 0, Hq, 0, B, Hq, Hkv, S, S, D, 1,
                           1.0 / D ** 0.5, dtype_code(q.dtype))
    torch.cuda.synchronize()
    for o, l in zip(outs, lses):
        assert torch.equal(o.view(torch.int16), o_ref.view(torch.int16))
        assert torch.equal(l, lse_ref)
    import numpy as np
    from _parity import compare_outputs_with_oracle, sample_rows
    rows = sample_rows(S, np.random.default_rng(0))
    for o, l in zip(outs, lses):  # every output buffer against the fp64 oracle
        compare_outputs_with_oracle(q, k, v, o, l, True, 1.0 / D ** 0.5, rows, label="repl")


def test_eight_outputs_and_no_lse():
    """The maximum fan-out (8 outputs) with lse_outs = NULL, D = 64 kernel, a shard at a
    head offset: only the shard's heads are written, the rest of every buffer is untouched."""
    from paper_2504_17577_b200 import attention, tl_attn_fwd_replicated
    from paper_2504_17577_b200.inputs import gen_qkv
    from paper_2504_17577_b200.tlattn import dtype_code
    B, Hq_total, Hl, Hkvl, S, D = 1, 8, 2, 1, 200, 64
    q, k, v = gen_qkv(B, Hl, Hkvl, S, S, D, torch.float16, 9, "cuda")
    o_ref, _ = attention(q, k, v, causal=False)
    outs = [torch.full((B, S, Hq_total, D), 7.0, dtype=torch.float16, device="cuda") for _ in range(8)]
    tl_attn_fwd_replicated(q, k, v, outs, None, B, 0, Hq_total, 4, B, Hl, Hkvl, S, S, D, 0,
                           1.0 / D ** 0.5, dtype_code(q.dtype))
    torch.cuda.synchronize()
    import numpy as np
    from _parity import compare_outputs_with_oracle
    for o in outs:
        assert torch.equal(o[:, :, 4:6].view(torch.int16), o_ref.view(torch.int16))
        assert (o[:, :, :4] == 7.0).all() and (o[:, :, 6:] == 7.0).all()
        compare_outputs_with_oracle(q, k, v, o[:, :, 4:6].contiguous(), None, False,
                                    1.0 / D ** 0.5, list(range(S)), label="repl8")


def test_replicated_bad_args():
    from paper_2504_17577_b200 import TlAttnError, tl_attn_fwd_replicated
    q = torch.zeros(1, 128, 2, 128, dtype=torch.bfloat16, device="cuda")
    o = torch.zeros(1, 128, 4, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(TlAttnError):  # h_off + Hq > Hq_total
        tl_attn_fwd_replicated(q, q, q, [o], None, 1, 0, 4, 3, 1, 2, 2, 128, 128, 128, 0, 0.1, 1)
    with pytest.raises(TlAttnError):  # too many outputs
        tl_attn_fwd_replicated(q, q, q, [o] * 9, None, 1, 0, 4, 0, 1, 2, 2, 128, 128, 128, 0, 0.1, 1)


def test_replicated_single_cta_after_gemm():
    """Regression: each kernel instantiation sets its dynamic-shared-memory attribute once
    per device; the replicated-output instantiations once shared the GEMM's slots, so a GEMM
    call first left the replicated single-CTA kernel without its attribute."""
    from paper_2504_17577_b200 import attention, gemm, tl_attn_fwd_replicated
    from paper_2504_17577_b200.inputs import gen_qkv
    from paper_2504_17577_b200.tlattn import dtype_code
    a = torch.randn(256, 256, device="cuda").to(torch.bfloat16)
    gemm(a, a)
    from paper_2504_17577_b200.tlattn import TL_OPT_FORCE_1CTA, option
    B, Hq, Hkv, S, D = 1, 2, 1, 300, 128
    q, k, v = gen_qkv(B, Hq, Hkv, S, S, D, torch.bfloat16, 12, "cuda")
    with option(TL_OPT_FORCE_1CTA, 1):
        o_ref, _ = attention(q, k, v, causal=True)
        out = torch.zeros_like(o_ref)
        tl_attn_fwd_replicated(q, k, v, [out], None, B, 0, Hq, 0, B, Hq, Hkv, S, S, D, 1,
                               D ** -0.5, dtype_code(q.dtype))
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), o_ref.view(torch.int16))
