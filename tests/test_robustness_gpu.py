"""Robustness on the GPU:

* a device barrier whose peer never arrives times out (status TL_ERR_TIMEOUT) instead of
  hanging the stream;
* the Python binding refuses mismatched outputs / inputs before launching anything
  (the kernels build their tensor maps from the problem sizes);
* ReplicatedOutput refuses a call that does not match its buffers or its shard.
"""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_peer_barrier_with_missing_peer_times_out():
    from paper_2504_17577_b200 import TL_ERR_TIMEOUT, TlAttnError
    from paper_2504_17577_b200.tlattn import (TL_PEER_FLAG_WORDS, tl_peer_barrier,
                                              tl_peer_barrier_check, tl_peer_barrier_set_timeout_ns)
    own = torch.zeros(TL_PEER_FLAG_WORDS, dtype=torch.int32, device="cuda")
    peer = torch.zeros(TL_PEER_FLAG_WORDS, dtype=torch.int32, device="cuda")  # never arrives
    tl_peer_barrier_set_timeout_ns(200_000_000)  # 0.2 s
    try:
        tl_peer_barrier([own.data_ptr(), peer.data_ptr()], 0, 1)
        with pytest.raises(TlAttnError) as ei:
            tl_peer_barrier_check(own.data_ptr())
        assert ei.value.status == TL_ERR_TIMEOUT
        assert int(peer[0].item()) == 1  # our arrival was published to the "peer"
        # a complete barrier (both arrivals present) reports OK
        own.zero_()
        peer.zero_()
        own[1] = 1  # the peer's arrival for epoch 1
        tl_peer_barrier([own.data_ptr(), peer.data_ptr()], 0, 1)
        tl_peer_barrier_check(own.data_ptr())
    finally:
        tl_peer_barrier_set_timeout_ns(10_000_000_000)


def test_attention_rejects_mismatched_outputs():
    from paper_2504_17577_b200 import TlAttnError, attention
    from paper_2504_17577_b200.inputs import gen_qkv
    q, k, v = gen_qkv(1, 2, 1, 256, 256, 128, torch.bfloat16, 1, "cuda")
    with pytest.raises(TlAttnError):  # O too small
        attention(q, k, v, out=torch.empty(1, 128, 2, 128, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(TlAttnError):  # O of another dtype
        attention(q, k, v, out=torch.empty_like(q, dtype=torch.float16))
    with pytest.raises(TlAttnError):  # LSE of the wrong shape
        attention(q, k, v, lse_out=torch.empty(1, 2, 128, dtype=torch.float32, device="cuda"))
    with pytest.raises(TlAttnError):  # K on another device
        attention(q, k.cpu(), v)
    with pytest.raises(TlAttnError):  # non-contiguous output
        attention(q, k, v, out=torch.empty(1, 256, 4, 128, dtype=torch.bfloat16,
                                           device="cuda")[:, :, ::2])


def test_mla_decode_rejects_mismatched_shapes():
    from paper_2504_17577_b200 import TlAttnError, mla_decode
    from paper_2504_17577_b200.inputs import gen_mla
    q, qp, kv, kp = gen_mla(2, 32, 1, 300, 512, 64, torch.bfloat16, 5, "cuda")
    with pytest.raises(TlAttnError):  # k_pe shorter than kv (would be read out of bounds)
        mla_decode(q, qp, kv, kp[:, :200].contiguous())
    with pytest.raises(TlAttnError):  # q_pe of another batch size
        mla_decode(q, qp[:1].contiguous(), kv, kp)
    with pytest.raises(TlAttnError):  # too few seqlens
        mla_decode(q, qp, kv, kp, seqlens=torch.ones(1, dtype=torch.int32, device="cuda"))
    with pytest.raises(TlAttnError):  # output of the wrong shape
        mla_decode(q, qp, kv, kp, out=torch.empty(2, 32, 256, dtype=torch.bfloat16, device="cuda"))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_replicated_output_rejects_mismatched_calls():
    import torch.distributed as dist
    from paper_2504_17577_b200.dist import ReplicatedOutput, make_shard
    from paper_2504_17577_b200.inputs import gen_qkv
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sh = make_shard("head", 0, 1, 1, 4, 2)
        rep = ReplicatedOutput(sh, 1, 256, 4, 128, torch.bfloat16)
        q, k, v = gen_qkv(1, 4, 2, 256, 256, 128, torch.bfloat16, 3, "cuda")
        o, _ = rep(q, k, v, causal=True)  # the matching call works
        rep.check()
        torch.cuda.synchronize()
        assert torch.isfinite(o.float()).all()
        q2, k2, v2 = gen_qkv(1, 4, 2, 384, 384, 128, torch.bfloat16, 3, "cuda")
        with pytest.raises(ValueError):  # Sq differs from the buffers
            rep(q2, k2, v2)
        with pytest.raises(ValueError):  # dtype differs
            rep(q.half(), k.half(), v.half())
        with pytest.raises(ValueError):  # not this rank's shard (2 of 4 heads)
            rep(q[:, :, :2].contiguous(), k[:, :, :1].contiguous(), v[:, :, :1].contiguous())
        rep.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("D,causal", [(128, True), (128, False), (64, True)])
def test_back_to_back_dependent_calls_under_pdl(D, causal):
    """The attention kernels are launched with programmatic dependent launch and trigger
    their dependents right after their prologue, so call i+1 starts while call i still
    runs. A chain where each call's OUTPUT is the next call's Q (and, alternately, its V)
    must equal the same chain with a device synchronisation between the calls, bitwise:
    every global read and write of a kernel happens after its griddepcontrol.wait.
    (A regression check of the launch path: on this part a build without the wait also
    passed it, i.e. the dependent grid did not start reading before the primary's end in
    that run; the wait is what guarantees it.)"""
    from paper_2504_17577_b200 import attention
    from paper_2504_17577_b200.inputs import gen_qkv
    dt = torch.bfloat16 if D == 128 else torch.float16
    q, k, v = gen_qkv(2, 8, 8, 1024, 1024, D, dt, 77, "cuda")

    def chain(sync):
        x, vv = q.clone(), v.clone()
        outs = []
        for i in range(8):
            o, _ = attention(x, k, vv, causal=causal)
            if sync:
                torch.cuda.synchronize()
            if i % 2 == 0:
                x = o   # next call reads this call's output as Q
            else:
                vv = o  # ... or as V
            outs.append(o)
        torch.cuda.synchronize()
        return outs

    got = chain(False)
    ref = chain(True)
    for a, b in zip(got, ref):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
