"""Pins for the fp64 MLA decode oracle (oracle/mla_oracle.c), CPU only (`-m "not gpu"`).

What the oracle computes is PAPER.md Appendix B.3, Fig. 18: scores =
Q KV^T + Q_pe K_pe^T, O = softmax(scale * scores) KV (V = KV),
kv head h / (H/Hkv), plus per-batch cache lengths (reading M1).
It is pinned to things other than itself: hand-derived closed forms
(tests/golden/mla_hand_examples.json), an independent explicit-matrix formulation,
special cases (zero queries, one key, no key), and invariances (key permutation, k_pe
shift, prefix property, GQA == repeated MHA, hard-attention gather). A dropped pe term,
a wrong value operand, a wrong GQA index, ignoring seqlens or a missing scale each
fails several of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2504_17577_b200.inputs import from_values, gen_mla, gen_seqlens, to_bits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "mla_hand_examples.json")
DT = {"f16": (torch.float16, oracle.ORACLE_F16), "bf16": (torch.bfloat16, oracle.ORACLE_BF16)}


def bits(values, tdtype, shape):
    return to_bits(from_values(np.asarray(values, np.float64).reshape(shape), tdtype))


def mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, seed):
    return [to_bits(t) for t in gen_mla(B, H, Hkv, Skv, Dl, Dr, tdt, seed, "cpu")]


def _eval(expr):
    return float(eval(expr, {"e": math.e, "log": math.log, "__builtins__": {}}))


@pytest.mark.parametrize("dtn", ["f16", "bf16"])
def test_hand_examples(dtn):
    tdt, dt = DT[dtn]
    ex_all = json.load(open(GOLDEN))["examples"]
    for ex in ex_all:
        B, H, Hkv, Skv, Dl, Dr = (ex[k] for k in ("B", "H", "Hkv", "Skv", "Dl", "Dr"))
        q = bits(ex["q"], tdt, (B, H, Dl))
        qp = bits(ex["q_pe"], tdt, (B, H, Dr))
        kv = bits(ex["kv"], tdt, (B, Skv, Hkv, Dl))
        kp = bits(ex["k_pe"], tdt, (B, Skv, Hkv, Dr))
        o, lse = oracle.mla_decode(q, qp, kv, kp, dt, _eval(ex["scale"]), ex["seqlens"])
        o_exp = np.array([_eval(x) for x in ex["o"]]).reshape(B, H, Dl)
        lse_exp = np.array([_eval(x) for x in ex["lse"]]).reshape(B, H)
        np.testing.assert_allclose(o, o_exp, rtol=1e-13, atol=1e-13, err_msg=ex["name"])
        np.testing.assert_allclose(lse, lse_exp, rtol=1e-13, atol=1e-13, err_msg=ex["name"])


@pytest.mark.parametrize("shape", [
    # B, H, Hkv, Skv, Dl, Dr, seqlens-kind
    (1, 1, 1, 1, 4, 2, None),
    (2, 4, 1, 37, 16, 8, "ragged"),
    (2, 8, 2, 50, 8, 4, None),
    (3, 16, 1, 24, 512, 64, "ragged"),
    (2, 4, 4, 9, 6, 0, None),
])
@pytest.mark.parametrize("dtn", ["f16", "bf16"])
def test_brute_force_agrees(shape, dtn):
    # independent algebra (explicit concatenation, no max subtraction, P KV as a product)
    B, H, Hkv, Skv, Dl, Dr, kind = shape
    tdt, dt = DT[dtn]
    q, qp, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 17 + Skv)
    sl = gen_seqlens(B, Skv, 3) if kind == "ragged" else None
    scale = 1.0 / math.sqrt(Dl + Dr)
    o, lse = oracle.mla_decode(q, qp, kv, kp, dt, scale, sl)
    for b in range(B):
        S, P, O, L = oracle.mla_brute(q, qp, kv, kp, dt, scale, b, sl)
        np.testing.assert_allclose(o[b], O, rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(lse[b], L, rtol=1e-12, atol=1e-12)
        if P.size:
            np.testing.assert_allclose(P.sum(axis=1), 1.0, atol=1e-12)  # softmax rows sum to 1


@pytest.mark.parametrize("dtn", ["f16", "bf16"])
def test_zero_queries_give_mean_of_kv(dtn):
    # q = q_pe = 0: every score is 0 -> uniform weights over the n_b keys:
    # o = mean_{j<n_b} kv_j, lse = log n_b
    tdt, dt = DT[dtn]
    B, H, Hkv, Skv, Dl, Dr = 3, 4, 2, 40, 32, 8
    _, _, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 5)
    q = np.zeros((B, H, Dl), np.uint16)
    qp = np.zeros((B, H, Dr), np.uint16)
    sl = np.array([40, 7, 1], np.int32)
    o, lse = oracle.mla_decode(q, qp, kv, kp, dt, 0.3, sl)
    kvd = np.vectorize(lambda x: oracle.widen(int(x), dt))(kv).astype(np.float64)
    for b in range(B):
        n = sl[b]
        for h in range(H):
            g = h // (H // Hkv)
            np.testing.assert_allclose(o[b, h], kvd[b, :n, g, :].mean(axis=0), rtol=1e-13,
                                       atol=1e-14)
            assert abs(lse[b, h] - math.log(n)) < 1e-13


def test_one_key_and_no_key():
    tdt, dt = DT["bf16"]
    B, H, Hkv, Skv, Dl, Dr = 2, 2, 1, 5, 16, 4
    q, qp, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 8)
    sl = np.array([1, 0], np.int32)
    scale = 0.125
    o, lse = oracle.mla_decode(q, qp, kv, kp, dt, scale, sl)
    w = lambda a: np.vectorize(lambda x: oracle.widen(int(x), dt))(a).astype(np.float64)
    qd, qpd, kvd, kpd = w(q), w(qp), w(kv), w(kp)
    for h in range(H):
        # n_b = 1: o = kv_0 exactly, lse = s_0
        assert np.array_equal(o[0, h], kvd[0, 0, 0])
        s0 = scale * (qd[0, h] @ kvd[0, 0, 0] + qpd[0, h] @ kpd[0, 0, 0])
        assert abs(lse[0, h] - s0) < 1e-13
        # n_b = 0: o = 0, lse = -inf (reading M1 / R4)
        assert np.all(o[1, h] == 0.0) and lse[1, h] == -math.inf


def test_q_pe_zero_makes_k_pe_irrelevant():
    tdt, dt = DT["f16"]
    q, qp, kv, kp = mla_inputs(2, 4, 1, 33, 16, 8, tdt, 11)
    qp0 = np.zeros_like(qp)
    o1, l1 = oracle.mla_decode(q, qp0, kv, kp, dt, 0.2)
    kp2 = mla_inputs(2, 4, 1, 33, 16, 8, tdt, 12)[3]
    o2, l2 = oracle.mla_decode(q, qp0, kv, kp2, dt, 0.2)
    assert np.array_equal(o1, o2) and np.array_equal(l1, l2)
    # ...and with q_pe != 0 the pe term does change the result (it is not dropped)
    o3, _ = oracle.mla_decode(q, qp, kv, kp, dt, 0.2)
    o4, _ = oracle.mla_decode(q, qp, kv, kp2, dt, 0.2)
    assert not np.allclose(o3, o4)


def test_k_pe_shift():
    # adding u to every k_pe row adds scale * q_pe.u to every score of a head:
    # o unchanged, lse += scale * q_pe.u
    tdt, dt = DT["bf16"]
    B, H, Hkv, Skv, Dl, Dr = 1, 3, 1, 20, 8, 4
    q, qp, kv, _ = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 21)
    rng = np.random.default_rng(4)
    kpv = rng.integers(-4, 5, size=(B, Skv, Hkv, Dr)).astype(np.float64)
    u = np.array([1.0, -2.0, 0.5, 3.0])
    kp = bits(kpv, tdt, kpv.shape)
    kps = bits(kpv + u, tdt, kpv.shape)
    scale = 0.25
    o1, l1 = oracle.mla_decode(q, qp, kv, kp, dt, scale)
    o2, l2 = oracle.mla_decode(q, qp, kv, kps, dt, scale)
    qpd = np.vectorize(lambda x: oracle.widen(int(x), dt))(qp).astype(np.float64)
    np.testing.assert_allclose(o2, o1, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(l2, l1 + scale * (qpd[0] @ u)[None, :], atol=1e-11)


def test_key_permutation_invariance():
    tdt, dt = DT["f16"]
    B, H, Hkv, Skv, Dl, Dr = 1, 4, 1, 31, 16, 8
    q, qp, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 31)
    perm = np.random.default_rng(0).permutation(Skv)
    o1, l1 = oracle.mla_decode(q, qp, kv, kp, dt, 0.2)
    o2, l2 = oracle.mla_decode(q, qp, np.ascontiguousarray(kv[:, perm]),
                               np.ascontiguousarray(kp[:, perm]), dt, 0.2)
    np.testing.assert_allclose(o2, o1, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(l2, l1, atol=1e-12)


def test_prefix_property_of_seqlens():
    # keys j >= n_b do not take part: overwriting them changes nothing (bitwise)
    tdt, dt = DT["bf16"]
    B, H, Hkv, Skv, Dl, Dr = 2, 4, 1, 30, 16, 8
    q, qp, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 41)
    sl = np.array([13, 30], np.int32)
    o1, l1 = oracle.mla_decode(q, qp, kv, kp, dt, 0.3, sl)
    kv2, kp2 = kv.copy(), kp.copy()
    kv2[0, 13:] = bits(np.full((17, Hkv, Dl), 50.0), tdt, (17, Hkv, Dl))
    kp2[0, 13:] = bits(np.full((17, Hkv, Dr), -9.0), tdt, (17, Hkv, Dr))
    o2, l2 = oracle.mla_decode(q, qp, kv2, kp2, dt, 0.3, sl)
    assert np.array_equal(o1, o2) and np.array_equal(l1, l2)
    # ...while for the full-length batch the same edit would matter
    o3, _ = oracle.mla_decode(q, qp, kv2, kp2, dt, 0.3, np.array([30, 30], np.int32))
    assert not np.allclose(o3[0], o1[0])


def test_gqa_equals_repeated_mha():
    # Hkv < H equals Hkv = H with kv head g repeated for its H/Hkv query heads (bitwise)
    tdt, dt = DT["bf16"]
    B, H, Hkv, Skv, Dl, Dr = 2, 8, 2, 19, 16, 8
    q, qp, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, tdt, 51)
    o1, l1 = oracle.mla_decode(q, qp, kv, kp, dt, 0.25)
    rep = lambda a: np.ascontiguousarray(np.repeat(a, H // Hkv, axis=2))
    o2, l2 = oracle.mla_decode(q, qp, rep(kv), rep(kp), dt, 0.25)
    assert np.array_equal(o1, o2) and np.array_equal(l1, l2)


def test_hard_attention_gather():
    # q = 64 e_pi (in the first Dl dims), kv_j = 64 e_j in dims < Skv plus noise in dims
    # >= Skv where q is 0: s_j = scale*4096*[j == pi]; with scale = 1/8 every other key is
    # exp(-512) ~ 1e-222 below -> o = kv_pi (to fp64 rounding), lse = 512 + log(1 + ~0)
    tdt, dt = DT["bf16"]
    B, H, Hkv, Skv, Dl, Dr = 1, 4, 1, 24, 64, 8
    rng = np.random.default_rng(7)
    pis = [3, 0, 23, 11]
    qv = np.zeros((B, H, Dl))
    for h, pi in enumerate(pis):
        qv[0, h, pi] = 64.0
    kvv = np.zeros((B, Skv, Hkv, Dl))
    for j in range(Skv):
        kvv[0, j, 0, j] = 64.0
        kvv[0, j, 0, Skv:] = rng.integers(-8, 9, size=Dl - Skv)
    q = bits(qv, tdt, qv.shape)
    qp = np.zeros((B, H, Dr), np.uint16)
    kv = bits(kvv, tdt, kvv.shape)
    kp = bits(rng.integers(-3, 4, size=(B, Skv, Hkv, Dr)), tdt, (B, Skv, Hkv, Dr))
    o, lse = oracle.mla_decode(q, qp, kv, kp, dt, 0.125)
    for h, pi in enumerate(pis):
        np.testing.assert_allclose(o[0, h], kvv[0, pi, 0], rtol=1e-15, atol=1e-150)
        assert abs(lse[0, h] - 512.0) < 1e-12


def test_rejects_bad_arguments():
    tdt, _ = DT["bf16"]
    q, qp, kv, kp = mla_inputs(1, 3, 2, 4, 8, 4, tdt, 1)  # H % Hkv != 0
    with pytest.raises(ValueError):
        oracle.mla_decode(q, qp, kv, kp, 1, 0.1)
    q, qp, kv, kp = mla_inputs(1, 2, 1, 4, 8, 4, tdt, 1)
    with pytest.raises(ValueError):
        oracle.mla_decode(q, qp, kv, kp, 1, 0.1, np.array([5], np.int32))  # n_b > Skv


@pytest.mark.parametrize("ragged", [True, False])
def test_parallel_helper_equals_whole_batch_oracle(ragged):
    """oracle.mla_decode_parallel (per-batch slices on host threads; it produces every MLA
    GPU expected value) must equal the whole-batch oracle.mla_decode exactly — including
    the per-batch seqlens slice (a mis-sliced length or batch index changes the result) —
    for any batch subset in any order, and its batch-0 row must equal the independent
    explicit-matrix form (oracle.mla_brute)."""
    B, H, Hkv, Skv, Dl, Dr = 6, 8, 2, 70, 32, 16
    q, qp, kv, kp = mla_inputs(B, H, Hkv, Skv, Dl, Dr, torch.bfloat16, 31)
    sl = gen_seqlens(B, Skv, 31, lo=0) if ragged else None
    if ragged:
        sl[3] = 0  # an empty cache among the requested batches
        sl[1] = Skv
    scale = 0.17
    o_all, l_all = oracle.mla_decode(q, qp, kv, kp, oracle.ORACLE_BF16, scale, sl)
    subset = [5, 0, 3, 1] if ragged else [2, 4]
    got = oracle.mla_decode_parallel(q, qp, kv, kp, oracle.ORACLE_BF16, scale, sl, batches=subset,
                                     threads=3)
    assert sorted(got) == sorted(subset)
    for b in subset:
        o_b, l_b = got[b]
        assert np.array_equal(o_b, o_all[b]), b
        assert np.array_equal(l_b, l_all[b]), b
    if ragged:
        assert np.all(got[3][0] == 0.0) and np.all(np.isneginf(got[3][1]))
    _, _, o_bf, l_bf = oracle.mla_brute(q, qp, kv, kp, oracle.ORACLE_BF16, scale, subset[1], sl)
    np.testing.assert_allclose(got[subset[1]][0], o_bf, rtol=0, atol=1e-12)
    np.testing.assert_allclose(got[subset[1]][1], l_bf, rtol=0, atol=1e-12)
