"""Pins for the fp64 oracle (CPU only, `-m "not gpu"`).

The oracle (oracle/attn_oracle.c) is pinned to things other than itself:
hand-derived worked examples (tests/golden/hand_examples.json), closed forms,
invariants, special cases, and an independent brute-force formulation on tiny
shapes. Each test names the passage or identity it checks. A plausible mistake in
the oracle — a dropped term (scale, last key), a wrong sign, a wrong index
(GQA grouping, causal alignment), a transposed operand — fails at least one test.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2504_17577_b200.inputs import from_values, gen_qkv, to_bits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")
DT = {"f16": (torch.float16, oracle.ORACLE_F16), "bf16": (torch.bfloat16, oracle.ORACLE_BF16)}


def bits(values, tdtype, shape):
    return to_bits(from_values(np.asarray(values, np.float64).reshape(shape), tdtype))


def rand_bits(shape, tdtype, seed, lo=-3.0, hi=3.0):
    rng = np.random.default_rng(seed)
    return bits(rng.uniform(lo, hi, size=shape), tdtype, shape)


def widen_arr(a, dt):
    return np.vectorize(lambda x: oracle.widen(int(x), dt))(a).astype(np.float64)


# --------------------------------------------------------------------------- widening
@pytest.mark.parametrize("pattern,expect", [
    (0x3C00, 1.0), (0xC000, -2.0), (0x0001, 2.0 ** -24), (0x0400, 2.0 ** -14),
    (0x7BFF, 65504.0), (0x3555, 0.333251953125), (0x8000, -0.0), (0x7C00, math.inf),
])
def test_widen_f16_bit_patterns(pattern, expect):
    # IEEE 754 binary16 decoding: sign, 5-bit exponent (bias 15), 10-bit mantissa
    assert oracle.widen(pattern, oracle.ORACLE_F16) == expect


@pytest.mark.parametrize("pattern,expect", [
    (0x3F80, 1.0), (0xC0A0, -5.0), (0x0001, 2.0 ** -133), (0x7F7F, 3.3895313892515355e38),
    (0x3EAB, 0.333984375), (0xFF80, -math.inf),
])
def test_widen_bf16_bit_patterns(pattern, expect):
    # bfloat16 = top 16 bits of IEEE binary32
    assert oracle.widen(pattern, oracle.ORACLE_BF16) == expect


def test_widen_matches_torch_on_all_patterns():
    # Every finite 16-bit pattern widens to the value torch assigns to it.
    pats = np.arange(0, 1 << 16, 97, dtype=np.uint16)
    for tdt, dt in DT.values():
        ref = torch.from_numpy(pats.view(np.int16).copy()).view(tdt).to(torch.float64).numpy()
        got = widen_arr(pats, dt)
        fin = np.isfinite(ref)
        np.testing.assert_array_equal(got[fin], ref[fin])


# --------------------------------------------------------------------------- golden
def _eval(expr):
    return float(eval(expr, {"__builtins__": {}}, {"e": math.e, "log": math.log}))


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)["examples"]


@pytest.mark.parametrize("dtname", ["f16", "bf16"])
@pytest.mark.parametrize("ex", _golden(), ids=lambda e: e["name"])
def test_hand_worked_examples(ex, dtname):
    tdt, dt = DT[dtname]
    B, Hq, Hkv, Sq, Skv, D = (ex[k] for k in ("B", "Hq", "Hkv", "Sq", "Skv", "D"))
    q = bits(ex["q"], tdt, (B, Sq, Hq, D))
    k = bits(ex["k"], tdt, (B, Skv, Hkv, D))
    v = bits(ex["v"], tdt, (B, Skv, Hkv, D))
    o, lse = oracle.attn_full(q, k, v, dt, ex["causal"], ex["scale"])
    o_exp = np.array([_eval(s) for s in ex["o"]]).reshape(o.shape)
    lse_exp = np.array([_eval(s) for s in ex["lse"]]).reshape(lse.shape)
    np.testing.assert_allclose(o, o_exp, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(lse, lse_exp, rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------- brute force
CASES = [
    # (B, Hq, Hkv, Sq, Skv, D, causal)
    (1, 1, 1, 7, 7, 5, 0),
    (1, 1, 1, 7, 7, 5, 1),
    (2, 4, 2, 5, 9, 8, 0),
    (2, 4, 2, 5, 9, 8, 1),   # Sq < Skv, causal bottom-right
    (1, 2, 1, 9, 4, 3, 1),   # Sq > Skv: rows 0..4 have no key
    (1, 3, 3, 16, 16, 16, 1),
]


@pytest.mark.parametrize("dtname", ["f16", "bf16"])
@pytest.mark.parametrize("case", CASES)
def test_two_pass_equals_brute_force(case, dtname):
    """Two-pass (max-first) oracle == explicit-matrix P_ij = 1/sum_k exp(s_ik - s_ij)."""
    B, Hq, Hkv, Sq, Skv, D, causal = case
    tdt, dt = DT[dtname]
    q = rand_bits((B, Sq, Hq, D), tdt, 1)
    k = rand_bits((B, Skv, Hkv, D), tdt, 2)
    v = rand_bits((B, Skv, Hkv, D), tdt, 3)
    scale = 1.0 / math.sqrt(D)
    o, lse = oracle.attn_full(q, k, v, dt, causal, scale)
    for b in range(B):
        for h in range(Hq):
            S, P, O, L = oracle.brute_force(q, k, v, dt, causal, scale, b, h)
            np.testing.assert_allclose(o[b, :, h, :], O, rtol=1e-12, atol=1e-12)
            fin = np.isfinite(L)
            np.testing.assert_allclose(lse[b, h][fin], L[fin], rtol=1e-12, atol=1e-12)
            assert np.array_equal(np.isfinite(lse[b, h]), fin)
            # softmax rows sum to 1 (rows with a non-empty key set), else all zero
            rs = P.sum(axis=1)
            np.testing.assert_allclose(rs[fin], 1.0, atol=1e-12)
            assert np.all(rs[~fin] == 0.0)


def test_brute_force_scores_are_q_dot_k_not_transposed():
    """S_ij = scale * q_i . k_j with Sq != Skv and distinct Q/K (catches a Q/K swap)."""
    tdt, dt = DT["bf16"]
    qv = np.arange(1, 7, dtype=np.float64).reshape(1, 3, 1, 2)        # 3 queries
    kv = np.array([1, 0, 0, 1, 1, 1, 2, -1, 0, 0]).reshape(1, 5, 1, 2)  # 5 keys
    q, k = bits(qv, tdt, qv.shape), bits(kv, tdt, kv.shape)
    v = bits(np.zeros((1, 5, 1, 2)), tdt, (1, 5, 1, 2))
    S, _, _, _ = oracle.brute_force(q, k, v, dt, 0, 0.5, 0, 0)
    expect = 0.5 * qv[0, :, 0, :] @ kv[0, :, 0, :].T
    np.testing.assert_array_equal(S, expect)


# --------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("causal", [0, 1])
def test_constant_v_gives_constant_o(causal):
    """V_j == c  ->  O_i = c for every row with a key (softmax weights sum to 1)."""
    tdt, dt = DT["f16"]
    B, Hq, Hkv, Sq, Skv, D = 1, 2, 1, 11, 11, 4
    q = rand_bits((B, Sq, Hq, D), tdt, 5)
    k = rand_bits((B, Skv, Hkv, D), tdt, 6)
    v = bits(np.full((B, Skv, Hkv, D), 1.75), tdt, (B, Skv, Hkv, D))
    o, _ = oracle.attn_full(q, k, v, dt, causal, 0.7)
    np.testing.assert_allclose(o, 1.75, rtol=1e-14)


@pytest.mark.parametrize("causal", [0, 1])
@pytest.mark.parametrize("Sq,Skv", [(6, 6), (5, 8), (8, 5)])
@pytest.mark.parametrize("zero", ["q", "scale"])
def test_equal_scores_give_mean_v_and_log_count(causal, Sq, Skv, zero):
    """All scores equal (Q = 0 or scale = 0): O_i = mean_{j in J_i} V_j, LSE_i = ln|J_i|.

    |J_i| is written out by hand from the bottom-right causal rule j <= i + Skv - Sq
    (R3): e.g. Sq=5, Skv=8 -> |J_i| = i + 4; Sq=8, Skv=5 -> |J_i| = max(0, i - 2).
    """
    tdt, dt = DT["bf16"]
    B, Hq, Hkv, D = 1, 1, 1, 3
    qv = np.zeros((B, Sq, Hq, D)) if zero == "q" else np.random.default_rng(9).integers(-3, 4, (B, Sq, Hq, D))
    q = bits(qv, tdt, qv.shape)
    k = rand_bits((B, Skv, Hkv, D), tdt, 10)
    vv = np.random.default_rng(11).integers(-8, 9, (B, Skv, Hkv, D)).astype(np.float64)
    v = bits(vv, tdt, vv.shape)
    scale = 0.3 if zero == "q" else 0.0
    o, lse = oracle.attn_full(q, k, v, dt, causal, scale)
    hand_counts = {(6, 6): [1, 2, 3, 4, 5, 6], (5, 8): [4, 5, 6, 7, 8], (8, 5): [0, 0, 0, 1, 2, 3, 4, 5]}
    for i in range(Sq):
        n = hand_counts[(Sq, Skv)][i] if causal else Skv
        if n == 0:
            assert lse[0, 0, i] == -math.inf and np.all(o[0, i, 0] == 0.0)
            continue
        np.testing.assert_allclose(lse[0, 0, i], math.log(n), rtol=0, atol=1e-15)
        np.testing.assert_allclose(o[0, i, 0], vv[0, :n, 0].mean(axis=0), rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("dtname", ["f16", "bf16"])
def test_causal_first_row_is_v0(dtname):
    """Causal, Sq == Skv: row 0 sees only key 0 -> O[0] = V[0] exactly, LSE[0] = scale*q0.k0."""
    tdt, dt = DT[dtname]
    B, Hq, Hkv, S, D = 2, 4, 2, 9, 6
    q = rand_bits((B, S, Hq, D), tdt, 12)
    k = rand_bits((B, S, Hkv, D), tdt, 13)
    v = rand_bits((B, S, Hkv, D), tdt, 14)
    scale = 0.4
    o, lse = oracle.attn_full(q, k, v, dt, 1, scale)
    qf, kf, vf = widen_arr(q, dt), widen_arr(k, dt), widen_arr(v, dt)
    for b in range(B):
        for h in range(Hq):
            g = h // (Hq // Hkv)
            assert np.array_equal(o[b, 0, h], vf[b, 0, g])
            assert lse[b, h, 0] == pytest.approx(scale * float(qf[b, 0, h] @ kf[b, 0, g]), abs=1e-14)


def test_single_key_gives_v0():
    """Skv = 1: O = V_0 exactly and LSE = s_0 for every row (non-causal)."""
    tdt, dt = DT["f16"]
    q = rand_bits((1, 5, 2, 4), tdt, 15)
    k = rand_bits((1, 1, 2, 4), tdt, 16)
    v = rand_bits((1, 1, 2, 4), tdt, 17)
    o, lse = oracle.attn_full(q, k, v, dt, 0, 0.5)
    qf, kf, vf = widen_arr(q, dt), widen_arr(k, dt), widen_arr(v, dt)
    for h in range(2):
        assert np.array_equal(o[0, :, h], np.broadcast_to(vf[0, 0, h], (5, 4)))
        np.testing.assert_allclose(lse[0, h], 0.5 * qf[0, :, h] @ kf[0, 0, h], atol=1e-14)


def test_hard_attention_gather():
    """K rows = 64*e_{j mod D} (signed), Q rows = 64*e_{pi(i)}: exp of every non-matching
    key underflows in fp64 relative to the match (gap 4096*scale = 362 nats), so O_i = V_{pi(i)}
    and LSE_i = 4096*scale up to the e^-362 terms."""
    tdt, dt = DT["bf16"]
    D, S = 128, 256
    rng = np.random.default_rng(18)
    kv = np.zeros((1, S, 1, D))
    for j in range(S):
        kv[0, j, 0, j % D] = 64.0 if j < D else -64.0
    perm = rng.permutation(S)
    qv = np.zeros((1, S, 1, D))
    for i in range(S):
        t = perm[i]
        qv[0, i, 0, t % D] = 64.0 if t < D else -64.0
    q, k = bits(qv, tdt, qv.shape), bits(kv, tdt, kv.shape)
    v = rand_bits((1, S, 1, D), tdt, 19)
    scale = 1.0 / math.sqrt(D)
    o, lse = oracle.attn_full(q, k, v, dt, 0, scale)
    vf = widen_arr(v, dt)
    np.testing.assert_allclose(o[0, :, 0], vf[0, perm, 0], rtol=0, atol=1e-150)
    np.testing.assert_allclose(lse[0, 0], 4096.0 * scale, rtol=1e-15)


def test_key_permutation_invariance():
    """Non-causal attention is invariant under a joint permutation of K and V rows."""
    tdt, dt = DT["bf16"]
    q = rand_bits((1, 6, 2, 8), tdt, 20)
    k = rand_bits((1, 13, 2, 8), tdt, 21)
    v = rand_bits((1, 13, 2, 8), tdt, 22)
    perm = np.random.default_rng(23).permutation(13)
    o1, l1 = oracle.attn_full(q, k, v, dt, 0, 0.35)
    o2, l2 = oracle.attn_full(q, np.ascontiguousarray(k[:, perm]), np.ascontiguousarray(v[:, perm]), dt, 0, 0.35)
    np.testing.assert_allclose(o1, o2, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(l1, l2, rtol=1e-13, atol=1e-13)


def test_key_shift_changes_lse_only():
    """Adding u to every key row: O unchanged, LSE_i += scale * q_i . u (softmax shift invariance).
    Integer-valued inputs keep k + u exact in bf16."""
    tdt, dt = DT["bf16"]
    rng = np.random.default_rng(24)
    qv = rng.integers(-3, 4, (1, 5, 1, 4)).astype(np.float64)
    kv = rng.integers(-3, 4, (1, 7, 1, 4)).astype(np.float64)
    u = np.array([1.0, -2.0, 3.0, 0.0])
    q, k, k2 = bits(qv, tdt, qv.shape), bits(kv, tdt, kv.shape), bits(kv + u, tdt, kv.shape)
    v = rand_bits((1, 7, 1, 4), tdt, 25)
    o1, l1 = oracle.attn_full(q, k, v, dt, 0, 0.25)
    o2, l2 = oracle.attn_full(q, k2, v, dt, 0, 0.25)
    np.testing.assert_allclose(o1, o2, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(l2[0, 0], l1[0, 0] + 0.25 * qv[0, :, 0] @ u, rtol=1e-13, atol=1e-12)


def test_linearity_in_v():
    """O(V1 + V2) = O(V1) + O(V2) (integer V keeps the sum exact in fp16)."""
    tdt, dt = DT["f16"]
    rng = np.random.default_rng(26)
    q = rand_bits((1, 4, 1, 4), tdt, 27)
    k = rand_bits((1, 6, 1, 4), tdt, 28)
    v1 = rng.integers(-50, 50, (1, 6, 1, 4)).astype(np.float64)
    v2 = rng.integers(-50, 50, (1, 6, 1, 4)).astype(np.float64)
    oa, _ = oracle.attn_full(q, k, bits(v1, tdt, v1.shape), dt, 1, 0.5)
    ob, _ = oracle.attn_full(q, k, bits(v2, tdt, v2.shape), dt, 1, 0.5)
    oc, _ = oracle.attn_full(q, k, bits(v1 + v2, tdt, v1.shape), dt, 1, 0.5)
    np.testing.assert_allclose(oc, oa + ob, rtol=1e-12, atol=1e-11)


def test_causal_prefix_property():
    """Causal: changing K/V rows j > i + Skv - Sq does not change O_i / LSE_i."""
    tdt, dt = DT["bf16"]
    q = rand_bits((1, 10, 1, 4), tdt, 29)
    k = rand_bits((1, 10, 1, 4), tdt, 30)
    v = rand_bits((1, 10, 1, 4), tdt, 31)
    o1, l1 = oracle.attn_full(q, k, v, dt, 1, 0.5)
    k2, v2 = k.copy(), v.copy()
    k2[:, 6:] = rand_bits((1, 4, 1, 4), tdt, 32)
    v2[:, 6:] = rand_bits((1, 4, 1, 4), tdt, 33)
    o2, l2 = oracle.attn_full(q, k2, v2, dt, 1, 0.5)
    assert np.array_equal(o1[:, :6], o2[:, :6]) and np.array_equal(l1[:, :, :6], l2[:, :, :6])
    assert not np.array_equal(o1[:, 6:], o2[:, 6:])


def test_gqa_equals_mha_with_repeated_kv():
    """Hkv < Hq equals MHA with each KV head repeated Hq/Hkv times (contiguous)."""
    tdt, dt = DT["bf16"]
    q = rand_bits((2, 5, 6, 4), tdt, 34)
    k = rand_bits((2, 7, 2, 4), tdt, 35)
    v = rand_bits((2, 7, 2, 4), tdt, 36)
    o1, l1 = oracle.attn_full(q, k, v, dt, 1, 0.5)
    kr = np.ascontiguousarray(np.repeat(k, 3, axis=2))
    vr = np.ascontiguousarray(np.repeat(v, 3, axis=2))
    o2, l2 = oracle.attn_full(q, kr, vr, dt, 1, 0.5)
    assert np.array_equal(o1, o2) and np.array_equal(l1, l2)


def test_rows_api_matches_full_and_rejects_bad_args():
    tdt, dt = DT["f16"]
    q = rand_bits((1, 9, 2, 4), tdt, 37)
    k = rand_bits((1, 9, 1, 4), tdt, 38)
    v = rand_bits((1, 9, 1, 4), tdt, 39)
    o, lse = oracle.attn_full(q, k, v, dt, 1, 0.5)
    rows = [8, 0, 3]
    orow, lrow = oracle.attn_rows(q, k, v, dt, 1, 0.5, 0, 1, rows)
    assert np.array_equal(orow, o[0, rows, 1]) and np.array_equal(lrow, lse[0, 1, rows])
    with pytest.raises(ValueError):
        oracle.attn_rows(q, k, v, dt, 1, 0.5, 0, 2, [0])          # h out of range
    with pytest.raises(ValueError):
        oracle.attn_rows(q, k, v, dt, 1, 0.5, 0, 0, [9])          # row out of range
    with pytest.raises(ValueError):
        oracle.attn_rows(q, k, v, 7, 1, 0.5, 0, 0, [0])           # bad dtype


def test_parallel_rows_match_serial():
    B, Hq, Hkv, S, D = 1, 2, 1, 33, 16
    q, k, v = (to_bits(t) for t in gen_qkv(B, Hq, Hkv, S, S, D, torch.bfloat16, 7, "cpu"))
    work = [(0, h, list(range(S))) for h in range(Hq)]
    res = oracle.attn_rows_parallel(q, k, v, oracle.ORACLE_BF16, 1, 0.25, work, threads=2)
    for (b, h, rows), (o, l) in zip(work, res):
        o2, l2 = oracle.attn_rows(q, k, v, oracle.ORACLE_BF16, 1, 0.25, b, h, rows)
        assert np.array_equal(o, o2) and np.array_equal(l, l2)
