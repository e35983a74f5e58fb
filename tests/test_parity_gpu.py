"""GPU parity: libtlattn (through the C ABI) vs the fp64 oracle, element by element.

Small shapes are checked on every row; they span several 128-row tiles / 256-row
units and ragged tails. Structured inputs pin masking, rescaling and GQA bitwise.
The full BASELINE configs are in test_configs_gpu.py.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2504_17577_b200 import attention, tl_attn_last_launch_count
from paper_2504_17577_b200.inputs import from_values, to_bits

from _parity import check_against_oracle, default_scale, gen, odt

pytestmark = pytest.mark.gpu

BF, F16 = torch.bfloat16, torch.float16


@pytest.mark.parametrize("B,Hq,Hkv,Sq,Skv,D,dtype,causal", [
    (1, 1, 1, 128, 128, 64, F16, False),      # C1 shape
    (1, 1, 1, 128, 128, 64, F16, True),
    (2, 4, 2, 300, 300, 128, BF, False),      # ragged tails, 2 units, GQA
    (2, 4, 2, 300, 300, 128, BF, True),
    (1, 2, 1, 1000, 1000, 64, F16, True),     # ragged, many blocks
    (1, 2, 2, 1000, 1000, 64, BF, False),
    (1, 3, 3, 640, 640, 128, F16, True),
    (1, 2, 1, 200, 520, 128, BF, True),       # Sq < Skv, causal bottom-right
    (1, 2, 1, 520, 200, 128, BF, True),       # Sq > Skv: leading rows have no key
    (1, 2, 1, 520, 200, 64, F16, False),
    (2, 2, 2, 1, 1, 128, BF, False),          # single element
    (1, 2, 2, 1, 777, 64, F16, True),         # one query row
    (1, 1, 1, 129, 1, 128, BF, False),        # one key
    (1, 4, 4, 257, 257, 128, BF, True),
])
def test_parity_small(B, Hq, Hkv, Sq, Skv, D, dtype, causal):
    q, k, v = gen(B, Hq, Hkv, Sq, Skv, D, dtype, 7 + Sq + Skv)
    stats, _ = check_against_oracle(q, k, v, causal, default_scale(D),
                                    label=f"B{B} H{Hq}/{Hkv} S{Sq}x{Skv} D{D} {dtype} c{causal}")
    assert tl_attn_last_launch_count() == 1
    print(stats)


@pytest.mark.parametrize("B,Hq,Hkv,Sq,Skv,causal", [
    (1, 32, 32, 512, 512, True),     # Table 3 FA0 shape (the mode's own trigger)
    (1, 32, 32, 512, 512, False),    # Table 3 FA1 shape
    (2, 4, 2, 300, 300, True),       # ragged, GQA
    (1, 3, 1, 700, 900, True),       # Sq < Skv, ragged, odd unit count
    (1, 2, 2, 900, 600, False),      # Sq > Skv
    # several units per CTA pair, so both slots of the pair run tiles (the one-tile units
    # of the short-sequence mode go to the slot that is ahead; causal 512-row units give
    # the longer tile to it, slot_assign)
    (4, 32, 8, 512, 512, True),
    (2, 16, 16, 768, 640, False),
])
@pytest.mark.parametrize("tiles", ["1", "2"])
def test_pair_kernel_unit_modes(B, Hq, Hkv, Sq, Skv, causal, tiles):
    """CTA-pair kernel with 512-row units (2 tiles) and the short-sequence 256-row units
    (TL_OPT_UNIT_TILES forces the mode): same parity bar on every row."""
    from paper_2504_17577_b200.tlattn import TL_OPT_UNIT_TILES, option, tl_attn_get_option
    q, k, v = gen(B, Hq, Hkv, Sq, Skv, 128, BF, 5 + Sq)
    with option(TL_OPT_UNIT_TILES, int(tiles)):
        assert tl_attn_get_option(TL_OPT_UNIT_TILES) == int(tiles)
        check_against_oracle(q, k, v, causal, default_scale(128),
                             label=f"tiles={tiles} B{B} H{Hq}/{Hkv} S{Sq}x{Skv} c{causal}")


@pytest.mark.parametrize("scale", [0.0, -0.125, 0.37])
def test_scale_values(scale):
    """scale is used literally: 0 (uniform attention) and negative values are legal."""
    q, k, v = gen(1, 2, 1, 384, 384, 128, BF, 11)
    check_against_oracle(q, k, v, True, scale, label=f"scale={scale}")


@pytest.mark.parametrize("D,dtype", [(64, F16), (128, BF)])
def test_causal_row0_is_v0_bitwise(D, dtype):
    """Causal, Sq == Skv: row 0 attends only key 0: p = exp2(0) = 1, l = 1 -> O[0] == V[0]
    bitwise and LSE[0] == scale * q0.k0."""
    q, k, v = gen(2, 4, 2, 512, 512, D, dtype, 21)
    o, lse = attention(q, k, v, causal=True)
    torch.cuda.synchronize()
    for h in range(4):
        assert torch.equal(o[:, 0, h], v[:, 0, h // 2])
    s00 = (q[:, 0].float() * k[:, 0].float().repeat_interleave(2, dim=1)).sum(-1) / math.sqrt(D)
    torch.testing.assert_close(lse[:, :, 0], s00, atol=1e-4, rtol=1e-5)


def test_hard_attention_gather_bitwise():
    """K rows = +-64 e_{j mod D}, Q rows = +-64 e_{pi(i)}, D=128, S=256, scale=1/sqrt(D):
    the score gap 4096*c (522 in log2 units) underflows every non-matching exp2 to 0,
    so O_i == V_{pi(i)} bitwise and LSE_i = 4096*scale. Matches in block 1 exercise the
    running-max rescale with alpha = 0."""
    D, S = 128, 256
    kv = np.zeros((1, S, 1, D), np.float32)
    for j in range(S):
        kv[0, j, 0, j % D] = 64.0 if j < D else -64.0
    perm = np.random.default_rng(5).permutation(S)
    qv = np.zeros((1, S, 1, D), np.float32)
    for i in range(S):
        qv[0, i, 0, perm[i] % D] = 64.0 if perm[i] < D else -64.0
    q = from_values(qv, BF, "cuda")
    k = from_values(kv, BF, "cuda")
    _, _, v = gen(1, 1, 1, S, S, D, BF, 6)
    o, lse = attention(q, k, v, causal=False)
    torch.cuda.synchronize()
    assert torch.equal(o[0, :, 0], v[0, perm, 0])
    torch.testing.assert_close(lse[0, 0], torch.full((S,), 4096.0 / math.sqrt(D), device="cuda"),
                               atol=1e-3, rtol=0)


@pytest.mark.parametrize("causal", [False, True])
def test_gqa_equals_repeated_mha_bitwise(causal):
    """Hkv < Hq gives exactly the result of MHA with K/V heads repeated."""
    q, k, v = gen(2, 8, 2, 384, 384, 128, BF, 31)
    o1, l1 = attention(q, k, v, causal=causal)
    kr = k.repeat_interleave(4, dim=2).contiguous()
    vr = v.repeat_interleave(4, dim=2).contiguous()
    o2, l2 = attention(q, kr, vr, causal=causal)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("causal", [False, True])
def test_equal_scores_give_mean_v(causal):
    """Q = 0: all allowed scores are 0 -> O_i = mean of V over J_i, LSE_i = ln|J_i|."""
    Sq = Skv = 300
    q = torch.zeros(1, Sq, 2, 64, dtype=F16, device="cuda")
    _, k, v = gen(1, 2, 2, Sq, Skv, 64, F16, 41)
    o, lse = attention(q, k, v, causal=causal)
    torch.cuda.synchronize()
    cnt = torch.arange(1, Sq + 1, device="cuda", dtype=torch.float64) if causal else \
        torch.full((Sq,), float(Skv), device="cuda", dtype=torch.float64)
    vf = v.double()
    ref = (vf.cumsum(1) / cnt[None, :, None, None]) if causal else vf.mean(1, keepdim=True).expand_as(vf)
    torch.testing.assert_close(o.double(), ref, atol=2e-3, rtol=2e-3)
    torch.testing.assert_close(lse.double(), cnt.log()[None, None, :].expand(1, 2, Sq), atol=1e-5, rtol=0)


def test_deterministic():
    q, k, v = gen(2, 4, 4, 700, 700, 128, BF, 51)
    o1, l1 = attention(q, k, v, causal=True)
    o2, l2 = attention(q, k, v, causal=True)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_lse_optional_and_stream_ordered():
    q, k, v = gen(1, 2, 2, 256, 256, 64, F16, 61)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        o = attention(q, k, v, causal=True, return_lse=False)
    s.synchronize()
    o2, _ = attention(q, k, v, causal=True)
    torch.cuda.synchronize()
    assert torch.equal(o, o2)


def test_host_entry_matches_device_entry():
    """tl_attn_fwd_host (host buffers, chunked H2D/compute/D2H) == tl_attn_fwd."""
    from paper_2504_17577_b200 import HostAttention
    B, Hq, Hkv, S, D = 5, 4, 2, 384, 128
    q, k, v = gen(B, Hq, Hkv, S, S, D, BF, 71)
    o_ref, l_ref = attention(q, k, v, causal=True)
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    lh = torch.empty((B, Hq, S), dtype=torch.float32).pin_memory()
    ha = HostAttention(B, Hq, Hkv, S, S, D, with_lse=True)
    ha(qh, kh, vh, oh, lh, causal=True)
    torch.cuda.synchronize()
    assert torch.equal(oh, o_ref.cpu()) and torch.equal(lh, l_ref.cpu())
    assert tl_attn_last_launch_count() >= 1


def test_bad_args_raise_before_launch():
    from paper_2504_17577_b200 import TlAttnError, tl_attn_fwd
    q, k, v = gen(1, 2, 2, 128, 128, 96, BF, 1)  # D=96 unsupported
    o = torch.empty_like(q)
    with pytest.raises(TlAttnError) as e:
        tl_attn_fwd(q, k, v, o, None, 1, 2, 2, 128, 128, 96, 0, 0.1, 1)
    assert e.value.status == 2
    _ = oracle, odt, to_bits  # imported for parity with the other GPU test modules


@pytest.mark.parametrize("mode", ["head", "batch"])
def test_shards_equal_unsharded_slices_bitwise(mode):
    """Multi-GPU partition (run here as successive shards on one GPU): every rank's
    tl_attn_fwd over its shard, generated from global indices, equals the matching slice
    of the unsharded output bitwise (deterministic kernel, no cross-unit reduction)."""
    from paper_2504_17577_b200.dist import make_shard
    from paper_2504_17577_b200.inputs import gen_qkv
    Bz, Hq, Hkv, S, D = 4, 8, 4, 640, 128
    q, k, v = gen_qkv(Bz, Hq, Hkv, S, S, D, BF, 77, "cuda")
    o_full, l_full = attention(q, k, v, causal=True)
    for r in range(4):
        sh = make_shard(mode, r, 4, Bz, Hq, Hkv)
        ql, kl, vl = gen_qkv(Bz, Hq, Hkv, S, S, D, BF, 77, "cuda", b_slice=sh.b, hq_slice=sh.hq,
                             hkv_slice=sh.hkv)
        o, l = attention(ql, kl, vl, causal=True)
        torch.cuda.synchronize()
        assert torch.equal(o, o_full[sh.b, :, sh.hq]) and torch.equal(l, l_full[sh.b, sh.hq])


@pytest.mark.parametrize("causal", [False, True])
def test_single_cta_kernel_at_d128(causal):
    """D=128 normally runs on CTA pairs; the single-CTA kernel (TL_OPT_FORCE_1CTA) stays
    correct too, and both kernels agree within rounding."""
    from paper_2504_17577_b200.tlattn import TL_OPT_FORCE_1CTA, option
    q, k, v = gen(2, 4, 2, 700, 700, 128, BF, 91)
    o2, l2 = attention(q, k, v, causal=causal)
    with option(TL_OPT_FORCE_1CTA, 1):
        check_against_oracle(q, k, v, causal, default_scale(128), label="1cta")
        o1, l1 = attention(q, k, v, causal=causal)
    torch.cuda.synchronize()
    assert (o1.float() - o2.float()).abs().max().item() < 2e-2
    assert (l1 - l2).abs().max().item() < 1e-4


@pytest.mark.parametrize("B,Hq,Hkv,S,D,dtype,causal", [
    (2, 4, 2, 520, 128, F16, True),    # fp16 on the CTA-pair kernel
    (2, 4, 4, 520, 64, BF, True),      # bf16 on the single-CTA D=64 kernel
    (1, 8, 1, 777, 128, BF, False),    # MQA, ragged
])
def test_parity_dtype_kernel_matrix(B, Hq, Hkv, S, D, dtype, causal):
    q, k, v = gen(B, Hq, Hkv, S, S, D, dtype, 101 + S)
    check_against_oracle(q, k, v, causal, default_scale(D), label=f"{dtype} D{D}")


def test_cuda_graph_capture_replays_identically():
    """tl_attn_fwd allocates nothing and never syncs, so it is graph-capturable; replays
    reproduce the eager result bitwise."""
    q, k, v = gen(2, 4, 2, 512, 512, 128, BF, 111)
    o_ref, l_ref = attention(q, k, v, causal=True)
    o = torch.empty_like(q)
    lse = torch.empty_like(l_ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        attention(q, k, v, causal=True, out=o, lse_out=lse)  # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        attention(q, k, v, causal=True, out=o, lse_out=lse)
    o.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o, o_ref) and torch.equal(lse, l_ref)


def test_concurrent_streams():
    """Two independent problems on two streams at once give the same results as serially."""
    a = gen(1, 4, 4, 640, 640, 128, BF, 121)
    b = gen(2, 2, 2, 384, 384, 64, F16, 122)
    ra = attention(*a, causal=True)
    rb = attention(*b, causal=False)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        oa = attention(*a, causal=True)
    with torch.cuda.stream(s2):
        ob = attention(*b, causal=False)
    torch.cuda.synchronize()
    assert torch.equal(oa[0], ra[0]) and torch.equal(ob[0], rb[0])


@pytest.mark.parametrize("D,dtype", [(128, BF), (64, F16)])
def test_unit_order_does_not_change_results(D, dtype):
    """The LPT (query-block-major) and the (b, h)-major unit orders schedule the same
    units differently over persistent CTAs that each run several units; every unit's
    arithmetic is the same, so O and LSE must be bitwise equal. Both orders are also
    checked against the oracle on sampled rows."""
    from _parity import sample_rows
    B, Hq, Hkv, S = 4, 16, 4, 2048  # 256 pair units / 512 single-CTA units: several per CTA
    q, k, v = gen(B, Hq, Hkv, S, S, D, dtype, 303 + D)
    outs = {}
    from paper_2504_17577_b200.tlattn import TL_OPT_LPT, option
    for order in ("0", "1"):
        with option(TL_OPT_LPT, int(order)):
            outs[order] = attention(q, k, v, causal=True)
    torch.cuda.synchronize()
    assert torch.equal(outs["0"][0].view(torch.int16), outs["1"][0].view(torch.int16))
    assert torch.equal(outs["0"][1], outs["1"][1])
    rows = sample_rows(S, np.random.default_rng(D), extra=64)
    check_against_oracle(q, k, v, True, default_scale(D), rows_per_head=rows,
                         label=f"LPT D{D}", full_rows_heads=((0, 0),))


def _fuzz_cases(n=40, seed=2504):
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        D = int(rng.choice([64, 128]))
        dtype = [BF, F16][int(rng.integers(2))]
        Hkv = int(rng.choice([1, 2, 3]))
        Hq = Hkv * int(rng.choice([1, 2, 4]))
        B = int(rng.integers(1, 4))
        Sq = int(rng.integers(1, 1300))
        Skv = Sq if rng.random() < 0.5 else int(rng.integers(1, 1300))
        causal = bool(rng.random() < 0.6)
        cases.append((B, Hq, Hkv, Sq, Skv, D, dtype, causal))
    return cases


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: "B{}H{}/{}S{}x{}D{}{}{}".format(
    c[0], c[1], c[2], c[3], c[4], c[5], "bf" if c[6] == BF else "h", "c" if c[7] else ""))
def test_parity_fuzz(case):
    """Seeded random shapes (batch, GQA ratio, ragged Sq / Skv, Sq != Skv, D, dtype, causal):
    every element against the oracle, through whichever kernel, unit mode and unit order the
    launcher picks for the shape."""
    B, Hq, Hkv, Sq, Skv, D, dtype, causal = case
    q, k, v = gen(B, Hq, Hkv, Sq, Skv, D, dtype, 9000 + Sq * 7 + Skv)
    check_against_oracle(q, k, v, causal, default_scale(D), label=str(case))


def _fuzz_many_units(n=12, seed=4017):
    """Shapes with several 512-row units per CTA pair (so both tile slots of a pair move
    through many units, the longer causal tile alternating between them) and ragged or
    offset causal geometry (Sq != Skv: units whose first tile sees no key at all)."""
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        Hkv = int(rng.choice([2, 4, 8]))
        Hq = Hkv * int(rng.choice([1, 2, 4]))
        B = int(rng.integers(2, 9))
        Sq = int(rng.integers(300, 2600))
        Skv = Sq if rng.random() < 0.5 else int(rng.integers(200, 2600))
        causal = bool(rng.random() < 0.7)
        cases.append((B, Hq, Hkv, Sq, Skv, causal))
    return cases


@pytest.mark.parametrize("case", _fuzz_many_units(), ids=lambda c: "B{}H{}/{}S{}x{}{}".format(
    c[0], c[1], c[2], c[3], c[4], "c" if c[5] else ""))
def test_parity_fuzz_many_units(case):
    """CTA-pair kernel (D = 128) with many units per pair: sampled rows of every head (the
    first 64, every unit / tile boundary, the last 16) against the oracle."""
    B, Hq, Hkv, Sq, Skv, causal = case
    q, k, v = gen(B, Hq, Hkv, Sq, Skv, 128, BF, 7000 + Sq * 3 + Skv)
    rows = sorted(set(list(range(min(64, Sq))) +
                      [r for t in range(0, Sq, 128) for r in (t, t + 127) if r < Sq] +
                      list(range(max(0, Sq - 16), Sq))))
    check_against_oracle(q, k, v, causal, default_scale(128), rows_per_head=rows,
                         label=str(case))
