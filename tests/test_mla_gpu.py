"""GPU parity for tl_mla_decode (Fig. 18) against the fp64 MLA
oracle, element by element, through the C ABI.

Small shapes are checked on every (b, h) and every output element; they cover ragged
cache lengths (tails inside a 128-key block, n_b = 0 and 1), GQA (Hkv > 1), head counts
that are not a multiple of the 32-head tile, batches split across several CTAs
(split-KV pieces merged by the combine kernel) and whole batches written directly. The
full-size MLA configs (configs.py) are checked on sampled batches in the bench's launch
configuration. Tolerances: the north_star bar (tests/_parity.py).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2504_17577_b200 import mla_decode, tl_attn_last_launch_count
from paper_2504_17577_b200.configs import MLA_CONFIGS
from paper_2504_17577_b200.inputs import from_values, gen_mla, gen_seqlens, to_bits

from _parity import compare, odt

pytestmark = pytest.mark.gpu

BF, F16 = torch.bfloat16, torch.float16
DL, DR = 512, 64


def run_and_check(B, H, Hkv, Skv, dtype, seqlens=None, scale=None, seed=7, batches=None,
                  label=""):
    q, qp, kv, kp = gen_mla(B, H, Hkv, Skv, DL, DR, dtype, seed, "cuda")
    scale = 1.0 / math.sqrt(DL + DR) if scale is None else scale
    sl_dev = None if seqlens is None else torch.as_tensor(seqlens, dtype=torch.int32, device="cuda")
    o, lse = mla_decode(q, qp, kv, kp, seqlens=sl_dev, scale=scale)
    torch.cuda.synchronize()
    assert tl_attn_last_launch_count() == 3
    bits = [to_bits(t) for t in (q, qp, kv, kp)]
    res = oracle.mla_decode_parallel(*bits, odt(dtype), scale, seqlens, batches)
    bs = sorted(res)
    o_ref = np.concatenate([res[b][0] for b in bs])
    l_ref = np.concatenate([res[b][1] for b in bs])
    idx = torch.tensor(bs, device="cuda")
    og = o[idx].reshape(-1, DL).double().cpu().numpy()
    lg = lse[idx].reshape(-1).double().cpu().numpy()
    return compare(og, lg, o_ref, l_ref, label), (o, lse)


@pytest.mark.parametrize("B,H,Hkv,Skv,dtype,kind", [
    (1, 16, 1, 128, BF, None),          # one block, 16 of 32 heads valid
    (1, 32, 1, 130, F16, None),         # ragged tail (2 keys in block 2)
    (2, 128, 1, 300, BF, "ragged"),     # 4 head tiles, ragged lengths
    (3, 64, 2, 1000, BF, "ragged"),     # GQA Hkv=2 (two kv heads)
    (1, 128, 1, 4096, BF, None),        # one batch split over many CTAs (combine)
    (4, 40, 1, 777, F16, "ragged"),     # 40 heads: a full and a partial head tile
    (5, 128, 1, 2048, F16, "edge"),     # n_b in {0, 1, 127, 128, 129}
    (16, 16, 1, 1024, BF, "ragged"),    # TP8-style head count
    (2, 96, 1, 600, F16, "ragged"),     # 64-head tiles: one full, one with 32 valid heads
    (3, 256, 2, 700, BF, "ragged"),     # 64-head tiles, GQA (2 kv heads x 2 tiles)
])
def test_mla_parity_small(B, H, Hkv, Skv, dtype, kind):
    if kind == "ragged":
        sl = gen_seqlens(B, Skv, 11 + B)
    elif kind == "edge":
        sl = np.array([0, 1, 127, 128, 129][:B], np.int32)
    else:
        sl = None
    stats, _ = run_and_check(B, H, Hkv, Skv, dtype, sl, label=f"mla {B}x{H}x{Hkv}x{Skv}")
    print(stats)


@pytest.mark.parametrize("scale", [0.0, -0.05, 0.3])
def test_mla_scale_values(scale):
    # scale = 0: uniform weights (O = mean of kv, LSE = ln n); negative: Qhat negated in the
    # instruction descriptor; 0.3: sharp softmax (rescales across blocks)
    run_and_check(2, 64, 1, 700, BF, gen_seqlens(2, 700, 5), scale=scale, label=f"scale {scale}")


@pytest.mark.parametrize("hc", ["32", "64"])
def test_mla_head_tile_widths_agree(hc):
    # the same problem through 32-head and 64-head tiles (TL_OPT_MLA_HC)
    from paper_2504_17577_b200.tlattn import TL_OPT_MLA_HC, option
    with option(TL_OPT_MLA_HC, int(hc)):
        run_and_check(2, 128, 1, 900, BF, gen_seqlens(2, 900, 8), label=f"HC={hc}")


def test_mla_deterministic_and_zero_length():
    B, H, Skv = 3, 128, 1500
    sl = np.array([1500, 0, 700], np.int32)
    q, qp, kv, kp = gen_mla(B, H, 1, Skv, DL, DR, BF, 3, "cuda")
    sld = torch.as_tensor(sl, device="cuda")
    o1, l1 = mla_decode(q, qp, kv, kp, seqlens=sld)
    o2, l2 = mla_decode(q, qp, kv, kp, seqlens=sld)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)  # no atomics: bitwise repeatable
    assert torch.all(o1[1] == 0) and torch.all(torch.isneginf(l1[1]))


def test_mla_hard_attention_gather_bitwise():
    # q = 64 e_pi, kv_j = 64 e_(j mod 512) (+ values in dims the query does not see):
    # s_pi - s_other = 4096 * scale = 170.7 nats -> exp2 underflows to 0 for every other
    # key, so o = kv_pi exactly (bitwise) and lse = 4096 * scale, across block / split
    # boundaries (pi in late blocks).
    B, H, Skv = 2, 32, 1024
    rng = np.random.default_rng(0)
    pis = rng.integers(0, 512, size=(B, H))
    qv = np.zeros((B, H, DL), np.float32)
    for b in range(B):
        for h in range(H):
            qv[b, h, pis[b, h]] = 64.0
    kvv = np.zeros((B, Skv, 1, DL), np.float32)
    for j in range(Skv):
        kvv[:, j, 0, j % 512] = 64.0
    # make keys j >= 512 lose: shift their one-hot to a dim the query ignores is not
    # possible (every dim may be queried), so give them a negative pe score instead
    qpv = np.ones((B, H, DR), np.float32)
    kpv = np.zeros((B, Skv, 1, DR), np.float32)
    kpv[:, 512:, 0, :] = -8.0  # s_j -= 512 * scale for the second copy
    q = from_values(qv, BF, "cuda")
    qp = from_values(qpv, BF, "cuda")
    kv = from_values(kvv, BF, "cuda")
    kp = from_values(kpv, BF, "cuda")
    scale = 1.0 / math.sqrt(DL + DR)
    o, lse = mla_decode(q, qp, kv, kp, scale=scale)
    torch.cuda.synchronize()
    for b in range(B):
        for h in range(H):
            assert torch.equal(o[b, h], kv[b, pis[b, h], 0]), (b, h)
    np.testing.assert_allclose(lse.cpu().numpy(), 4096 * scale, atol=1e-3)


def test_mla_cuda_graph_capture():
    # three launches, caller-provided workspace, no allocation or sync: graph-capturable
    from paper_2504_17577_b200 import tl_mla_decode_workspace_bytes
    B, H, Skv = 4, 128, 1000
    q, qp, kv, kp = gen_mla(B, H, 1, Skv, DL, DR, BF, 12, "cuda")
    sl = torch.as_tensor(gen_seqlens(B, Skv, 2), device="cuda")
    ws = torch.empty(tl_mla_decode_workspace_bytes(B, H, 1), dtype=torch.uint8, device="cuda")
    o = torch.empty((B, H, DL), dtype=BF, device="cuda")
    lse = torch.empty((B, H), dtype=torch.float32, device="cuda")
    ref_o, ref_l = mla_decode(q, qp, kv, kp, seqlens=sl)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        mla_decode(q, qp, kv, kp, seqlens=sl, out=o, lse_out=lse, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mla_decode(q, qp, kv, kp, seqlens=sl, out=o, lse_out=lse, workspace=ws)
    o.zero_()
    lse.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o, ref_o) and torch.equal(lse, ref_l)


@pytest.mark.parametrize("name", [c.name for c in MLA_CONFIGS])
def test_mla_configs_sampled(name):
    # full-size configs in the bench's launch configuration, sampled batches
    cfg = next(c for c in MLA_CONFIGS if c.name == name)
    sl = cfg.seqlens()
    rng = np.random.default_rng(1)
    nb = min(cfg.B, 6)
    batches = sorted(set([0, cfg.B - 1] + [int(x) for x in rng.integers(0, cfg.B, nb)]))
    stats, _ = run_and_check(cfg.B, cfg.H, cfg.Hkv, cfg.Skv, cfg.torch_dtype, sl,
                             seed=cfg.seed, batches=batches, label=name)
    print(name, stats)
