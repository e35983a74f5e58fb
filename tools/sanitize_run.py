"""Small forward passes for compute-sanitizer (memcheck / racecheck / synccheck):
both attention kernels (CTA pair at D=128, single CTA at D=64), causal and ragged shapes
(small causal problems take the LPT unit order), the short-sequence pair mode, the
replicated-output epilogue (two outputs in one process), and MLA decode (32- and 64-head
tiles, split + merge)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_17577_b200 import attention
from paper_2504_17577_b200.inputs import gen_qkv

for (B, Hq, Hkv, Sq, Skv, D, dt, causal) in [(1, 2, 1, 300, 300, 128, torch.bfloat16, True),
                                            (1, 1, 1, 600, 600, 128, torch.bfloat16, False),
                                            (1, 2, 2, 300, 200, 64, torch.float16, True)]:
    q, k, v = gen_qkv(B, Hq, Hkv, Sq, Skv, D, dt, 5, "cuda")
    o, l = attention(q, k, v, causal=causal)
    torch.cuda.synchronize()
    print(B, Hq, Hkv, Sq, Skv, D, causal, float(o.float().abs().sum()), bool(torch.isfinite(l[l > -1e30]).all()))

os.environ["TLATTN_UNIT_TILES"] = "1"
q, k, v = gen_qkv(1, 2, 1, 300, 300, 128, torch.bfloat16, 6, "cuda")
o, l = attention(q, k, v, causal=True)
torch.cuda.synchronize()
print("unit_tiles=1", float(o.float().abs().sum()))
del os.environ["TLATTN_UNIT_TILES"]

from paper_2504_17577_b200 import tl_attn_fwd_replicated  # noqa: E402
from paper_2504_17577_b200.tlattn import dtype_code  # noqa: E402
for D, dt in ((128, torch.bfloat16), (64, torch.float16)):
    q, k, v = gen_qkv(1, 2, 1, 300, 300, D, dt, 7, "cuda")
    outs = [torch.zeros(1, 300, 4, D, dtype=dt, device="cuda") for _ in range(2)]
    lses = [torch.zeros(1, 4, 300, dtype=torch.float32, device="cuda") for _ in range(2)]
    tl_attn_fwd_replicated(q, k, v, outs, lses, 1, 0, 4, 2, 1, 2, 1, 300, 300, D, 1, D ** -0.5,
                           dtype_code(dt))
    torch.cuda.synchronize()
    print("replicated", D, float(outs[0].float().abs().sum()), float(outs[1].float().abs().sum()))

from paper_2504_17577_b200 import mla_decode  # noqa: E402
from paper_2504_17577_b200.inputs import gen_mla  # noqa: E402
for (B, H, Skv) in [(2, 32, 700), (2, 128, 700)]:
    qm, qp, kv, kp = gen_mla(B, H, 1, Skv, 512, 64, torch.bfloat16, 9, "cuda")
    sl = torch.tensor([700, 333], dtype=torch.int32, device="cuda")
    om, lm = mla_decode(qm, qp, kv, kp, seqlens=sl)
    torch.cuda.synchronize()
    print("mla", B, H, Skv, float(om.float().abs().sum()), bool(torch.isfinite(lm).all()))
