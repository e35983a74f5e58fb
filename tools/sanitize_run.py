"""Small forward passes for compute-sanitizer (memcheck / racecheck / synccheck):
both kernels (CTA pair at D=128, single CTA at D=64), causal and ragged shapes."""
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
