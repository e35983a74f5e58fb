"""One tl_attn_fwd call on an arbitrary shape, checked against the fp64 oracle on all rows
(debugging aid).  python tools/run_shape.py B Hq Hkv Sq Skv D causal [unit_tiles]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402
from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402
B, Hq, Hkv, Sq, Skv, D, causal = (int(x) for x in sys.argv[1:8])
if len(sys.argv) > 8:
    from paper_2504_17577_b200.tlattn import TL_OPT_UNIT_TILES, tl_attn_set_option
    tl_attn_set_option(TL_OPT_UNIT_TILES, int(sys.argv[8]))
dt = torch.bfloat16 if D == 128 else torch.float16
q, k, v = gen_qkv(B, Hq, Hkv, Sq, Skv, D, dt, 5 + Sq, "cuda")
o, lse = attention(q, k, v, causal=bool(causal))
torch.cuda.synchronize()
print("done", sys.argv[1:], float(o.float().abs().sum()), flush=True)
