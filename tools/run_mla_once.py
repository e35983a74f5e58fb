"""Run tl_mla_decode on one MLA config a few times (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17577_b200 import mla_decode, tl_mla_decode_workspace_bytes  # noqa: E402
from paper_2504_17577_b200.configs import MLA_CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_mla  # noqa: E402

c = next(x for x in MLA_CONFIGS if x.name == sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
q, qp, kv, kp = gen_mla(c.B, c.H, c.Hkv, c.Skv, c.Dl, c.Dr, c.dtype, c.seed, "cuda")
sl = c.seqlens()
sld = None if sl is None else torch.as_tensor(sl, device="cuda")
ws = torch.empty(tl_mla_decode_workspace_bytes(c.B, c.H, c.Hkv), dtype=torch.uint8, device="cuda")
for _ in range(iters):
    mla_decode(q, qp, kv, kp, seqlens=sld, workspace=ws)
torch.cuda.synchronize()
