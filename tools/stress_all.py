"""Back-to-back launches of every attention config (hang / trap check for the default build):
N launches each of C2, C3, C4, C5, T0 and the Table 3 shapes, one synchronize per config.
  python tools/stress_all.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS, PAPER_T3  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for name, c in list(CONFIGS.items()) + list(PAPER_T3.items()):
    q, k, v = gen_qkv(c.B, c.Hq, c.Hkv, c.Sq, c.Skv, c.D, c.dtype, c.seed, "cuda")
    o = torch.empty_like(q)
    lse = torch.empty((c.B, c.Hq, c.Sq), dtype=torch.float32, device="cuda")
    ref, _ = attention(q, k, v, causal=c.causal, scale=c.scale)
    t0 = time.time()
    for _ in range(n):
        attention(q, k, v, causal=c.causal, scale=c.scale, out=o, lse_out=lse)
    torch.cuda.synchronize()
    same = torch.equal(o.view(torch.int16), ref.view(torch.int16))
    print(f"{name}: {n} launches in {time.time() - t0:.2f} s, last output bitwise == first: {same}",
          flush=True)
    del q, k, v, o, lse, ref
    torch.cuda.empty_cache()
