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

# SSD chunk kernels (Table 4 shapes) and MLA decode: the same check
from paper_2504_17577_b200 import mla_decode, ssd_chunk_scan, ssd_chunk_state  # noqa: E402
from paper_2504_17577_b200 import tl_mla_decode_workspace_bytes  # noqa: E402
from paper_2504_17577_b200.configs import MLA_CONFIGS, SSD_CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_mla, gen_ssd, gen_ssd_cb_prev, ssd_chunked_dt  # noqa: E402

for name in ("CT3", "CC3", "CT5", "CC5"):
    c = SSD_CONFIGS[name]
    x, Bm, C, dtv, A, D = gen_ssd(c.B, c.L, c.H, c.G, c.P, c.N, c.dtype, c.seed, "cuda")
    dt, dA = ssd_chunked_dt(dtv, A, c.Q)
    if c.kind == "state":
        f = lambda out=None: ssd_chunk_state(x, Bm, dt, dA, out=out)  # noqa: E731
    else:
        cb, prev = gen_ssd_cb_prev(c.B, c.L, c.H, c.G, c.P, c.N, c.dtype, c.seed, "cuda")
        f = lambda out=None: ssd_chunk_scan(cb, x, dt, dA, C, prev, D, out=out)  # noqa: E731
    ref = f()
    o = torch.empty_like(ref)
    t0 = time.time()
    for _ in range(n):
        f(o)
    torch.cuda.synchronize()
    same = torch.equal(o.view(torch.int16), ref.view(torch.int16))
    print(f"{name}: {n} launches in {time.time() - t0:.2f} s, last output bitwise == first: {same}",
          flush=True)
    del x, Bm, C, o, ref
    torch.cuda.empty_cache()

for c in MLA_CONFIGS:
    q, qp, kv, kp = gen_mla(c.B, c.H, c.Hkv, c.Skv, c.Dl, c.Dr, c.dtype, c.seed, "cuda")
    sl = c.seqlens()
    sld = None if sl is None else torch.as_tensor(sl, device="cuda")
    ws = torch.empty(tl_mla_decode_workspace_bytes(c.B, c.H, c.Hkv), dtype=torch.uint8, device="cuda")
    ref, _ = mla_decode(q, qp, kv, kp, seqlens=sld, workspace=ws)
    ref = ref.clone()
    o = torch.empty_like(ref)
    t0 = time.time()
    for _ in range(n):
        mla_decode(q, qp, kv, kp, seqlens=sld, out=o, workspace=ws)
    torch.cuda.synchronize()
    same = torch.equal(o.view(torch.int16), ref.view(torch.int16))
    print(f"{c.name}: {n} launches in {time.time() - t0:.2f} s, last output bitwise == first: {same}",
          flush=True)
    del q, qp, kv, kp, o, ref, ws
    torch.cuda.empty_cache()
