"""Run one config with the debug trace build and print the pipeline timeline of CTA 0.

  TLATTN_LIB=build/var/tr.so python tools/trace_run.py T0
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_17577_b200 import attention, load_library  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "T0"]
nblk = int(sys.argv[2]) if len(sys.argv) > 2 else 12
lib = load_library()
lib.tl_attn_debug_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(16000, dtype=torch.int64, device="cuda")
q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
attention(q, k, v, causal=cfg.causal)  # warm
assert lib.tl_attn_debug_trace(buf.data_ptr()) == 0
attention(q, k, v, causal=cfg.causal)
torch.cuda.synchronize()
tr = buf.cpu().tolist()
nz = [x for x in tr if x]
t0 = min(nz)
print("events relative to first (SM clocks); softmax: Sfull Sread expdone Odone Pfull | issuer: S_issue PV_issue")
nzp = [x for x in tr[8000:] if x]
t0p = min(nzp) if nzp else 0
for j in range(nblk):
    row = []
    for t in (0, 1):
        sm = [tr[1000 * t + 8 * j + e] for e in range(5)]
        iss = [tr[4000 + 1000 * t + 4 * j + e] for e in range(2)]
        f = lambda x: f"{x - t0:7d}" if x else "      -"
        row.append("t%d sm[%s] iss[%s]" % (t, " ".join(f(x) for x in sm), " ".join(f(x) for x in iss)))
    print(f"j={j:2d} " + " || ".join(row))
print("peer CTA softmax (own clock, relative to its first event):")
for j in range(nblk):
    row = []
    for t in (0, 1):
        sm = [tr[8000 + 1000 * t + 8 * j + e] for e in range(5)]
        g = lambda x: f"{x - t0p:7d}" if x else "      -"
        row.append("t%d sm[%s]" % (t, " ".join(g(x) for x in sm)))
    print(f"j={j:2d} " + " || ".join(row))
