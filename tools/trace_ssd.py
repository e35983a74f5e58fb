"""Trace the SSD chunk_scan kernel's pipeline for the first units of CTA 0 (debug build with
-DTLATTN_TRACE):   TLATTN_LIB=build/libtr.so python tools/trace_ssd.py [CC3]

Per unit: producer TMA issue clock of each of the 13 ring items, W blocks loaded / built
(key quarter 0 and 2 warps), MMA issue stamps and the epilogue's start / end."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_17577_b200 import load_library, ssd_chunk_scan  # noqa: E402
from paper_2504_17577_b200.configs import SSD_CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_ssd, gen_ssd_cb_prev, ssd_chunked_dt  # noqa: E402

cfg = SSD_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "CC3"]
lib = load_library()
lib.tl_attn_debug_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(4000, dtype=torch.int64, device="cuda")
x, Bm, C, dtv, A, D = gen_ssd(cfg.B, cfg.L, cfg.H, cfg.G, cfg.P, cfg.N, cfg.dtype, cfg.seed, "cuda")
dt, dA = ssd_chunked_dt(dtv, A, cfg.Q)
cb, prev = gen_ssd_cb_prev(cfg.B, cfg.L, cfg.H, cfg.G, cfg.P, cfg.N, cfg.dtype, cfg.seed, "cuda")
o = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
assert lib.tl_attn_debug_trace(buf.data_ptr()) == 0
o = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
torch.cuda.synchronize()
tr = buf.cpu().tolist()
t0 = min(v for v in tr if v)
f = lambda v: f"{v - t0:7d}" if v else "      -"  # noqa: E731
# CTA 0 owns units 0, G, 2G, ... (G = the odd persistent grid): mt alternates 0, 1, 0, ...
f0 = 0
for lu in range(8):
    mt = lu & 1
    ni = 9 if mt else 6
    print(f"unit {lu} (mt {mt}): items issued", " ".join(f(tr[f0 + i]) for i in range(ni)))
    f0 += ni
    print("   W block0 k-half0 loaded/built, k-half1 loaded/built; block1 ...",
          " ".join(f(tr[1000 + lu * 12 + j]) for j in range(4 + 4 * mt)))
    print("   MMA start / after C.prev / after W0.x / end", " ".join(f(tr[1400 + lu * 8 + j]) for j in range(4)))
    print("   epi", f(tr[1600 + lu * 2]), f(tr[1601 + lu * 2]))
