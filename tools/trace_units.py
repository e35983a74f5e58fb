"""Trace several units of CTA 0 (debug build): per block Sfull/Sread/expdone/Odone/Pfull and
per unit epilogue (o_final, stats, o_free).  TLATTN_LIB=build/var/tr.so python tools/trace_units.py C5"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_17577_b200 import attention, load_library
from paper_2504_17577_b200.configs import CONFIGS
from paper_2504_17577_b200.inputs import gen_qkv
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
lib = load_library(); lib.tl_attn_debug_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(16000, dtype=torch.int64, device="cuda")
q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
attention(q, k, v, causal=cfg.causal)
assert lib.tl_attn_debug_trace(buf.data_ptr()) == 0
attention(q, k, v, causal=cfg.causal); torch.cuda.synchronize()
tr = buf.cpu().tolist()
t0 = min(x for x in tr[:8000] if x)
f = lambda x: f"{x - t0:7d}" if x else "      -"
for kk in range(4):
    print(f"--- unit {kk}: epilogue t0 [{f(tr[6000+20*kk+0])} {f(tr[6000+20*kk+1])} {f(tr[6000+20*kk+2])}]"
          f"  t1 [{f(tr[6000+20*kk+10])} {f(tr[6000+20*kk+11])} {f(tr[6000+20*kk+12])}]")
    for j in range(16):
        a = [tr[200*kk + 8*j + e] for e in range(5)]
        b = [tr[200*kk + 1000 + 8*j + e] for e in range(5)]
        if not any(a) and not any(b): continue
        print(f" j={j:2d} t0[{' '.join(f(x) for x in a)}] t1[{' '.join(f(x) for x in b)}]")
