"""Trace the CTA-pair kernel's softmax AND MMA-issuer events for the first units of CTA 0
(debug build with -DTLATTN_TRACE).   TLATTN_LIB=build/libtr.so python tools/trace_issue.py C5

softmax per block: Sfull Sread exp0 Odone Pdone; issuer S(j): pre-Kwait Kfull Sissued,
issuer PV(j): pre-Vwait Vfull P0ready (all relative to the first event, SM clocks)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_17577_b200 import attention, load_library
from paper_2504_17577_b200.configs import CONFIGS
from paper_2504_17577_b200.inputs import gen_qkv
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
nunits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lib = load_library(); lib.tl_attn_debug_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(16000, dtype=torch.int64, device="cuda")
q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
attention(q, k, v, causal=cfg.causal)
assert lib.tl_attn_debug_trace(buf.data_ptr()) == 0
attention(q, k, v, causal=cfg.causal); torch.cuda.synchronize()
tr = buf.cpu().tolist()
t0 = min(x for x in tr[:8000] if x)
f = lambda x: f"{x - t0:7d}" if x else "      -"
for kk in range(nunits):
    g = lambda t, e: f(tr[200 * kk + 4000 + 1000 * t + 8 * 15 + e])
    print(f"--- unit {kk}: issuer Q-ready t0 {g(0, 7)} t1 {g(1, 7)} | issuer done t0 {g(0, 6)} t1 {g(1, 6)}")
    for j in range(16):
        rows = []
        for t in (0, 1):
            sm = [tr[200 * kk + 1000 * t + 8 * j + e] for e in range(5)]
            iss = [tr[200 * kk + 4000 + 1000 * t + 8 * j + e] for e in range(6)]
            rows.append(f"t{t} sm[{' '.join(f(x) for x in sm)}] S[{' '.join(f(x) for x in iss[:3])}] "
                        f"PV[{' '.join(f(x) for x in iss[3:])}]")
        if any(tr[200 * kk + 1000 * t + 8 * j] for t in (0, 1)):
            print(f" j={j:2d} " + " | ".join(rows))
