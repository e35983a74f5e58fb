"""Dump the raw TL_TRACE2 buffer of the CTA-pair kernel (debug build, -DTLATTN_TRACE) for one
config to a .npy file (both CTAs of cluster 0; offline analysis with tools/trace_boundary.py).
   TLATTN_LIB=build/libtr.so python tools/trace_dump.py C5 out.npy"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2504_17577_b200 import attention, load_library
from paper_2504_17577_b200.configs import CONFIGS
from paper_2504_17577_b200.inputs import gen_qkv
cfg = CONFIGS[sys.argv[1]]
lib = load_library(); lib.tl_attn_debug_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(16000 + 16 * 4096, dtype=torch.int64, device="cuda")
q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
attention(q, k, v, causal=cfg.causal)
assert lib.tl_attn_debug_trace(buf.data_ptr()) == 0
attention(q, k, v, causal=cfg.causal); torch.cuda.synchronize()
np.save(sys.argv[2], buf.cpu().numpy())
print("saved", sys.argv[2])
