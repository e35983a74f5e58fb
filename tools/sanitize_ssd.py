"""Small SSD chunk_state / chunk_scan calls for compute-sanitizer (memcheck / racecheck /
synccheck): ragged last chunk, groups > 1, several units per persistent CTA (tiny grid
forced by many units on few SMs is not controllable, so shapes with more units than SMs)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_17577_b200 import ssd_chunk_scan, ssd_chunk_state
from paper_2504_17577_b200.inputs import gen_ssd, gen_ssd_cb_prev, ssd_chunked_dt

for (B, L, H, G) in [(1, 300, 4, 2), (2, 1100, 8, 1), (1, 4096, 80, 1)]:
    P, N, Q = 64, 128, 256
    x, Bm, C, dtv, A, D = gen_ssd(B, L, H, G, P, N, torch.bfloat16, 7, "cuda")
    dt, dA = ssd_chunked_dt(dtv, A, Q)
    st = ssd_chunk_state(x, Bm, dt, dA)
    cb, prev = gen_ssd_cb_prev(B, L, H, G, P, N, torch.bfloat16, 7, "cuda")
    out = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
    torch.cuda.synchronize()
    print(B, L, H, G, float(st.float().abs().sum()), float(out.float().abs().sum()), flush=True)
