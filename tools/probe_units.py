"""Per-unit cost probe: time tl_attn_fwd on shapes whose 512-row units have a fixed number
of K/V block steps (non-causal Sq = 512, Skv = 128 n) next to C5, to separate the per-step
cost from the per-unit (transition) cost and the causal losses.

  python tools/probe_units.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402


def run(B, H, Sq, Skv, causal, iters=12):
    q, k, v = gen_qkv(B, H, H, Sq, Skv, 128, torch.bfloat16, 1, "cuda")
    o = torch.empty_like(q)
    lse = torch.empty((B, H, Sq), dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        attention(q, k, v, causal=causal, scale=128 ** -0.5, out=o, lse_out=lse)
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    ms = statistics.median(s.elapsed_time(e) for s, e in ts[1:])
    if causal:
        fl = 4.0 * B * H * D_ * Sq * Skv / 2
    else:
        fl = 4.0 * B * H * D_ * Sq * Skv
    return ms, fl / ms / 1e9


D_ = 128
if __name__ == "__main__":
    ms, tf = run(64, 32, 2048, 2048, True)
    units = 64 * 32 * 4
    print(f"C5 causal 2048: {ms:.3f} ms {tf:.0f} TFLOP/s  us/unit/pair {ms * 1e3 * 74 / units:.2f}")
    for n in (2, 4, 6, 8, 10, 12, 16, 32):
        B = max(1, 8192 * 10 // (32 * n * 4)) if n < 10 else 64
        B = 256 if n <= 4 else (128 if n <= 8 else 64)
        ms, tf = run(B, 32, 512, 128 * n, False)
        units = B * 32
        print(f"noncausal Sq512 Skv{128 * n}: B{B} {ms:.3f} ms {tf:.0f} TFLOP/s  "
              f"us/unit/pair {ms * 1e3 * 74 / units:.3f}  us/step {ms * 1e3 * 74 / units / n:.3f}")
