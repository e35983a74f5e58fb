"""Run tl_attn_fwd on one config a few times (for ncu captures / quick timing).

  python tools/run_config.py C5 [--iters 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS, EXTRA, PAPER_T3  # noqa: E402
CONFIGS = {**CONFIGS, **EXTRA, **PAPER_T3}
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--time", action="store_true")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
    o = torch.empty_like(q)
    lse = torch.empty((cfg.B, cfg.Hq, cfg.Sq), dtype=torch.float32, device="cuda")
    evs = []
    for _ in range(a.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        attention(q, k, v, causal=cfg.causal, scale=cfg.scale, out=o, lse_out=lse)
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    if a.time:
        import statistics
        ms_all = [s.elapsed_time(e) for s, e in evs[1:]] or [evs[0][0].elapsed_time(evs[0][1])]
        ms = statistics.median(ms_all)
        print(f"{cfg.name}: median {ms:.3f} ms  {cfg.flops() / ms / 1e9:.1f} TFLOP/s "
              f"(min {min(ms_all):.3f} max {max(ms_all):.3f}, n={len(ms_all)})")


if __name__ == "__main__":
    main()
