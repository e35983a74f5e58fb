"""Time the paper's Table 3 FlashAttention shapes with tl_attn_fwd,
L2 flushed between launches, and torch SDPA (cuDNN / flash backends) as context.
  python tools/run_table3.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.configs import PAPER_T3, CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402


def timeit(fn, iters=20, flush=None):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    names = sys.argv[1:] or list(PAPER_T3)
    for n in names:
        c = PAPER_T3.get(n) or CONFIGS[n]
        q, k, v = gen_qkv(c.B, c.Hq, c.Hkv, c.Sq, c.Skv, c.D, c.dtype, c.seed, "cuda")
        o = torch.empty_like(q)
        lse = torch.empty((c.B, c.Hq, c.Sq), dtype=torch.float32, device="cuda")
        ms = timeit(lambda: attention(q, k, v, causal=c.causal, scale=c.scale, out=o, lse_out=lse),
                    flush=flush)
        qt, kt, vt = (x.transpose(1, 2) for x in (q, k, v))
        try:
            ms_sdpa = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(
                qt, kt, vt, is_causal=c.causal, scale=c.scale), flush=flush)
        except Exception as e:  # noqa: BLE001
            ms_sdpa = float("nan")
        tf = c.flops() / ms / 1e9
        print(f"{n}: S={c.Sq} causal={int(c.causal)}  tl {ms*1e3:7.1f} us {tf:7.1f} TFLOP/s | "
              f"torch sdpa {ms_sdpa*1e3:7.1f} us {c.flops()/ms_sdpa/1e9:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
