"""Host overhead and device time of small launches: eager vs CUDA-graph replay.
  python tools/run_overhead.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS, PAPER_T3  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402

ALL = {**CONFIGS, **PAPER_T3}


def main():
    for n in sys.argv[1:] or ["C1", "FA1", "FA3", "FA4"]:
        c = ALL[n]
        q, k, v = gen_qkv(c.B, c.Hq, c.Hkv, c.Sq, c.Skv, c.D, c.dtype, c.seed, "cuda")
        o = torch.empty_like(q)
        lse = torch.empty((c.B, c.Hq, c.Sq), dtype=torch.float32, device="cuda")
        f = lambda: attention(q, k, v, causal=c.causal, scale=c.scale, out=o, lse_out=lse)  # noqa: E731
        for _ in range(10):
            f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            f()
        t_host = (time.perf_counter() - t0) / 200
        torch.cuda.synchronize()
        t_all = (time.perf_counter() - t0) / 200
        # graph: 20 launches back to back in one graph
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                f()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        dev = a.elapsed_time(b) / 100
        print(f"{n}: host {t_host*1e6:.1f} us/call, eager throughput {t_all*1e6:.1f} us/call, "
              f"graph device {dev*1e3:.1f} us/launch ({c.flops()/dev/1e9:.0f} TFLOP/s, L2-warm)", flush=True)


if __name__ == "__main__":
    main()
