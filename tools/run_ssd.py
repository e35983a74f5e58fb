"""Time the Mamba-2 SSD chunk kernels on the paper's Table 4 shapes.

  python tools/run_ssd.py [--iters 10]
Reports device time (CUDA events, median), algorithmic HBM GB/s and TFLOP/s per shape.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17577_b200 import ssd_chunk_scan, ssd_chunk_state  # noqa: E402
from paper_2504_17577_b200.configs import SSD_CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_ssd, gen_ssd_cb_prev, ssd_chunked_dt  # noqa: E402


def med(fn, iters):
    for _ in range(3):
        fn()
    evs = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    for cfg in SSD_CONFIGS.values():
        if a.only and cfg.name not in a.only.split(","):
            continue
        x, Bm, C, dtv, A, D = gen_ssd(cfg.B, cfg.L, cfg.H, cfg.G, cfg.P, cfg.N, cfg.dtype, cfg.seed, "cuda")
        dt, dA = ssd_chunked_dt(dtv, A, cfg.Q)
        if cfg.kind == "state":
            out = torch.empty((cfg.B, cfg.nc, cfg.H, cfg.P, cfg.N), dtype=cfg.dtype, device="cuda")
            ms = med(lambda: ssd_chunk_state(x, Bm, dt, dA, out=out), a.iters)
        else:
            cb, prev = gen_ssd_cb_prev(cfg.B, cfg.L, cfg.H, cfg.G, cfg.P, cfg.N, cfg.dtype, cfg.seed, "cuda")
            out = torch.empty_like(x)
            ms = med(lambda: ssd_chunk_scan(cb, x, dt, dA, C, prev, D, out=out), a.iters)
        gbs = cfg.hbm_bytes() / ms / 1e6
        print(f"{cfg.name}: {ms * 1e3:8.1f} us  {gbs:7.0f} GB/s  {cfg.flops() / ms / 1e9:7.1f} TFLOP/s",
              flush=True)
        del x, Bm, C, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
