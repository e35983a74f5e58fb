"""Time tl_mla_decode on the MLA configs (CUDA events, median of N launches).
Usage: python tools/run_mla.py [MLA1 MLA2 ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17577_b200 import mla_decode, tl_mla_decode_workspace_bytes  # noqa: E402
from paper_2504_17577_b200.configs import MLA_CONFIGS  # noqa: E402
from paper_2504_17577_b200.inputs import gen_mla  # noqa: E402


def main():
    names = sys.argv[1:] or [c.name for c in MLA_CONFIGS]
    peaks = {"hbm": 6533.5, "tf": 1639.8}
    for c in MLA_CONFIGS:
        if c.name not in names:
            continue
        q, qp, kv, kp = gen_mla(c.B, c.H, c.Hkv, c.Skv, c.Dl, c.Dr, c.dtype, c.seed, "cuda")
        sl = c.seqlens()
        sld = None if sl is None else torch.as_tensor(sl, device="cuda")
        ws = torch.empty(tl_mla_decode_workspace_bytes(c.B, c.H, c.Hkv), dtype=torch.uint8, device="cuda")
        o = torch.empty((c.B, c.H, c.Dl), dtype=c.dtype, device="cuda")
        lse = torch.empty((c.B, c.H), dtype=torch.float32, device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(15):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mla_decode(q, qp, kv, kp, seqlens=sld, out=o, lse_out=lse, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        gbs = c.hbm_bytes() / ms / 1e6
        tf = c.flops() / ms / 1e9
        print(f"{c.name}: {ms*1e3:.1f} us  {gbs:.0f} GB/s ({gbs/peaks['hbm']*100:.1f}% HBM)  "
              f"{tf:.0f} TFLOP/s ({tf/peaks['tf']*100:.1f}% bf16)", flush=True)


if __name__ == "__main__":
    main()
