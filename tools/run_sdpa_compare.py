"""Context only: torch SDPA backends (cuDNN / flash / efficient) vs tl_attn_fwd on the
BASELINE configs and Table 3 shapes (CUDA events, L2 flushed for small shapes).
  python tools/run_sdpa_compare.py [C2 T0 ...]"""
import os
import sys

import numpy as np
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17577_b200 import attention  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS, PAPER_T3  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402

ALL = {**CONFIGS, **PAPER_T3}


def timeit(fn, iters=10, flush=None):
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
    for n in sys.argv[1:] or ["C2", "C3", "C5", "T0", "C4", "FA4"]:
        c = ALL[n]
        q, k, v = gen_qkv(c.B, c.Hq, c.Hkv, c.Sq, c.Skv, c.D, c.dtype, c.seed, "cuda")
        fl = flush if c.hbm_bytes() < 64e6 else None
        o = torch.empty_like(q)
        lse = torch.empty((c.B, c.Hq, c.Sq), dtype=torch.float32, device="cuda")
        ms = timeit(lambda: attention(q, k, v, causal=c.causal, scale=c.scale, out=o, lse_out=lse), flush=fl)
        res = {"tl": c.flops() / ms / 1e9}
        qt, kt, vt = (x.transpose(1, 2) for x in (q, k, v))
        for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                         ("eff", SDPBackend.EFFICIENT_ATTENTION)):
            try:
                with sdpa_kernel([be]):
                    m2 = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(
                        qt, kt, vt, is_causal=c.causal, scale=c.scale, enable_gqa=c.Hq != c.Hkv), flush=fl)
                res[name] = c.flops() / m2 / 1e9
            except Exception as e:  # noqa: BLE001
                res[name] = None
        print(n, {a: (round(b, 1) if b else b) for a, b in res.items()}, flush=True)
        del q, k, v, o, lse, qt, kt, vt
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
