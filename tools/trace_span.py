"""Per-CTA timeline of the CTA-pair attention kernel (debug build with -DTLATTN_TRACE):
globaltimer at kernel entry, first S of units 0-3, O store issued, kernel end, for every CTA.
  TLATTN_LIB=build/libtr.so python tools/trace_span.py FA3"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_17577_b200 import attention, load_library  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS, PAPER_T3  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402

ALL = {**CONFIGS, **PAPER_T3}


def main():
    for name in sys.argv[1:] or ["FA3"]:
        cfg = ALL[name]
        lib = load_library()
        lib.tl_attn_debug_trace.argtypes = [ctypes.c_void_p]
        buf = torch.zeros(16000 + 32 * 160, dtype=torch.int64, device="cuda")
        q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
        o = torch.empty_like(q)
        f = lambda: attention(q, k, v, causal=cfg.causal, scale=cfg.scale, out=o)  # noqa: E731
        f()
        assert lib.tl_attn_debug_trace(buf.data_ptr()) == 0
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for cold in (True, False):
            buf.zero_()
            if cold:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            sp = buf[16000:16000 + 16 * 160].view(160, 16).cpu().numpy().astype(np.int64)
            pr = buf[16000 + 16 * 160:].view(160, 16).cpu().numpy().astype(np.int64)
            live = sp[:, 0] > 0
            sp, pr = sp[live], pr[live]
            t0 = sp[:, 0].min()
            prel = np.where(pr > 0, pr - t0, -1) / 1000.0
            names = ["Q0 issue", "Q0 issued", "ring0", "ring1", "ring2", "ring3", "ring4", "ring5", "producer start"]
            print("  producer (median us): " + ", ".join(
                f"{names[i]} {np.median(prel[prel[:, i] >= 0, i]):.2f}" for i in (8, 0, 1, 2, 3, 4, 5, 6, 7)
                if (prel[:, i] >= 0).any()))
            rel = np.where(sp > 0, sp - t0, -1) / 1000.0  # us
            print(f"== {name} {'cold L2' if cold else 'warm L2'}: event {a.elapsed_time(b) * 1e3:.1f} us, "
                  f"{len(sp)} CTAs")
            print(f"  entry spread  {rel[:, 0].max():.2f} us; setup done median {np.median(rel[:, 14]):.2f}; "
                  f"leader Q ready median {np.median(rel[rel[:, 13] >= 0, 13]):.2f}")
            for kk in range(4):
                s, e = rel[:, 1 + 3 * kk], rel[:, 2 + 3 * kk]
                ok = (s >= 0) & (e >= 0)
                if ok.any():
                    print(f"  unit {kk}: CTAs {ok.sum():3d} first-S median {np.median(s[ok]):6.2f} "
                          f"(min {s[ok].min():.2f} max {s[ok].max():.2f}) store median {np.median(e[ok]):6.2f} "
                          f"max {e[ok].max():6.2f}; duration median {np.median(e[ok] - s[ok]):.2f}")
            print(f"  kernel end: median {np.median(rel[:, 15]):.2f} max {rel[:, 15].max():.2f} us")
        lib.tl_attn_debug_trace(None)


if __name__ == "__main__":
    main()
