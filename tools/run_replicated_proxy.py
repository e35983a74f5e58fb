"""One-GPU proxy for the fused replicated output: C5 head shard of one rank at
world size w (Hq/w query heads), timed (CUDA events, median of 11) as
  (a) tl_attn_fwd on the shard alone,
  (b) tl_attn_fwd_replicated writing the shard into w full-size output buffers (all local:
      the stores go to this GPU's HBM instead of NVLink peers),
  (c) (a) followed by w-1 device-to-device copies of the shard (the unfused fan-out).
  python tools/run_replicated_proxy.py [w]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_17577_b200 import attention, tl_attn_fwd_replicated  # noqa: E402
from paper_2504_17577_b200.configs import CONFIGS  # noqa: E402
from paper_2504_17577_b200.dist import make_shard  # noqa: E402
from paper_2504_17577_b200.inputs import gen_qkv  # noqa: E402
from paper_2504_17577_b200.tlattn import dtype_code  # noqa: E402


def med(fn, iters=11):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    c = CONFIGS["C5"]
    sh = make_shard("head", 0, w, c.B, c.Hq, c.Hkv)
    q, k, v = gen_qkv(c.B, c.Hq, c.Hkv, c.Sq, c.Skv, c.D, c.dtype, c.seed, "cuda",
                      b_slice=sh.b, hq_slice=sh.hq, hkv_slice=sh.hkv)
    Bl, S, Hl, D = q.shape
    outs = [torch.empty((c.B, c.Sq, c.Hq, c.D), dtype=c.dtype, device="cuda") for _ in range(w)]
    o = torch.empty_like(q)
    t_a = med(lambda: attention(q, k, v, causal=c.causal, scale=c.scale, out=o, return_lse=False))
    t_b = med(lambda: tl_attn_fwd_replicated(q, k, v, outs, None, c.B, 0, c.Hq, sh.hq.start, Bl, Hl,
                                             k.shape[2], S, S, D, int(c.causal), c.scale,
                                             dtype_code(q.dtype)))

    def unfused():
        attention(q, k, v, causal=c.causal, scale=c.scale, out=o, return_lse=False)
        for r in range(1, w):
            outs[r][:, :, sh.hq.start:sh.hq.stop].copy_(o)
    t_c = med(unfused)
    mb = o.numel() * 2 / 1e6
    print(f"C5 head shard w={w} ({Hl} heads, O shard {mb:.0f} MB): attention {t_a:.3f} ms | "
          f"fused replicated x{w} {t_b:.3f} ms | attention + {w - 1} copies {t_c:.3f} ms")


if __name__ == "__main__":
    main()
