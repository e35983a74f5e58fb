"""Unit-boundary timeline of the CTA-pair kernel from a tools/trace_dump.py .npy (SM clocks of
the leader CTA relative to its first event; softmax rows of both CTAs).
   python tools/trace_boundary.py tr.npy [units]"""
import sys
import numpy as np
tr = np.load(sys.argv[1]).astype(np.int64)
nun = int(sys.argv[2]) if len(sys.argv) > 2 else 4
base = [x for x in tr[:8000] if x]
t0 = min(base)
def f(x):
    return f"{int(x - t0):7d}" if x else "      -"
for k in range(nun):
    o = 200 * k
    print(f"=== unit {k}")
    for t in (0, 1):
        iss = tr[o + 4000 + 1000 * t + 8 * 15 + 6], tr[o + 4000 + 1000 * t + 8 * 15 + 7]
        ex = [tr[o + 6000 + 100 * t + e] for e in range(3)]
        print(f" issuer t{t}: Qready {f(iss[1])} done {f(iss[0])} | sched-seen {f(ex[0])} queried {f(ex[1])} decoded {f(ex[2])}")
        for cta in (0, 1):
            oc = 8000 * cta
            js = [j for j in range(16) if tr[oc + o + 1000 * t + 8 * j]]
            if not js:
                continue
            first = tr[oc + o + 1000 * t + 8 * js[0]]
            last = tr[oc + o + 1000 * t + 8 * js[-1] + 4]
            ep = [tr[oc + o + 6500 + 100 * t + e] for e in range(4)]
            print(f"   cta{cta} softmax t{t}: blocks {len(js)} first S {f(first)} last P {f(last)} | "
                  f"epi start {f(ep[0])} O staged {f(ep[1])} LSE {f(ep[2])} next known {f(ep[3])}")
            iss_s0 = tr[o + 4000 + 1000 * t + 0 * 8 + 2]
        print(f"   issuer t{t} S(0): pre-K {f(tr[o + 4000 + 1000 * t + 0])} Kfull {f(tr[o + 4000 + 1000 * t + 1])} issued {f(tr[o + 4000 + 1000 * t + 2])}")
