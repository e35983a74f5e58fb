"""Discrete-event model of the attention kernel's per-SM pipeline (design aid).

Tensor pipe: in-order FIFO, each MMA (S_t or PV_t of one 128x128xD block) takes
T_MMA clocks. Two query tiles; per tile: an issuer thread and a softmax warpgroup.
Latencies: W = mbarrier wake-up, LD = TMEM load of the S row block, SM = softmax
math after the load, ST = P store + fences. Variants:
  order="early":   S_t(j+1) issued after softmax t has loaded S_t(j) (P in smem)
  order="alias":   S_t(j+1) issued after PV_t(j) (P aliases S in TMEM, FA4-like)
  sbuf=2:          two S buffers per tile (S_t(j+2) needs S_t(j) loaded)
Shared MUFU: softmax compute of the two tiles is serialised on one resource when
mufu_shared=True (SM is the exclusive MUFU time per tile-block).
"""
import argparse
import heapq


def simulate(nblk=64, T_MMA=512, W=80, LD=250, SM=1024, ST=150, order="early", sbuf=1,
             mufu_shared=True, issue=60):
    t_pipe = 0.0
    s_done = {}     # (t, j) -> completion time of S_t(j)
    pv_done = {}
    s_read = {}     # (t, j) -> time softmax loaded S_t(j)
    p_ready = {}
    busy = 0.0
    mufu_free = 0.0
    # event-driven over a simple fixed-point iteration: issue MMAs in order of readiness
    issued = []
    # per tile next ops
    nxt_s = {0: 0, 1: 0}
    nxt_pv = {0: 0, 1: 0}
    sm_next = {0: 0, 1: 0}
    INF = float("inf")

    def s_ready(t, j):
        if j < sbuf:
            return 0.0
        if order == "alias":
            return pv_done.get((t, j - 1), INF) + W
        return s_read.get((t, j - sbuf), INF) + W

    def pv_ready(t, j):
        return p_ready.get((t, j), INF) + W

    steps = 0
    while (nxt_pv[0] < nblk or nxt_pv[1] < nblk) and steps < 100000:
        steps += 1
        # advance softmax where possible
        for t in (0, 1):
            j = sm_next[t]
            if j < nblk and (t, j) in s_done and (j == 0 or (t, j - 1) in pv_done):
                start = s_done[(t, j)] + W
                rd = start + LD
                s_read[(t, j)] = rd
                c0 = rd
                if mufu_shared:
                    c0 = max(c0, mufu_free)
                    mufu_free = c0 + SM
                comp = c0 + SM
                if j > 0:
                    comp = max(comp, pv_done[(t, j - 1)] + W)
                p_ready[(t, j)] = comp + ST
                sm_next[t] += 1
        # choose the earliest-ready MMA among the 4 candidates; in-order pipe
        cands = []
        for t in (0, 1):
            if nxt_s[t] < nblk:
                r = s_ready(t, nxt_s[t])
                if r < INF:
                    cands.append((r, 0, t))
            if nxt_pv[t] < nblk and nxt_pv[t] < nxt_s[t]:
                r = pv_ready(t, nxt_pv[t])
                if r < INF:
                    cands.append((r, 1, t))
        if not cands:
            continue
        r, kind, t = min(cands)
        start = max(t_pipe, r + issue)
        t_pipe = start + T_MMA
        busy += T_MMA
        if kind == 0:
            s_done[(t, nxt_s[t])] = t_pipe
            nxt_s[t] += 1
        else:
            pv_done[(t, nxt_pv[t])] = t_pipe
            nxt_pv[t] += 1
    return busy / t_pipe


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--sm", type=float, default=1024)
    a = ap.parse_args()
    for order, sbuf in (("early", 1), ("alias", 1), ("early", 2)):
        for SM in (0, 400, 700, 1024):
            for LD in (100, 250, 400):
                u = simulate(order=order, sbuf=sbuf, SM=SM, LD=LD)
                print(f"order={order:5s} sbuf={sbuf} SM={SM:5d} LD={LD:4d} tensor_util={u:.2f}")
