"""Plain fp64 steps of the Mamba-2 SSD pipeline around the two chunk kernels — TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

The chunk kernels (oracle.ssd_chunk_state / ssd_chunk_scan, ssd_oracle.c) take the chunked
cumulative decay dA, the per-chunk C B^T (cb) and the entering states (prev) as inputs
(readings L4, L6 in DESIGN.md §3). Chaining them with the three steps below reproduces the
SSM recurrence (oracle.ssd_recurrence), which is how the chunk oracles are pinned.
Each step is the textbook definition written out with numpy loops / einsum in fp64.
"""
from __future__ import annotations

import numpy as np


def chunk_dt(dtv, Q):
    """dt per position [B,L,H] -> [B,H,nc,Q] (entries past the sequence end are 0)."""
    Bn, L, H = dtv.shape
    nc = (L + Q - 1) // Q
    out = np.zeros((Bn, H, nc, Q), np.float64)
    for c in range(nc):
        seg = np.asarray(dtv[:, c * Q:(c + 1) * Q, :], np.float64)  # [B, len, H]
        out[:, :, c, :seg.shape[1]] = seg.transpose(0, 2, 1)
    return out


def chunk_cumsum(dt_c, A):
    """dA[b,h,c,i] = sum_{j <= i} dt[b,h,c,j] * A[h] (inclusive, restarting every chunk)."""
    dA = np.zeros_like(dt_c, dtype=np.float64)
    run = np.zeros(dt_c.shape[:3], np.float64)
    for i in range(dt_c.shape[3]):
        run = run + dt_c[..., i] * np.asarray(A, np.float64)[None, :, None]
        dA[..., i] = run
    return dA


def bmm_chunk(C, Bm, Q):
    """cb[b,c,g,i,j] = sum_n C[b,cQ+i,g,n] Bm[b,cQ+j,g,n] (zero past the sequence end)."""
    Bn, L, G, N = C.shape
    nc = (L + Q - 1) // Q
    cb = np.zeros((Bn, nc, G, Q, Q), np.float64)
    for c in range(nc):
        cc = np.asarray(C[:, c * Q:(c + 1) * Q], np.float64)
        bb = np.asarray(Bm[:, c * Q:(c + 1) * Q], np.float64)
        n = cc.shape[1]
        cb[:, c, :, :n, :n] = np.einsum("bign,bjgn->bgij", cc, bb)
    return cb


def state_passing(states, dA, L, Q):
    """prev[b,c] = state entering chunk c: prev[b,0] = 0,
    prev[b,c+1] = exp(dA[b,h,c,len_c - 1]) prev[b,c] + states[b,c] (per head)."""
    Bn, nc, H, P, N = states.shape
    prev = np.zeros_like(states, dtype=np.float64)
    cur = np.zeros((Bn, H, P, N), np.float64)
    for c in range(nc):
        prev[:, c] = cur
        last = min(Q, L - c * Q) - 1
        cur = np.exp(dA[:, :, c, last])[:, :, None, None] * cur + states[:, c]
    return prev, cur
