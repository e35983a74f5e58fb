"""Shared helpers for GPU parity tests: run libtlattn, check against the fp64 oracle.

Tolerances (BASELINE.json north_star):
  O: max-abs <= 2e-2 and relative L2 (||dO||_2 / ||O_ref||_2 over checked elements) <= 5e-3
  LSE: max-abs <= 1e-3 (natural log); rows with an empty key set: O == 0, LSE == -inf.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
from paper_2504_17577_b200 import attention
from paper_2504_17577_b200.inputs import gen_qkv, to_bits

MAX_ABS = 2e-2
REL_L2 = 5e-3
LSE_ABS = 1e-3


def odt(tdtype):
    return oracle.ORACLE_BF16 if tdtype == torch.bfloat16 else oracle.ORACLE_F16


def sample_rows(Sq, rng, extra=0):
    """Rows checked per (b, h): 0..63 (where bf16 causal error peaks), tile/unit
    boundaries, and the last 16 rows (SURVEY §8c row sampling)."""
    base = set(range(min(64, Sq)))
    base |= {r for r in (127, 128, 129, 255, 256, 383, 384, 511, 512) if r < Sq}
    base |= set(range(max(0, Sq - 16), Sq))
    if extra:
        base |= set(int(x) for x in rng.integers(0, Sq, extra))
    return sorted(base)


def compare(o_gpu, lse_gpu, o_ref, lse_ref, label=""):
    """o_gpu/o_ref: [n, D] arrays (float64), lse: [n]. Returns dict of metrics; asserts."""
    o_gpu = np.asarray(o_gpu, np.float64)
    o_ref = np.asarray(o_ref, np.float64)
    empty = ~np.isfinite(lse_ref)
    stats = {}
    if empty.any():
        assert np.all(o_gpu[empty] == 0.0), f"{label}: empty-key rows must give O = 0"
        if lse_gpu is not None:
            assert np.all(np.isneginf(lse_gpu[empty])), f"{label}: empty-key rows must give LSE=-inf"
    ok = ~empty
    d = o_gpu[ok] - o_ref[ok]
    stats["max_abs"] = float(np.abs(d).max()) if d.size else 0.0
    nref = float(np.linalg.norm(o_ref[ok]))
    stats["rel_l2"] = float(np.linalg.norm(d) / nref) if nref > 0 else float(np.linalg.norm(d))
    if lse_gpu is not None and ok.any():
        stats["lse_abs"] = float(np.abs(np.asarray(lse_gpu, np.float64)[ok] - lse_ref[ok]).max())
    assert np.all(np.isfinite(o_gpu)), f"{label}: non-finite output"
    assert stats["max_abs"] <= MAX_ABS, f"{label}: max-abs {stats['max_abs']:.3e} > {MAX_ABS}"
    assert stats["rel_l2"] <= REL_L2, f"{label}: rel-L2 {stats['rel_l2']:.3e} > {REL_L2}"
    if "lse_abs" in stats:
        assert stats["lse_abs"] <= LSE_ABS, f"{label}: LSE abs {stats['lse_abs']:.3e} > {LSE_ABS}"
    return stats


def run_gpu(q, k, v, causal, scale):
    o, lse = attention(q, k, v, causal=causal, scale=scale)
    torch.cuda.synchronize()
    return o, lse


def check_against_oracle(q, k, v, causal, scale, rows_per_head=None, heads=None, label="",
                         full_rows_heads=()):
    """Run the GPU path and compare the given rows of the given (b, h) against the oracle.

    rows_per_head: None = all rows; else a list of row indices for every head.
    heads: iterable of (b, h) (default: all). full_rows_heads: (b, h) checked on all rows.
    """
    B, Sq, Hq, D = q.shape
    o, lse = run_gpu(q, k, v, causal, scale)
    qb, kb, vb = to_bits(q), to_bits(k), to_bits(v)
    if heads is None:
        heads = [(b, h) for b in range(B) for h in range(Hq)]
    all_rows = list(range(Sq))
    work = []
    for (b, h) in heads:
        rows = all_rows if (rows_per_head is None or (b, h) in full_rows_heads) else rows_per_head
        work.append((b, h, rows))
    for (b, h) in full_rows_heads:
        if (b, h) not in heads:
            work.append((b, h, all_rows))
    res = oracle.attn_rows_parallel(qb, kb, vb, odt(q.dtype), int(causal), scale, work)
    # gather the checked rows on the device (full-size outputs never leave HBM)
    bi = torch.tensor([b for (b, h, rows) in work for _ in rows], device=o.device)
    hi = torch.tensor([h for (b, h, rows) in work for _ in rows], device=o.device)
    ri = torch.tensor([r for (b, h, rows) in work for r in rows], device=o.device)
    og = o[bi, ri, hi, :].double().cpu().numpy()
    lg = lse[bi, hi, ri].double().cpu().numpy()
    orf = np.concatenate([r[0] for r in res])
    lrf = np.concatenate([r[1] for r in res])
    stats = compare(og, lg, orf, lrf, label)
    stats["rows_checked"] = int(sum(len(w[2]) for w in work))
    return stats, (o, lse)


def compare_outputs_with_oracle(q, k, v, o, lse, causal, scale, rows_per_head, label=""):
    """Compare GIVEN outputs o[B,Sq,Hq,D] / lse[B,Hq,Sq] (any producer: e.g. a replicated
    output written by several ranks' epilogues) with the fp64 oracle on ``rows_per_head``
    rows of EVERY (b, h), computed from the same q/k/v."""
    B, Sq, Hq, D = q.shape
    qb, kb, vb = to_bits(q), to_bits(k), to_bits(v)
    work = [(b, h, rows_per_head) for b in range(B) for h in range(Hq)]
    res = oracle.attn_rows_parallel(qb, kb, vb, odt(q.dtype), int(causal), scale, work)
    bi = torch.tensor([b for (b, h, rows) in work for _ in rows], device=o.device)
    hi = torch.tensor([h for (b, h, rows) in work for _ in rows], device=o.device)
    ri = torch.tensor([r for (b, h, rows) in work for r in rows], device=o.device)
    og = o[bi, ri, hi, :].double().cpu().numpy()
    lg = None if lse is None else lse[bi, hi, ri].double().cpu().numpy()
    orf = np.concatenate([r[0] for r in res])
    lrf = np.concatenate([r[1] for r in res])
    stats = compare(og, lg, orf, lrf, label)
    stats["rows_checked"] = int(og.shape[0])
    return stats


def gen(B, Hq, Hkv, Sq, Skv, D, dtype, seed):
    return gen_qkv(B, Hq, Hkv, Sq, Skv, D, dtype, seed, "cuda")


def default_scale(D):
    return 1.0 / math.sqrt(D)
