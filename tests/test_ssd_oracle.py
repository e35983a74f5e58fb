"""Pins for the fp64 Mamba-2 SSD chunk oracles (oracle/ssd_oracle.c), CPU only.

What the oracles compute is PAPER.md §5.2 P:L370 ("the chunk-scan and chunk-state functions
from Mamba-2", Table 4) under readings L1-L8. They are pinned to
things other than themselves:
  * the SSM recurrence evaluated position by position (oracle_ssd_recurrence: no chunks,
    no cumulative sums) equals chunk_state -> state passing -> chunk_scan, for ragged
    lengths, several groups and chunk sizes — a dropped decay term, a wrong sign, a wrong
    group index, an off-by-one in the causal sum or the chunk's last position each break it;
  * a hand-derived worked example (tests/golden/ssd_hand_examples.json);
  * special cases: A = 0 (no decay) reduces chunk_state to x^T diag(dt) B; dt = 0 leaves
    only the entering state and the D skip term; linearity in x; causality (out[i] does not
    depend on positions > i).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import ssd as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ssd_hand_examples.json")


def rand_inputs(Bn, L, H, G, P, N, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((Bn, L, H, P))
    Bm = rng.standard_normal((Bn, L, G, N))
    C = rng.standard_normal((Bn, L, G, N))
    dtv = np.exp(rng.uniform(math.log(1e-3), math.log(0.5), (Bn, L, H)))
    A = -rng.uniform(1.0, 16.0, H)
    D = rng.uniform(0.5, 1.5, H)
    return x, Bm, C, dtv, A, D


def chunked(x, Bm, C, dtv, A, D, Q):
    L = x.shape[1]
    dt_c = S.chunk_dt(dtv, Q)
    dA = S.chunk_cumsum(dt_c, A)
    states = oracle.ssd_chunk_state(x, Bm, dt_c, dA, Q)
    prev, final = S.state_passing(states, dA, L, Q)
    cb = S.bmm_chunk(C, Bm, Q)
    y = oracle.ssd_chunk_scan(cb, x, dt_c, dA, C, prev, D, Q)
    return y, final, states


@pytest.mark.parametrize("Bn,L,H,G,P,N,Q", [
    (1, 16, 1, 1, 2, 3, 4),
    (2, 37, 4, 2, 3, 5, 8),     # ragged last chunk, two groups
    (1, 64, 2, 1, 4, 6, 16),
    (2, 50, 6, 3, 2, 4, 64),    # one partial chunk
    (1, 129, 2, 2, 3, 3, 32),
])
def test_chunked_pipeline_equals_recurrence(Bn, L, H, G, P, N, Q):
    x, Bm, C, dtv, A, D = rand_inputs(Bn, L, H, G, P, N, 11 + L)
    y, final, _ = chunked(x, Bm, C, dtv, A, D, Q)
    y_rec, h_rec = oracle.ssd_recurrence(x, dtv, A, Bm, C, D)
    scale = np.abs(y_rec).max()
    assert np.abs(y - y_rec).max() <= 1e-11 * max(scale, 1.0)
    assert np.abs(final - h_rec).max() <= 1e-11 * max(np.abs(h_rec).max(), 1.0)


def test_hand_example():
    g = json.load(open(GOLDEN))
    inp = g["inputs"]
    ev = lambda e: float(eval(e, {"log": math.log, "__builtins__": {}}))  # noqa: E731
    x = np.array(inp["x"]).reshape(1, 3, 1, 1)
    Bm = np.array(inp["B"]).reshape(1, 3, 1, 1)
    C = np.array(inp["C"]).reshape(1, 3, 1, 1)
    dtv = np.array(inp["dt"]).reshape(1, 3, 1)
    A = np.array([ev(inp["A"])])
    D = np.array([inp["D"]])
    Q = inp["Q"]
    y, final, states = chunked(x, Bm, C, dtv, A, D, Q)
    exp_y = [ev(e) for e in g["expected"]["y"]]
    exp_s = [ev(e) for e in g["expected"]["states"]]
    np.testing.assert_allclose(y.ravel(), exp_y, rtol=0, atol=1e-12)
    np.testing.assert_allclose(states.ravel(), exp_s, rtol=0, atol=1e-12)
    np.testing.assert_allclose(final.ravel(), [ev(g["expected"]["final_state"])], rtol=0, atol=1e-12)
    y_rec, _ = oracle.ssd_recurrence(x, dtv, A, Bm, C, D)
    np.testing.assert_allclose(y_rec.ravel(), exp_y, rtol=0, atol=1e-12)


def test_no_decay_reduces_to_weighted_outer_products():
    """A = 0: dA = 0, every decay factor is 1 and states_c = sum_i dt_i x_i B_i^T."""
    Bn, L, H, G, P, N, Q = 2, 40, 2, 1, 3, 4, 16
    x, Bm, C, dtv, A, D = rand_inputs(Bn, L, H, G, P, N, 5)
    dt_c = S.chunk_dt(dtv, Q)
    dA = np.zeros_like(dt_c)
    st = oracle.ssd_chunk_state(x, Bm, dt_c, dA, Q)
    for c in range(st.shape[1]):
        seg = slice(c * Q, min(L, (c + 1) * Q))
        ref = np.einsum("blhp,blh,blgn->bhpn", x[:, seg], dtv[:, seg], Bm[:, seg])
        np.testing.assert_allclose(st[:, c], ref, rtol=1e-12, atol=1e-12)


def test_zero_dt_keeps_only_entering_state_and_skip():
    Bn, L, H, G, P, N, Q = 1, 24, 2, 2, 3, 4, 8
    x, Bm, C, _, _, D = rand_inputs(Bn, L, H, G, P, N, 6)
    nc = (L + Q - 1) // Q
    dt_c = np.zeros((Bn, H, nc, Q))
    dA = np.zeros_like(dt_c)
    rng = np.random.default_rng(1)
    prev = rng.standard_normal((Bn, nc, H, P, N))
    cb = rng.standard_normal((Bn, nc, G, Q, Q))
    assert np.all(oracle.ssd_chunk_state(x, Bm, dt_c, dA, Q) == 0.0)
    y = oracle.ssd_chunk_scan(cb, x, dt_c, dA, C, prev, D, Q)
    for t in range(L):
        c = t // Q
        for h in range(H):
            g = h // (H // G)
            ref = prev[0, c, h] @ C[0, t, g] + D[h] * x[0, t, h]
            np.testing.assert_allclose(y[0, t, h], ref, rtol=1e-12, atol=1e-12)


def test_linearity_and_causality():
    Bn, L, H, G, P, N, Q = 1, 48, 2, 1, 2, 3, 16
    x, Bm, C, dtv, A, D = rand_inputs(Bn, L, H, G, P, N, 8)
    y1, _, s1 = chunked(x, Bm, C, dtv, A, D, Q)
    y2, _, s2 = chunked(2.5 * x, Bm, C, dtv, A, D, Q)
    np.testing.assert_allclose(s2, 2.5 * s1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y2, 2.5 * y1, rtol=1e-12, atol=1e-12)
    x3 = x.copy()
    x3[:, 30:] += 7.0  # positions > 29 must not change out[0..29]
    y3, _, _ = chunked(x3, Bm, C, dtv, A, D, Q)
    np.testing.assert_array_equal(y3[:, :30], y1[:, :30])


def test_rejects_bad_arguments():
    x = np.zeros((1, 4, 3, 2))
    Bm = np.zeros((1, 4, 2, 2))  # H = 3 not a multiple of G = 2
    dt = np.zeros((1, 3, 1, 4))
    with pytest.raises(ValueError):
        oracle.ssd_chunk_state(x, Bm, dt, dt, 4)


def test_groups_equal_repeated_per_head_inputs():
    """Head h uses group h / (H / G) (contiguous grouping, reading L3): G = 2 shared groups
    over H = 4 heads equals G = H with the groups' B / C repeated as [g0, g0, g1, g1] (a
    modulo mapping would give [g0, g1, g0, g1] and fail)."""
    Bn, L, H, G, P, N, Q = 1, 40, 4, 2, 2, 3, 16
    x, Bm, C, dtv, A, D = rand_inputs(Bn, L, H, G, P, N, 12)
    rep = [h // (H // G) for h in range(H)]
    y_g, _, s_g = chunked(x, Bm, C, dtv, A, D, Q)
    y_h, _, s_h = chunked(x, Bm[:, :, rep], C[:, :, rep], dtv, A, D, Q)
    np.testing.assert_allclose(s_g, s_h, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(y_g, y_h, rtol=1e-13, atol=1e-13)
    y_rec, _ = oracle.ssd_recurrence(x, dtv, A, Bm[:, :, rep], C[:, :, rep], D)
    np.testing.assert_allclose(y_g, y_rec, rtol=0, atol=1e-10)
