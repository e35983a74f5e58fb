"""GPU parity of the Mamba-2 SSD chunk kernels (tl_ssd_chunk_state / tl_ssd_chunk_scan,
SURVEY §8(f) N4; Table 4) against the fp64 oracles, through the
C ABI.

Both sides take the SAME inputs: the 16-bit x / B / C / cb / prev and the fp32 dt / dA the
kernel reads are widened exactly to fp64 for the oracle. cb and prev come from the oracle
pipeline (C B^T per chunk, state passing of the oracle's chunk states), rounded to the dtype.
Bar: per element |gpu - ref| <= 2^-7 |ref| + 2^-5 rms(ref) and relative L2
<= 5e-3. Derivation: fp32 accumulation; the 16-bit operands the tensor core multiplies are
the decay-scaled x' = RN(w x) (chunk_state) and W = RN(cb exp(..) dt) (chunk_scan), each
rounded with unit roundoff u = 2^-8 (bf16), so a sum of n random-sign terms carries an
absolute error of ~u/sqrt(3) * rms(ref) (measured rel-L2 2.3e-3 on every block) — up to
~5 sigma over a block is < 2^-5 rms(ref) — plus the RN rounding of the output itself,
<= u |ref| < 2^-7 |ref|."""
import numpy as np
import pytest
import torch

import oracle
from oracle import ssd as S
from paper_2504_17577_b200 import ssd_chunk_scan, ssd_chunk_state
from paper_2504_17577_b200.inputs import gen_ssd, gen_ssd_cb_prev, ssd_chunked_dt

pytestmark = pytest.mark.gpu
Q = 256
BF, F16 = torch.bfloat16, torch.float16


def f64(t):
    return t.detach().double().cpu().numpy()


def check(got, ref, label):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert np.all(np.isfinite(got)), f"{label}: non-finite output"
    rms = float(np.sqrt(np.mean(ref ** 2))) if ref.size else 0.0
    err = np.abs(got - ref)
    bound = 2.0 ** -7 * np.abs(ref) + 2.0 ** -5 * rms
    worst = float((err - bound).max()) if ref.size else 0.0
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    assert worst <= 0.0, f"{label}: element error above 2^-7 |ref| + 2^-5 rms: max excess {worst:.3e}"
    assert rel <= 5e-3, f"{label}: rel-L2 {rel:.3e}"
    return {"max_abs": float(err.max()), "rel_l2": rel}


def make(Bn, L, H, G, dtype, seed):
    x, Bm, C, dtv, A, D = gen_ssd(Bn, L, H, G, 64, 128, dtype, seed, "cuda")
    dt, dA = ssd_chunked_dt(dtv, A, Q)
    return x, Bm, C, dt, dA, D


def oracle_prev_cb(x, Bm, C, dt, dA, L, dtype):
    """cb = C B^T and the entering states from the oracle pipeline, rounded to dtype."""
    states = oracle.ssd_chunk_state(f64(x), f64(Bm), f64(dt), f64(dA), Q)
    prev, _ = S.state_passing(states, f64(dA), L, Q)
    cb = S.bmm_chunk(f64(C), f64(Bm), Q)
    to = lambda a: torch.as_tensor(a, dtype=torch.float64).to(dtype).cuda().contiguous()  # noqa
    return to(cb), to(prev)


SMALL = [  # B, L, H, G, dtype
    (1, 256, 2, 1, BF),
    (2, 300, 4, 2, BF),     # ragged last chunk, two groups
    (1, 700, 6, 3, F16),    # three chunks, the last partial
    (1, 100, 2, 1, BF),     # one partial chunk (second row tile empty)
    (3, 512, 8, 1, F16),
    (2, 1100, 12, 3, BF),   # groups of 4 heads (four-head state units), ragged, 5 chunks
]


@pytest.mark.parametrize("Bn,L,H,G,dtype", SMALL)
def test_chunk_state_every_element(Bn, L, H, G, dtype):
    x, Bm, C, dt, dA, D = make(Bn, L, H, G, dtype, 17 + L)
    st = ssd_chunk_state(x, Bm, dt, dA)
    torch.cuda.synchronize()
    ref = oracle.ssd_chunk_state(f64(x), f64(Bm), f64(dt), f64(dA), Q)
    print(check(f64(st), ref, f"state B{Bn} L{L} H{H} G{G}"))


@pytest.mark.parametrize("Bn,L,H,G,dtype", SMALL)
def test_chunk_scan_every_element(Bn, L, H, G, dtype):
    x, Bm, C, dt, dA, D = make(Bn, L, H, G, dtype, 29 + L)
    cb, prev = oracle_prev_cb(x, Bm, C, dt, dA, L, dtype)
    out = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
    torch.cuda.synchronize()
    ref = oracle.ssd_chunk_scan(f64(cb), f64(x), f64(dt), f64(dA), f64(C), f64(prev), f64(D), Q)
    print(check(f64(out), ref, f"scan B{Bn} L{L} H{H} G{G}"))


def test_chunk_scan_without_skip_term():
    x, Bm, C, dt, dA, D = make(1, 384, 2, 1, BF, 5)
    cb, prev = oracle_prev_cb(x, Bm, C, dt, dA, 384, BF)
    out = ssd_chunk_scan(cb, x, dt, dA, C, prev, None)
    torch.cuda.synchronize()
    ref = oracle.ssd_chunk_scan(f64(cb), f64(x), f64(dt), f64(dA), f64(C), f64(prev), None, Q)
    check(f64(out), ref, "scan no D")


def test_chained_kernels_reproduce_the_recurrence():
    """GPU chunk_state -> (host) state passing -> GPU chunk_scan equals the SSM recurrence
    evaluated position by position by the oracle (the end-to-end meaning of the two
    kernels); tolerance of the 16-bit intermediates."""
    Bn, L, H, G = 1, 600, 4, 1
    x, Bm, C, dtv, A, D = gen_ssd(Bn, L, H, G, 64, 128, BF, 41, "cuda")
    dt, dA = ssd_chunked_dt(dtv, A, Q)
    st = ssd_chunk_state(x, Bm, dt, dA)
    prev, _ = S.state_passing(f64(st), f64(dA), L, Q)
    cb = torch.as_tensor(S.bmm_chunk(f64(C), f64(Bm), Q)).to(BF).cuda()
    out = ssd_chunk_scan(cb, x, dt, dA, C, torch.as_tensor(prev).to(BF).cuda(), D)
    torch.cuda.synchronize()
    y, _ = oracle.ssd_recurrence(f64(x), f64(dtv), f64(A), f64(Bm), f64(C), f64(D))
    rel = np.linalg.norm(f64(out) - y) / np.linalg.norm(y)
    assert rel <= 2e-2, rel


def test_deterministic_and_launch_count():
    from paper_2504_17577_b200 import tl_attn_last_launch_count
    x, Bm, C, dt, dA, D = make(2, 512, 4, 1, BF, 3)
    a = ssd_chunk_state(x, Bm, dt, dA)
    assert tl_attn_last_launch_count() == 1
    b = ssd_chunk_state(x, Bm, dt, dA)
    cb, prev = oracle_prev_cb(x, Bm, C, dt, dA, 512, BF)
    o1 = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
    assert tl_attn_last_launch_count() == 1
    o2 = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))


def test_argument_errors():
    from paper_2504_17577_b200 import TlAttnError
    x, Bm, C, dt, dA, D = make(1, 256, 2, 1, BF, 1)
    with pytest.raises(TlAttnError):  # odd head count (head pairs)
        ssd_chunk_state(x[:, :, :1].contiguous(), Bm, dt[:, :1].contiguous(), dA[:, :1].contiguous())
    with pytest.raises(TlAttnError):  # dt of the wrong dtype
        ssd_chunk_state(x, Bm, dt.half(), dA)
    with pytest.raises(TlAttnError):  # headdim 32 unsupported
        ssd_chunk_state(x[..., :32].contiguous(), Bm, dt, dA)


# ------------------------------------------------------------------ the paper's Table 4 shapes
TABLE4 = {  # name: (batch, seq_len) — nheads 64, head_dim 64, d_state 128
    "0": (1, 1024), "1": (1, 2048), "2": (1, 8192), "3": (64, 1024), "4": (64, 2048), "5": (64, 8192),
}


def sample_pairs(Bn, nc, rng, n=6):
    pairs = {(0, 0), (Bn - 1, nc - 1)}
    while len(pairs) < min(n, Bn * nc):
        pairs.add((int(rng.integers(Bn)), int(rng.integers(nc))))
    return sorted(pairs)


@pytest.mark.slow
@pytest.mark.parametrize("name", list(TABLE4))
def test_table4_full_size_sampled(name):
    """CT<i> / CC<i> at full size in the launch configuration bench.py times; the oracle
    recomputes every head of sampled chunks (b, c) from the same inputs."""
    Bn, L = TABLE4[name]
    H, G = 64, 1
    nc = L // Q
    x, Bm, C, dt, dA, D = make(Bn, L, H, G, BF, 500 + int(name))
    rng = np.random.default_rng(int(name))
    pairs = sample_pairs(Bn, nc, rng)
    # chunk_state (CT)
    st = ssd_chunk_state(x, Bm, dt, dA)
    # chunk_scan (CC): cb / prev for the sampled chunks from the oracle, the rest random
    cb, prev = gen_ssd_cb_prev(Bn, L, H, G, 64, 128, BF, 600 + int(name), "cuda")
    out = ssd_chunk_scan(cb, x, dt, dA, C, prev, D)
    torch.cuda.synchronize()
    sl = lambda t, b, c: f64(t[b:b + 1, c * Q:(c + 1) * Q])  # noqa: E731
    for (b, c) in pairs:
        xs, Bs, Cs = sl(x, b, c), sl(Bm, b, c), sl(C, b, c)
        dts, dAs = f64(dt[b:b + 1, :, c:c + 1]), f64(dA[b:b + 1, :, c:c + 1])
        ref = oracle.ssd_chunk_state(xs, Bs, dts, dAs, Q)
        check(f64(st[b:b + 1, c:c + 1]), ref, f"CT{name} (b={b}, c={c})")
        ref_o = oracle.ssd_chunk_scan(f64(cb[b:b + 1, c:c + 1]), xs, dts, dAs, Cs,
                                      f64(prev[b:b + 1, c:c + 1]), f64(D), Q)
        check(sl(out, b, c), ref_o, f"CC{name} (b={b}, c={c})")
