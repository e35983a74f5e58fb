"""GPU parity for tl_gemm (C = A @ B, Fig. 16; Table 2 shapes) against the fp64
oracle. Bar: per element |C - C_ref| <= 2^-7 (|C_ref| + rms(C_ref))
(bf16/fp16 output rounding is 2^-9 / 2^-12 relative; fp32 accumulation adds far less),
and relative L2 <= 5e-3 over the checked rows."""
import numpy as np
import pytest
import torch

import oracle
from paper_2504_17577_b200 import TlAttnError, gemm, tl_attn_last_launch_count
from paper_2504_17577_b200.inputs import gen_tensor, to_bits

pytestmark = pytest.mark.gpu

TABLE2 = {  # PAPER.md Table 2: name -> (m, n, k)
    "M0": (4096, 1024, 8192), "M1": (4096, 8192, 8192), "M2": (4096, 28672, 8192),
    "M3": (4096, 8192, 28672), "M4": (8192, 1024, 8192), "M5": (8192, 8192, 8192),
    "M6": (8192, 28672, 8192), "M7": (8192, 8192, 28672),
}
TABLE2_V = {  # the GEMV rows of Table 2 (m = 1): tl_gemm's M = 1 path (gemv_sm100.cuh)
    "V0": (1, 16384, 16384), "V1": (1, 43008, 14336), "V2": (1, 14336, 14336),
    "V3": (1, 57344, 14336), "V4": (1, 14336, 57344), "V5": (1, 9216, 9216),
    "V6": (1, 36864, 9216), "V7": (1, 9216, 36864),
}


def make(M, N, K, dt, seed):
    a = gen_tensor((M, K), seed, "q", dt, "cuda")
    b = gen_tensor((K, N), seed, "k", dt, "cuda")
    return a, b


def check(a, b, c, rows):
    code = oracle.ORACLE_BF16 if a.dtype == torch.bfloat16 else oracle.ORACLE_F16
    ref = oracle.gemm_rows_parallel(to_bits(a), to_bits(b), code, rows)
    got = c[torch.tensor(rows, device=c.device)].double().cpu().numpy()
    rms = float(np.sqrt(np.mean(ref ** 2)))
    err = np.abs(got - ref)
    assert np.all(np.isfinite(got))
    assert np.all(err <= 2.0 ** -7 * (np.abs(ref) + rms)), float((err / (np.abs(ref) + rms)).max())
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert rel <= 5e-3, rel
    return rel


@pytest.mark.parametrize("M,N,K,dt", [
    (300, 264, 200, torch.bfloat16),     # ragged in every dimension (tile 256, K stage 64)
    (256, 256, 64, torch.float16),       # exactly one tile, one K stage
    (1, 8, 8, torch.bfloat16),           # degenerate
    (513, 520, 1000, torch.float16),
])
def test_gemm_parity_small(M, N, K, dt):
    a, b = make(M, N, K, dt, 7 + M)
    c = gemm(a, b)
    torch.cuda.synchronize()
    assert tl_attn_last_launch_count() == 1
    check(a, b, c, list(range(M)))


@pytest.mark.parametrize("name", sorted(TABLE2))
def test_gemm_table2_shapes(name):
    M, N, K = TABLE2[name]
    a, b = make(M, N, K, torch.bfloat16, 11)
    c = gemm(a, b)
    torch.cuda.synchronize()
    rows = sorted({0, 1, 127, 128, 255, 256, M // 2, M - 129, M - 128, M - 1} |
                  set(np.random.default_rng(5).integers(0, M, 6).tolist()))
    check(a, b, c, rows)


def test_gemm_matches_torch_closely():
    """Against cuBLAS (torch.matmul, also fp32-accumulated): same value up to output
    rounding differences."""
    a, b = make(1024, 2048, 4096, torch.bfloat16, 3)
    c = gemm(a, b)
    ref = torch.matmul(a, b)
    torch.cuda.synchronize()
    d = (c.float() - ref.float()).abs()
    assert float(d.max()) <= 2.0 ** -6 * float(ref.float().abs().max())


def test_gemm_bad_args():
    a = torch.empty((16, 12), dtype=torch.bfloat16, device="cuda")  # K=12 not multiple of 8
    b = torch.empty((12, 16), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(TlAttnError) as e:
        gemm(a, b)
    assert e.value.status == 2


@pytest.mark.parametrize("N,K,dt", [
    (264, 1000, torch.bfloat16),    # ragged K split over the cluster, N below one tile
    (8192, 1000, torch.float16),    # K split with ragged 8-row load groups
    (1000, 8, torch.bfloat16),      # one row per CTA of the K split at most
    (57344, 64, torch.float16),     # many column tiles
])
def test_gemv_parity(N, K, dt):
    """M = 1 (GEMV path): every output element against the fp64 oracle."""
    a, b = make(1, N, K, dt, 31 + N + K)
    c = gemm(a, b)
    torch.cuda.synchronize()
    assert tl_attn_last_launch_count() == 1
    check(a, b, c, [0])


@pytest.mark.parametrize("name", sorted(TABLE2_V))
def test_gemv_table2_shapes(name):
    """The paper's GEMV shapes at full size, every output element."""
    M, N, K = TABLE2_V[name]
    a, b = make(M, N, K, torch.bfloat16, 77)
    c = gemm(a, b)
    torch.cuda.synchronize()
    check(a, b, c, [0])
    del a, b, c
    torch.cuda.empty_cache()

