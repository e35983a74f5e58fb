"""Pins for the fp64 GEMM oracle (Fig. 16 Matmul), CPU only."""
import numpy as np
import pytest
import torch

import oracle
from paper_2504_17577_b200.inputs import from_values, to_bits


def bits(x, dt):
    return to_bits(from_values(np.asarray(x, np.float64), dt))


@pytest.mark.parametrize("dt,code", [(torch.bfloat16, oracle.ORACLE_BF16), (torch.float16, oracle.ORACLE_F16)])
def test_identity_gives_b(dt, code):
    """A = I -> C = B exactly."""
    rng = np.random.default_rng(1)
    B = rng.integers(-20, 20, (7, 5)).astype(np.float64)
    C = oracle.gemm_rows(bits(np.eye(7), dt), bits(B, dt), code, range(7))
    assert np.array_equal(C, B)


def test_integer_matrices_exact():
    """Small-integer inputs: every product and partial sum is exact, so the oracle equals
    exact integer arithmetic (numpy int64 matmul) bit for bit."""
    rng = np.random.default_rng(2)
    A = rng.integers(-8, 9, (9, 33))
    B = rng.integers(-8, 9, (33, 6))
    C = oracle.gemm_rows(bits(A, torch.bfloat16), bits(B, torch.bfloat16), oracle.ORACLE_BF16, range(9))
    assert np.array_equal(C, (A @ B).astype(np.float64))


def test_rank_one_closed_form_and_transposition():
    """A = u 1^T, B = 1 v^T -> C_ij = K u_i v_j; a transposed operand would break the
    i/j dependence (u and v differ and M != N)."""
    u = np.array([1.0, -2.0, 3.0])
    v = np.array([0.5, 4.0, -1.0, 2.0, 8.0])
    K = 6
    A = np.outer(u, np.ones(K))
    B = np.outer(np.ones(K), v)
    C = oracle.gemm_rows(bits(A, torch.float16), bits(B, torch.float16), oracle.ORACLE_F16, [2, 0])
    np.testing.assert_array_equal(C, K * np.outer(u[[2, 0]], v))


def test_hand_example():
    """[[1,2],[3,4]] @ [[5,6],[7,8]] = [[19,22],[43,50]] (worked by hand)."""
    C = oracle.gemm_rows(bits([[1, 2], [3, 4]], torch.bfloat16), bits([[5, 6], [7, 8]], torch.bfloat16),
                         oracle.ORACLE_BF16, [0, 1])
    np.testing.assert_array_equal(C, [[19, 22], [43, 50]])


def test_parallel_rows_and_bad_args():
    rng = np.random.default_rng(3)
    a = bits(rng.standard_normal((20, 16)), torch.bfloat16)
    b = bits(rng.standard_normal((16, 12)), torch.bfloat16)
    rows = [19, 0, 7, 3]
    assert np.array_equal(oracle.gemm_rows_parallel(a, b, oracle.ORACLE_BF16, rows, threads=3),
                          oracle.gemm_rows(a, b, oracle.ORACLE_BF16, rows))
    with pytest.raises(ValueError):
        oracle.gemm_rows(a, b, oracle.ORACLE_BF16, [20])


def test_parallel_rows_keep_positions_of_repeated_rows():
    """gemm_rows_parallel returns one result per requested position (repeats included)."""
    rng = np.random.default_rng(3)
    a = bits(rng.standard_normal((3, 16)), torch.bfloat16)
    b = bits(rng.standard_normal((16, 8)), torch.bfloat16)
    got = oracle.gemm_rows_parallel(a, b, oracle.ORACLE_BF16, [2, 0, 2, 2], threads=3)
    one = oracle.gemm_rows(a, b, oracle.ORACLE_BF16, [2, 0])
    assert np.array_equal(got, one[[0, 1, 0, 0]])
