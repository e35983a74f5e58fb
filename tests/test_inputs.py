"""The seeded input generator (no attention arithmetic): determinism, shard
consistency and distribution."""
import numpy as np
import torch

from paper_2504_17577_b200.inputs import gen_qkv, gen_tensor, normal_from_index


def test_generator_is_deterministic_and_seeded():
    a = gen_tensor((2, 8, 4, 16), 1001, "q", torch.bfloat16, "cpu")
    b = gen_tensor((2, 8, 4, 16), 1001, "q", torch.bfloat16, "cpu")
    c = gen_tensor((2, 8, 4, 16), 1002, "q", torch.bfloat16, "cpu")
    d = gen_tensor((2, 8, 4, 16), 1001, "k", torch.bfloat16, "cpu")
    assert torch.equal(a, b)
    assert not torch.equal(a, c) and not torch.equal(a, d)


def test_shards_are_slices_of_the_global_tensor():
    B, S, H, D = 4, 6, 8, 16
    full = gen_tensor((B, S, H, D), 5, "v", torch.float16, "cpu")
    head = gen_tensor((B, S, H, D), 5, "v", torch.float16, "cpu",
                      (slice(0, B), slice(0, S), slice(2, 6), slice(0, D)))
    batch = gen_tensor((B, S, H, D), 5, "v", torch.float16, "cpu",
                       (slice(1, 3), slice(0, S), slice(0, H), slice(0, D)))
    assert torch.equal(head, full[:, :, 2:6].contiguous())
    assert torch.equal(batch, full[1:3])
    q, k, v = gen_qkv(B, 8, 4, S, S, D, torch.bfloat16, 3, "cpu", hq_slice=slice(4, 8), hkv_slice=slice(2, 4))
    qf, kf, vf = gen_qkv(B, 8, 4, S, S, D, torch.bfloat16, 3, "cpu")
    assert torch.equal(q, qf[:, :, 4:8]) and torch.equal(k, kf[:, :, 2:4]) and torch.equal(v, vf[:, :, 2:4])


def test_distribution_is_standard_normal():
    z = normal_from_index(torch.arange(1 << 20, dtype=torch.int64), 1003, 1).double()
    assert abs(z.mean().item()) < 5e-3
    assert abs(z.std().item() - 1.0) < 5e-3
    # fraction within one sigma ~ 0.6827
    assert abs((z.abs() < 1).double().mean().item() - 0.6827) < 3e-3
    assert torch.isfinite(z).all()
    _ = np  # numpy imported for parity with the other test modules
