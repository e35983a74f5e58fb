"""The CUDA generator kernel (csrc/gen.cu, libtlgen.so) reproduces the torch-op generator of
inputs.py bit for bit (full tensors, sub-block slices, every dtype), so tests and the bench
draw the same values with one launch per tensor."""
import pytest
import torch

from paper_2504_17577_b200.inputs import gen_tensor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("shape,slices", [
    ((3, 5, 7, 64), None),
    ((4, 33, 8, 128), (slice(1, 3), slice(0, 33), slice(2, 6), slice(0, 128))),
    ((2, 3, 4, 5, 6), (slice(0, 2), slice(1, 3), slice(0, 4), slice(2, 5), slice(0, 6))),
    ((1 << 20,), None),
])
def test_kernel_equals_torch_ops(dtype, shape, slices):
    a = gen_tensor(shape, 77, "q", dtype, "cuda", slices)
    b = gen_tensor(shape, 77, "q", dtype, "cuda", slices, use_kernel=False)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))


def test_large_index_counter_bits():
    """Indices >= 2^31 use the extra counter bits (idx >> 31): a slice far into a big
    virtual tensor matches the torch-op generator."""
    shape = (4, 1 << 30)
    sl = (slice(3, 4), slice((1 << 30) - 4096, 1 << 30))
    a = gen_tensor(shape, 5, "k", torch.bfloat16, "cuda", sl)
    b = gen_tensor(shape, 5, "k", torch.bfloat16, "cuda", sl, use_kernel=False)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
