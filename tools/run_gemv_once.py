import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2504_17577_b200 import gemm
from paper_2504_17577_b200.inputs import gen_tensor
M, N, K = 1, 14336, 57344
a = gen_tensor((M, K), 2024, "q", torch.bfloat16, "cuda")
b = gen_tensor((K, N), 2024, "k", torch.bfloat16, "cuda")
c = gemm(a, b); torch.cuda.synchronize()
c = gemm(a, b); torch.cuda.synchronize()
