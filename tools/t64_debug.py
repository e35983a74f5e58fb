import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2504_17577_b200 import attention
from paper_2504_17577_b200.inputs import gen_qkv
q, k, v = gen_qkv(1, 1, 1, 128, 128, 64, torch.float16, 5, "cuda")
o, l = attention(q, k, v, causal=False)
torch.cuda.synchronize()
print("ok", float(o.float().abs().sum()))
