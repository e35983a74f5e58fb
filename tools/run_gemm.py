"""Time tl_gemm vs cuBLAS (torch.matmul) on PAPER.md Table 2 M-shapes (bf16).
  python tools/run_gemm.py [M5 M2 ...]"""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_17577_b200 import gemm

TABLE2 = {"M0": (4096, 1024, 8192), "M1": (4096, 8192, 8192), "M2": (4096, 28672, 8192),
          "M3": (4096, 8192, 28672), "M4": (8192, 1024, 8192), "M5": (8192, 8192, 8192),
          "M6": (8192, 28672, 8192), "M7": (8192, 8192, 28672),
          # GEMV rows (m = 1): HBM-bound, reported in GB/s of B read
          "V0": (1, 16384, 16384), "V1": (1, 43008, 14336), "V2": (1, 14336, 14336),
          "V3": (1, 57344, 14336), "V4": (1, 14336, 57344), "V5": (1, 9216, 9216),
          "V6": (1, 36864, 9216), "V7": (1, 9216, 36864)}


def bench(fn, iters=10):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); ev.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev)


def main():
    names = sys.argv[1:] or sorted(TABLE2)
    for n in names:
        M, N, K = TABLE2[n]
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        b = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t_ours = bench(lambda: gemm(a, b, out=c))
        t_cublas = bench(lambda: torch.matmul(a, b, out=c))
        fl = 2.0 * M * N * K
        by = 2.0 * (M * K + K * N + M * N)
        print(f"{n} {M}x{N}x{K}: tl_gemm {fl / t_ours / 1e9:7.1f} TFLOP/s {by / t_ours / 1e6:7.0f} GB/s "
              f"({t_ours:.3f} ms)  cuBLAS {fl / t_cublas / 1e9:7.1f} TFLOP/s "
              f"{by / t_cublas / 1e6:7.0f} GB/s  ratio {t_cublas / t_ours:.3f}")


if __name__ == "__main__":
    main()
