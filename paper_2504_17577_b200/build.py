"""Build libtlattn.so in-tree: nvcc for sm_100a (cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtlattn.so")
SOURCES = [os.path.join(CSRC, "tlattn_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(ROOT, "include", "tlattn.h")]
# the seeded input generator as one CUDA kernel (test / bench infrastructure, inputs.py)
GEN_LIB = os.path.join(PKG, "libtlgen.so")
GEN_SRC = os.path.join(CSRC, "gen.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-shared",
]


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(GEN_LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS if os.path.exists(p)) or \
        os.path.getmtime(GEN_SRC) > os.path.getmtime(GEN_LIB)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-o", tmp, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libtlattn.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    tmpg = GEN_LIB + f".tmp{os.getpid()}"
    r = subprocess.run([NVCC, *NVCC_FLAGS, "-o", tmpg, GEN_SRC], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libtlgen.so")
    os.replace(tmpg, GEN_LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
