"""Seeded synthetic inputs shared by the tests, the bench and the oracle checks.

This module holds NO attention arithmetic: it only draws Q/K/V values. It is the one
module both the CUDA path's callers and the oracle's callers use (DESIGN.md "Input
recipe", reading R11).

Recipe: Q, K, V iid N(0, 1) rounded round-to-nearest-even to the config dtype,
contiguous BSHD. Each element is a pure function of (seed, tensor id, global BSHD
linear index) — a counter-based generator — so a shard of a tensor (a batch or head
slice) is bit-identical to the same slice of the unsharded tensor.

Generator: u32 = lowbias32(counter ^ key) (two rounds), uniforms from the top 24 bits,
Box-Muller in fp32. Integer hashing is done in int64 torch ops masked to 32 bits so
it runs identically on CPU and CUDA tensors. On CUDA devices gen_tensor runs the same
generator as ONE kernel per tensor (csrc/gen.cu, libtlgen.so; bit-identical to the torch
ops, tests/test_inputs_gpu.py) instead of dozens of elementwise launches per chunk.
"""
from __future__ import annotations

import math

import numpy as np
import torch

TENSOR_ID = {"q": 1, "k": 2, "v": 3, "q_pe": 4, "kv": 5, "k_pe": 6, "seqlens": 7,
             # Mamba-2 SSD chunk kernels (reading L8)
             "ssd_x": 8, "ssd_B": 9, "ssd_C": 10, "ssd_dt": 11, "ssd_A": 12, "ssd_D": 13,
             "ssd_cb": 14, "ssd_prev": 15}
_M32 = 0xFFFFFFFF


def _lowbias32(x: torch.Tensor) -> torch.Tensor:
    # x holds values in [0, 2^32) as int64; products wrap mod 2^64 and are masked to 32 bits
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & _M32
    x = x ^ (x >> 16)
    return x


def _key(seed: int, tensor_id: int) -> int:
    h = (seed * 0x9E3779B1 + tensor_id * 0x85EBCA77 + 0x165667B1) & _M32
    # scramble on the host with the same hash
    return int(_lowbias32(torch.tensor([h], dtype=torch.int64)).item())


def normal_from_index(idx: torch.Tensor, seed: int, tensor_id: int) -> torch.Tensor:
    """N(0,1) fp32 values for int64 global indices ``idx`` (any device)."""
    key = _key(seed, tensor_id)
    c0 = (idx * 2) & _M32
    c1 = (idx * 2 + 1) & _M32
    hi = (idx >> 31) & _M32  # extra counter bits for tensors with > 2^31 elements
    h0 = _lowbias32(_lowbias32(c0 ^ key) ^ hi)
    h1 = _lowbias32(_lowbias32(c1 ^ key) ^ hi)
    u1 = ((h0 >> 8).to(torch.float32) + 0.5) * (1.0 / 16777216.0)
    u2 = ((h1 >> 8).to(torch.float32) + 0.5) * (1.0 / 16777216.0)
    r = torch.sqrt(-2.0 * torch.log(u1))
    return r * torch.cos((2.0 * math.pi) * u2)


def uniform_from_index(idx: torch.Tensor, seed: int, tensor_id: int) -> torch.Tensor:
    """U(0, 1) fp32 values (open interval) for int64 global indices (any device)."""
    key = _key(seed, tensor_id)
    h = _lowbias32(_lowbias32((idx & _M32) ^ key) ^ ((idx >> 31) & _M32))
    return ((h >> 8).to(torch.float32) + 0.5) * (1.0 / 16777216.0)


_gen_lib = None


def _gen_library():
    """libtlgen.so (built by build.py next to libtlattn.so), or None if absent."""
    global _gen_lib
    if _gen_lib is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtlgen.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        P, I = ctypes.c_void_p, ctypes.c_int
        lib.tl_gen_normal.argtypes = [P, I, I, P, P, P, ctypes.c_uint32, P]
        lib.tl_gen_normal.restype = I
        _gen_lib = lib
    return _gen_lib


def _gen_cuda(out, shape, ranges, tid, seed, use_kernel=True):
    import numpy as np_
    lib = _gen_library() if use_kernel else None
    if lib is None:
        return False
    code = {torch.float16: 0, torch.bfloat16: 1, torch.float32: 2}.get(out.dtype)
    if code is None:
        return False
    nd = len(shape)
    sh = np_.array(shape, np_.int64)
    st = np_.array([r.start for r in ranges], np_.int64)
    osz = np_.array([len(r) for r in ranges], np_.int64)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = lib.tl_gen_normal(out.data_ptr(), code, nd, sh.ctypes.data, st.ctypes.data,
                           osz.ctypes.data, _key(seed, tid), stream)
    if rc != 0:
        raise RuntimeError(f"tl_gen_normal failed ({rc})")
    return True


def gen_tensor(shape, seed: int, name: str, dtype: torch.dtype, device,
               slices=None, chunk: int = 1 << 25, use_kernel: bool = True) -> torch.Tensor:
    """Contiguous tensor of ``shape`` (global BSHD shape), optionally a sub-block.

    ``slices`` is a tuple of python ``slice`` objects over the global shape (step 1);
    the result holds exactly those elements of the global tensor.
    """
    shape = tuple(int(s) for s in shape)
    if slices is None:
        slices = tuple(slice(0, s) for s in shape)
    ranges = [range(*sl.indices(s)) for sl, s in zip(slices, shape)]
    out_shape = tuple(len(r) for r in ranges)
    out = torch.empty(out_shape, dtype=dtype, device=device)
    n = out.numel()
    if n == 0:
        return out
    strides = [1] * len(shape)
    for i in range(len(shape) - 2, -1, -1):
        strides[i] = strides[i + 1] * shape[i + 1]
    flat = out.view(-1)
    # Enumerate local linear indices in chunks and map them to global linear indices.
    out_strides = [1] * len(out_shape)
    for i in range(len(out_shape) - 2, -1, -1):
        out_strides[i] = out_strides[i + 1] * out_shape[i + 1]
    tid = TENSOR_ID[name]
    if out.is_cuda and len(shape) <= 6 and _gen_cuda(out, shape, ranges, tid, seed, use_kernel):
        return out
    for start in range(0, n, chunk):
        stop = min(n, start + chunk)
        loc = torch.arange(start, stop, dtype=torch.int64, device=device)
        gidx = torch.zeros_like(loc)
        rem = loc
        for dim in range(len(out_shape)):
            coord = rem // out_strides[dim]
            rem = rem - coord * out_strides[dim]
            gidx += (coord + ranges[dim].start) * strides[dim]
        flat[start:stop] = normal_from_index(gidx, seed, tid).to(dtype)
    return out


def gen_qkv(B, Hq, Hkv, Sq, Skv, D, dtype, seed, device, b_slice=None, hq_slice=None,
            hkv_slice=None):
    """Q[B,Sq,Hq,D], K/V[B,Skv,Hkv,D] (or the given batch/head shard of them)."""
    bs = b_slice or slice(0, B)
    q = gen_tensor((B, Sq, Hq, D), seed, "q", dtype, device,
                   (bs, slice(0, Sq), hq_slice or slice(0, Hq), slice(0, D)))
    k = gen_tensor((B, Skv, Hkv, D), seed, "k", dtype, device,
                   (bs, slice(0, Skv), hkv_slice or slice(0, Hkv), slice(0, D)))
    v = gen_tensor((B, Skv, Hkv, D), seed, "v", dtype, device,
                   (bs, slice(0, Skv), hkv_slice or slice(0, Hkv), slice(0, D)))
    return q, k, v


def gen_mla(B, H, Hkv, Skv, Dl, Dr, dtype, seed, device):
    """MLA decode inputs (Fig. 18): q[B,H,Dl], q_pe[B,H,Dr],
    kv[B,Skv,Hkv,Dl], k_pe[B,Skv,Hkv,Dr], iid N(0,1) rounded RN to ``dtype``."""
    q = gen_tensor((B, H, Dl), seed, "q", dtype, device)
    q_pe = gen_tensor((B, H, Dr), seed, "q_pe", dtype, device)
    kv = gen_tensor((B, Skv, Hkv, Dl), seed, "kv", dtype, device)
    k_pe = gen_tensor((B, Skv, Hkv, Dr), seed, "k_pe", dtype, device)
    return q, q_pe, kv, k_pe


def gen_seqlens(B, Skv, seed, lo=1):
    """Ragged per-batch cache lengths, uniform integers in [lo, Skv] (int32 numpy),
    from the same counter-based hash (reading M1)."""
    key = _key(seed, TENSOR_ID["seqlens"])
    h = _lowbias32(_lowbias32(torch.arange(B, dtype=torch.int64) ^ key))
    span = Skv - lo + 1
    return (lo + (h % span)).to(torch.int32).numpy()


def to_bits(t: torch.Tensor) -> np.ndarray:
    """Raw 16-bit patterns of an fp16/bf16 tensor as a host numpy uint16 array."""
    assert t.dtype in (torch.float16, torch.bfloat16)
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view(np.uint16)


def from_values(values, dtype: torch.dtype, device="cpu") -> torch.Tensor:
    """Tensor of the given (float) values rounded RN to ``dtype``."""
    return torch.as_tensor(np.asarray(values, dtype=np.float32)).to(dtype).to(device)


def gen_ssd(B, L, H, G, P, N, dtype, seed, device):
    """Mamba-2 SSD inputs (Table 4; reading L8), drawn like the
    Mamba-2 initialisation: x[B,L,H,P], Bm / C [B,L,G,N] iid N(0,1) rounded to ``dtype``;
    per-position step sizes dt[B,L,H] log-uniform in [1e-3, 1e-1] (fp32); A[H] = -U[1, 16]
    (fp32); D[H] = U[0.5, 1.5] (fp32)."""
    x = gen_tensor((B, L, H, P), seed, "ssd_x", dtype, device)
    Bm = gen_tensor((B, L, G, N), seed, "ssd_B", dtype, device)
    C = gen_tensor((B, L, G, N), seed, "ssd_C", dtype, device)
    n_dt = B * L * H
    u = uniform_from_index(torch.arange(n_dt, dtype=torch.int64, device=device), seed,
                           TENSOR_ID["ssd_dt"])
    dtv = torch.exp(math.log(1e-3) + u * (math.log(1e-1) - math.log(1e-3))).view(B, L, H)
    ua = uniform_from_index(torch.arange(H, dtype=torch.int64, device=device), seed,
                            TENSOR_ID["ssd_A"])
    A = -(1.0 + 15.0 * ua)
    ud = uniform_from_index(torch.arange(H, dtype=torch.int64, device=device), seed,
                            TENSOR_ID["ssd_D"])
    D = 0.5 + ud
    return x, Bm, C, dtv.float(), A.float(), D.float()


def ssd_chunked_dt(dtv, A, Q):
    """The chunked step-size and cumulative-decay inputs of both chunk kernels (reading L4):
    dt[B,H,nc,Q] and dA[b,h,c,i] = sum_{j <= i} dt A_h inside chunk c (fp32; entries past the
    sequence end are 0). Input preparation (Mamba-2 computes dA_cumsum before the chunk
    kernels); accumulated in fp64 on the tensor's device, then rounded to fp32."""
    Bn, L, H = dtv.shape
    nc = (L + Q - 1) // Q
    dt_c = torch.zeros((Bn, nc * Q, H), dtype=torch.float64, device=dtv.device)
    dt_c[:, :L] = dtv.double()
    dt_c = dt_c.view(Bn, nc, Q, H).permute(0, 3, 1, 2).contiguous()  # [B, H, nc, Q]
    dA = torch.cumsum(dt_c * A.double().view(1, H, 1, 1), dim=3)
    return dt_c.float().contiguous(), dA.float().contiguous()


def gen_ssd_cb_prev(B, L, H, G, P, N, dtype, seed, device, Q=256):
    """Bench-only stand-ins for the two inputs chunk_scan takes from earlier pipeline steps
    (reading L8): cb[B,nc,G,Q,Q] iid N(0, N) (the spread of a C.B^T entry) and the entering
    states prev[B,nc,H,P,N] iid N(0,1), both rounded to ``dtype``."""
    nc = (L + Q - 1) // Q
    cb = gen_tensor((B, nc, G, Q, Q), seed, "ssd_cb", torch.float32, device) * math.sqrt(N)
    prev = gen_tensor((B, nc, H, P, N), seed, "ssd_prev", dtype, device)
    return cb.to(dtype), prev
