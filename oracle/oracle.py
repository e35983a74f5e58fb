"""ctypes loader for liboracle.so (plain C, fp64) — TEST INFRASTRUCTURE ONLY.

Inputs are numpy ``uint16`` arrays holding the raw fp16/bf16 bit patterns of
contiguous BSHD tensors (R6). Outputs are float64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ORACLE_F16 = 0
ORACLE_BF16 = 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "attn_oracle.c"), os.path.join(_HERE, "gemm_oracle.c"),
        os.path.join(_HERE, "mla_oracle.c"), os.path.join(_HERE, "ssd_oracle.c")]
_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 (no -ffast-math). Returns the path."""
    newest_src = max(os.path.getmtime(p) for p in _SRC + [os.path.join(_HERE, "oracle.h")])
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest_src:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-Wextra",
               "-o", tmp, *_SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_oracle())
            L, I, D = ctypes.c_long, ctypes.c_int, ctypes.c_double
            P16 = ctypes.POINTER(ctypes.c_uint16)
            PD = ctypes.POINTER(ctypes.c_double)
            PL = ctypes.POINTER(ctypes.c_long)
            lib.oracle_widen.argtypes = [ctypes.c_uint16, I]
            lib.oracle_widen.restype = D
            lib.oracle_attn_rows.argtypes = [P16, P16, P16, I, L, L, L, L, L, L, I, D, L, L,
                                             PL, L, PD, PD]
            lib.oracle_attn_rows.restype = I
            lib.oracle_attn_full.argtypes = [P16, P16, P16, I, L, L, L, L, L, L, I, D, PD, PD]
            lib.oracle_attn_full.restype = I
            lib.oracle_brute_force.argtypes = [P16, P16, P16, I, L, L, L, L, L, L, I, D, L, L,
                                               PD, PD, PD, PD]
            lib.oracle_brute_force.restype = I
            lib.oracle_gemm_rows.argtypes = [P16, P16, I, L, L, L, PL, L, PD]
            lib.oracle_gemm_rows.restype = I
            PI = ctypes.POINTER(ctypes.c_int32)
            lib.oracle_mla_decode.argtypes = [P16, P16, P16, P16, I, PI, L, L, L, L, L, L, D,
                                              PD, PD]
            lib.oracle_mla_decode.restype = I
            lib.oracle_mla_brute.argtypes = [P16, P16, P16, P16, I, PI, L, L, L, L, L, L, D, L,
                                             PD, PD, PD, PD]
            lib.oracle_mla_brute.restype = I
            lib.oracle_ssd_chunk_state.argtypes = [PD, PD, PD, PD, L, L, L, L, L, L, L, PD]
            lib.oracle_ssd_chunk_state.restype = I
            lib.oracle_ssd_chunk_scan.argtypes = [PD, PD, PD, PD, PD, PD, PD, L, L, L, L, L, L,
                                                  L, PD]
            lib.oracle_ssd_chunk_scan.restype = I
            lib.oracle_ssd_recurrence.argtypes = [PD, PD, PD, PD, PD, PD, L, L, L, L, L, L, PD,
                                                  PD]
            lib.oracle_ssd_recurrence.restype = I
            _lib = lib
    return _lib


def _p16(a: np.ndarray):
    assert a.dtype == np.uint16 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16))


def _pd(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _dims(q, k, v):
    assert q.ndim == 4 and k.ndim == 4 and v.ndim == 4 and k.shape == v.shape
    B, Sq, Hq, D = q.shape
    Bk, Skv, Hkv, Dk = k.shape
    assert Bk == B and Dk == D
    return B, Hq, Hkv, Sq, Skv, D


def widen(bits: int, dtype: int) -> float:
    return _load().oracle_widen(ctypes.c_uint16(bits), dtype)


def attn_rows(q, k, v, dtype, causal, scale, b, h, rows):
    """Oracle output for query rows ``rows`` of head (b, h): (o[nrows, D], lse[nrows])."""
    lib = _load()
    B, Hq, Hkv, Sq, Skv, D = _dims(q, k, v)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    n = rows.shape[0]
    o = np.zeros((n, D), np.float64)
    lse = np.zeros((n,), np.float64)
    rc = lib.oracle_attn_rows(_p16(q), _p16(k), _p16(v), dtype, B, Hq, Hkv, Sq, Skv, D,
                              int(causal), float(scale), int(b), int(h),
                              rows.ctypes.data_as(ctypes.POINTER(ctypes.c_long)), n,
                              _pd(o), _pd(lse))
    if rc != 0:
        raise ValueError(f"oracle_attn_rows rejected its arguments (rc={rc})")
    return o, lse


def attn_rows_parallel(q, k, v, dtype, causal, scale, work, threads=None):
    """Run ``attn_rows`` over independent (b, h, rows) items on host threads.

    ``work`` is a list of (b, h, rows). Each call is single-threaded C (ctypes drops
    the GIL), so the items run concurrently. Returns a list of (o, lse).
    """
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        futs = [ex.submit(attn_rows, q, k, v, dtype, causal, scale, b, h, rows)
                for (b, h, rows) in work]
        return [f.result() for f in futs]


def attn_full(q, k, v, dtype, causal, scale):
    """All rows: (o[B,Sq,Hq,D], lse[B,Hq,Sq]) in float64."""
    lib = _load()
    B, Hq, Hkv, Sq, Skv, D = _dims(q, k, v)
    o = np.zeros((B, Sq, Hq, D), np.float64)
    lse = np.zeros((B, Hq, Sq), np.float64)
    rc = lib.oracle_attn_full(_p16(q), _p16(k), _p16(v), dtype, B, Hq, Hkv, Sq, Skv, D,
                              int(causal), float(scale), _pd(o), _pd(lse))
    if rc != 0:
        raise ValueError(f"oracle_attn_full rejected its arguments (rc={rc})")
    return o, lse


def brute_force(q, k, v, dtype, causal, scale, b, h):
    """Explicit-matrix formulation for one (b, h): returns (S, P, O, lse)."""
    lib = _load()
    B, Hq, Hkv, Sq, Skv, D = _dims(q, k, v)
    S = np.zeros((Sq, Skv), np.float64)
    P = np.zeros((Sq, Skv), np.float64)
    O = np.zeros((Sq, D), np.float64)
    lse = np.zeros((Sq,), np.float64)
    rc = lib.oracle_brute_force(_p16(q), _p16(k), _p16(v), dtype, B, Hq, Hkv, Sq, Skv, D,
                                int(causal), float(scale), int(b), int(h),
                                _pd(S), _pd(P), _pd(O), _pd(lse))
    if rc != 0:
        raise ValueError(f"oracle_brute_force rejected its arguments (rc={rc})")
    return S, P, O, lse


def gemm_rows(a, b, dtype, rows):
    """Rows of C = A @ B (A [M,K], B [K,N] uint16 bit patterns) in float64."""
    lib = _load()
    assert a.ndim == 2 and b.ndim == 2 and a.shape[1] == b.shape[0]
    M, K = a.shape
    N = b.shape[1]
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    c = np.zeros((rows.shape[0], N), np.float64)
    rc = lib.oracle_gemm_rows(_p16(a), _p16(b), dtype, M, N, K,
                              rows.ctypes.data_as(ctypes.POINTER(ctypes.c_long)), rows.shape[0],
                              _pd(c))
    if rc != 0:
        raise ValueError(f"oracle_gemm_rows rejected its arguments (rc={rc})")
    return c


def gemm_rows_parallel(a, b, dtype, rows, threads=None):
    threads = threads or len(os.sched_getaffinity(0))
    rows = list(rows)
    # chunks of POSITIONS (a row index may repeat; each position gets its own result)
    pos_chunks = [list(range(i, len(rows), threads)) for i in range(threads) if i < len(rows)]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(lambda ps: gemm_rows(a, b, dtype, [rows[p] for p in ps]), pos_chunks))
    out = np.zeros((len(rows), b.shape[1]), np.float64)
    for ps, c in zip(pos_chunks, res):
        for k, p in enumerate(ps):
            out[p] = c[k]
    return out


# --------------------------------------------------------------------------- MLA decode
def _mla_dims(q, q_pe, kv, k_pe):
    assert q.ndim == 3 and kv.ndim == 4 and q_pe.ndim == 3 and k_pe.ndim == 4
    B, H, Dl = q.shape
    Bk, Skv, Hkv, Dlk = kv.shape
    Dr = q_pe.shape[2]
    assert Bk == B and Dlk == Dl and q_pe.shape[:2] == (B, H)
    assert k_pe.shape == (B, Skv, Hkv, Dr)
    return B, H, Hkv, Skv, Dl, Dr


def _pi32(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def mla_decode(q, q_pe, kv, k_pe, dtype, scale, seqlens=None):
    """Fig. 18 MLA decode, plain fp64 definition: (o[B,H,Dl], lse[B,H])."""
    lib = _load()
    B, H, Hkv, Skv, Dl, Dr = _mla_dims(q, q_pe, kv, k_pe)
    sl = None if seqlens is None else np.ascontiguousarray(np.asarray(seqlens, np.int32))
    o = np.zeros((B, H, Dl), np.float64)
    lse = np.zeros((B, H), np.float64)
    rc = lib.oracle_mla_decode(_p16(q), _p16(q_pe), _p16(kv), _p16(k_pe), dtype, _pi32(sl),
                               B, H, Hkv, Skv, Dl, Dr, float(scale), _pd(o), _pd(lse))
    if rc != 0:
        raise ValueError(f"oracle_mla_decode rejected its arguments (rc={rc})")
    return o, lse


def mla_decode_parallel(q, q_pe, kv, k_pe, dtype, scale, seqlens=None, batches=None,
                        threads=None):
    """mla_decode over independent batches on host threads; returns {b: (o[H,Dl], lse[H])}."""
    B = q.shape[0]
    batches = list(range(B)) if batches is None else list(batches)
    sl = None if seqlens is None else np.asarray(seqlens, np.int32)

    def one(b):
        return b, mla_decode(q[b:b + 1], q_pe[b:b + 1], kv[b:b + 1], k_pe[b:b + 1], dtype,
                             scale, None if sl is None else sl[b:b + 1])
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(one, batches))
    return {b: (o[0], lse[0]) for b, (o, lse) in res}


def mla_brute(q, q_pe, kv, k_pe, dtype, scale, b, seqlens=None):
    """Explicit-matrix MLA for batch b: (S[H,n], P[H,n], O[H,Dl], lse[H])."""
    lib = _load()
    B, H, Hkv, Skv, Dl, Dr = _mla_dims(q, q_pe, kv, k_pe)
    sl = None if seqlens is None else np.ascontiguousarray(np.asarray(seqlens, np.int32))
    n = Skv if sl is None else int(sl[b])
    S = np.zeros((H, n), np.float64)
    P = np.zeros((H, n), np.float64)
    O = np.zeros((H, Dl), np.float64)
    lse = np.zeros((H,), np.float64)
    rc = lib.oracle_mla_brute(_p16(q), _p16(q_pe), _p16(kv), _p16(k_pe), dtype, _pi32(sl),
                              B, H, Hkv, Skv, Dl, Dr, float(scale), int(b),
                              _pd(S), _pd(P), _pd(O), _pd(lse))
    if rc != 0:
        raise ValueError(f"oracle_mla_brute rejected its arguments (rc={rc})")
    return S, P, O, lse


# --------------------------------------------------------------------------- Mamba-2 SSD
# (Table 4; definitions and readings L1-L8 in ssd_oracle.c)
def _d(a):
    return np.ascontiguousarray(np.asarray(a, np.float64))


def ssd_chunk_state(x, Bm, dt, dA, Q):
    """states[B][nc][H][P][N] (fp64) of every chunk; x[B,L,H,P], Bm[B,L,G,N],
    dt/dA[B,H,nc,Q] (any float arrays, widened to fp64)."""
    x, Bm, dt, dA = _d(x), _d(Bm), _d(dt), _d(dA)
    Bn, L, H, P = x.shape
    G, N = Bm.shape[2], Bm.shape[3]
    nc = (L + Q - 1) // Q
    assert Bm.shape[:2] == (Bn, L) and dt.shape == (Bn, H, nc, Q) and dA.shape == dt.shape
    out = np.zeros((Bn, nc, H, P, N), np.float64)
    rc = _load().oracle_ssd_chunk_state(_pd(x), _pd(Bm), _pd(dt), _pd(dA), Bn, L, H, G, P, N,
                                        Q, _pd(out))
    if rc != 0:
        raise ValueError("oracle_ssd_chunk_state rejected its arguments")
    return out


def ssd_chunk_scan(cb, x, dt, dA, C, prev, D, Q):
    """out[B][L][H][P] (fp64); cb[B,nc,G,Q,Q], prev[B,nc,H,P,N], D[H] or None."""
    cb, x, dt, dA, C, prev = _d(cb), _d(x), _d(dt), _d(dA), _d(C), _d(prev)
    Dd = None if D is None else _d(D)
    Bn, L, H, P = x.shape
    G, N = C.shape[2], C.shape[3]
    nc = (L + Q - 1) // Q
    assert cb.shape == (Bn, nc, G, Q, Q) and prev.shape == (Bn, nc, H, P, N)
    assert C.shape[:2] == (Bn, L) and dt.shape == (Bn, H, nc, Q) and dA.shape == dt.shape
    out = np.zeros((Bn, L, H, P), np.float64)
    rc = _load().oracle_ssd_chunk_scan(_pd(cb), _pd(x), _pd(dt), _pd(dA), _pd(C), _pd(prev),
                                       _pd(Dd), Bn, L, H, G, P, N, Q, _pd(out))
    if rc != 0:
        raise ValueError("oracle_ssd_chunk_scan rejected its arguments")
    return out


def ssd_recurrence(x, dtv, A, Bm, C, D):
    """The SSM recurrence position by position: (y[B,L,H,P], final state h[B,H,P,N])."""
    x, dtv, A, Bm, C = _d(x), _d(dtv), _d(A), _d(Bm), _d(C)
    Dd = None if D is None else _d(D)
    Bn, L, H, P = x.shape
    G, N = Bm.shape[2], Bm.shape[3]
    y = np.zeros((Bn, L, H, P), np.float64)
    hf = np.zeros((Bn, H, P, N), np.float64)
    rc = _load().oracle_ssd_recurrence(_pd(x), _pd(dtv), _pd(A), _pd(Bm), _pd(C), _pd(Dd), Bn, L,
                                       H, G, P, N, _pd(y), _pd(hf))
    if rc != 0:
        raise ValueError("oracle_ssd_recurrence rejected its arguments")
    return y, hf


def ssd_sample_chunks(fn, pairs, threads=None):
    """Run fn(b, c) for the given (b, c) pairs on host threads; returns {(b, c): result}."""
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(lambda bc: (bc, fn(*bc)), pairs))
    return dict(res)
