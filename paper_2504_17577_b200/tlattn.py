"""Thin Python binding of libtlattn (include/tlattn.h): argument marshalling only.

Every step of the attention forward runs in the CUDA kernels of libtlattn.so; this
module only turns torch tensors into pointers/sizes and raises on error codes.
PyTorch is used for device memory and streams. There is no CPU fallback: if the
library is missing or the device is not sm_100 the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import torch

from .build import LIB

TL_DTYPE_F16 = 0
TL_DTYPE_BF16 = 1
TL_OK, TL_ERR_INVALID_VALUE, TL_ERR_UNSUPPORTED, TL_ERR_CUDA, TL_ERR_TIMEOUT = 0, 1, 2, 3, 4
TL_PEER_FLAG_WORDS, TL_PEER_STATUS_WORD = 16, 15  # include/tlattn.h
# experiment / test options (include/tlattn.h tl_option)
TL_OPT_FORCE_1CTA, TL_OPT_UNIT_TILES, TL_OPT_LPT, TL_OPT_GEMV_TC, TL_OPT_MLA_HC, TL_OPT_MLA_CL = range(6)

_lock = threading.Lock()
_lib = None


class TlAttnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def load_library(path: str | None = None):
    """Load libtlattn.so (in-tree). Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or os.environ.get("TLATTN_LIB") or LIB
        if not os.path.exists(path):
            raise RuntimeError(f"libtlattn.so not found at {path}: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        I, F, P, U64 = ctypes.c_int, ctypes.c_float, ctypes.c_void_p, ctypes.c_uint64
        lib.tl_attn_fwd.argtypes = [P, P, P, P, P, I, I, I, I, I, I, I, F, I, P]
        lib.tl_attn_fwd.restype = I
        lib.tl_attn_fwd_host.argtypes = [P, P, P, P, P, I, I, I, I, I, I, I, F, I, P, U64, P]
        lib.tl_attn_fwd_host.restype = I
        lib.tl_attn_host_workspace_bytes.argtypes = [I, I, I, I, I, I, I]
        lib.tl_attn_host_workspace_bytes.restype = U64
        lib.tl_attn_strerror.argtypes = [I]
        lib.tl_attn_strerror.restype = ctypes.c_char_p
        lib.tl_attn_version.argtypes = []
        lib.tl_attn_version.restype = I
        lib.tl_gemm.argtypes = [P, P, P, I, I, I, I, P]
        lib.tl_gemm.restype = I
        lib.tl_mla_decode.argtypes = [P, P, P, P, P, P, P, I, I, I, I, I, I, F, I, P, U64, P]
        lib.tl_mla_decode.restype = I
        lib.tl_mla_decode_workspace_bytes.argtypes = [I, I, I]
        lib.tl_mla_decode_workspace_bytes.restype = U64
        lib.tl_attn_last_launch_count.argtypes = []
        lib.tl_attn_last_launch_count.restype = I
        PP = ctypes.POINTER(ctypes.c_void_p)
        lib.tl_attn_fwd_replicated.argtypes = [P, P, P, PP, PP, I, I, I, I, I, I, I, I, I, I, I, I,
                                               F, I, P]
        lib.tl_attn_fwd_replicated.restype = I
        lib.tl_peer_barrier.argtypes = [PP, I, I, ctypes.c_uint32, P]
        lib.tl_peer_barrier.restype = I
        lib.tl_peer_barrier_set_timeout_ns.argtypes = [U64]
        lib.tl_peer_barrier_set_timeout_ns.restype = I
        lib.tl_peer_barrier_check.argtypes = [P]
        lib.tl_peer_barrier_check.restype = I
        lib.tl_ssd_chunk_state.argtypes = [P, P, P, P, P, I, I, I, I, I, I, I, I, P]
        lib.tl_ssd_chunk_state.restype = I
        lib.tl_ssd_chunk_scan.argtypes = [P, P, P, P, P, P, P, P, I, I, I, I, I, I, I, I, P]
        lib.tl_ssd_chunk_scan.restype = I
        lib.tl_attn_set_option.argtypes = [I, I]
        lib.tl_attn_set_option.restype = I
        lib.tl_attn_get_option.argtypes = [I]
        lib.tl_attn_get_option.restype = I
        lib.tl_ipc_handle_bytes.argtypes = []
        lib.tl_ipc_handle_bytes.restype = I
        lib.tl_ipc_get_handle.argtypes = [P, P]
        lib.tl_ipc_get_handle.restype = I
        lib.tl_ipc_open_handle.argtypes = [P, PP]
        lib.tl_ipc_open_handle.restype = I
        lib.tl_ipc_close_handle.argtypes = [P]
        lib.tl_ipc_close_handle.restype = I
        _lib = lib
        return lib


def tl_attn_strerror(status: int) -> str:
    return load_library().tl_attn_strerror(int(status)).decode()


def tl_attn_version() -> int:
    return load_library().tl_attn_version()


def tl_attn_last_launch_count() -> int:
    return load_library().tl_attn_last_launch_count()


def _check(rc: int):
    if rc != TL_OK:
        raise TlAttnError(rc, tl_attn_strerror(rc))


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(stream, device_index=None):
    if stream is None:
        if _raw_stream is not None and device_index is not None:
            return _raw_stream(device_index)  # no Stream object per call (host overhead)
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float16:
        return TL_DTYPE_F16
    if dt == torch.bfloat16:
        return TL_DTYPE_BF16
    raise TlAttnError(TL_ERR_INVALID_VALUE, f"unsupported dtype {dt}")


def tl_attn_fwd(q, k, v, o, lse, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype, stream=None):
    """Direct mirror of the C entry point (device pointers or tensors)."""
    dev = q.get_device() if isinstance(q, torch.Tensor) else None
    _check(load_library().tl_attn_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                      int(B), int(Hq), int(Hkv), int(Sq), int(Skv), int(D),
                                      int(causal), float(scale), int(dtype),
                                      _stream_handle(stream, dev)))


def _ptr_array(ptrs):
    if ptrs is None:
        return None
    arr = (ctypes.c_void_p * len(ptrs))(*[_ptr(x) for x in ptrs])
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))


def tl_attn_fwd_replicated(q, k, v, o_outs, lse_outs, B_total, b_off, Hq_total, h_off, B, Hq, Hkv,
                           Sq, Skv, D, causal, scale, dtype, stream=None):
    """Direct mirror of the C entry point: this rank's shard written into every output in
    ``o_outs`` (device pointers valid in this process, e.g. IPC-mapped peer buffers)."""
    dev = q.get_device() if isinstance(q, torch.Tensor) else None
    oa = _ptr_array(o_outs)
    la = _ptr_array(lse_outs)
    _check(load_library().tl_attn_fwd_replicated(
        _ptr(q), _ptr(k), _ptr(v), oa, la, len(o_outs), int(B_total), int(b_off), int(Hq_total),
        int(h_off), int(B), int(Hq), int(Hkv), int(Sq), int(Skv), int(D), int(causal), float(scale),
        int(dtype), _stream_handle(stream, dev)))


def tl_peer_barrier(flags, rank, epoch, stream=None):
    """Device-side barrier over the ranks whose flag arrays are ``flags`` (one per rank,
    TL_PEER_FLAG_WORDS uint32 each). Bounded: see tl_peer_barrier_check."""
    _check(load_library().tl_peer_barrier(_ptr_array(flags), len(flags), int(rank),
                                          int(epoch) & 0xFFFFFFFF, _stream_handle(stream)))


def tl_attn_set_option(option, value):
    _check(load_library().tl_attn_set_option(int(option), int(value)))


def tl_attn_get_option(option) -> int:
    return int(load_library().tl_attn_get_option(int(option)))


class option:
    """Context manager: set an experiment option (TL_OPT_*) and restore it afterwards."""

    def __init__(self, opt, value):
        self.opt, self.value = opt, value

    def __enter__(self):
        self.old = tl_attn_get_option(self.opt)
        tl_attn_set_option(self.opt, self.value)
        return self

    def __exit__(self, *a):
        tl_attn_set_option(self.opt, self.old)


def tl_peer_barrier_set_timeout_ns(ns):
    _check(load_library().tl_peer_barrier_set_timeout_ns(int(ns)))


def tl_peer_barrier_check(own_flags):
    """Synchronise the device and raise TlAttnError(TL_ERR_TIMEOUT) if a barrier on these
    (own) flags timed out."""
    _check(load_library().tl_peer_barrier_check(_ptr(own_flags)))


def tl_ipc_get_handle(t) -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(lib.tl_ipc_handle_bytes())
    _check(lib.tl_ipc_get_handle(_ptr(t), buf))
    return buf.raw


def tl_ipc_open_handle(handle: bytes) -> int:
    out = ctypes.c_void_p()
    _check(load_library().tl_ipc_open_handle(ctypes.c_char_p(handle), ctypes.byref(out)))
    return int(out.value)


def tl_ipc_close_handle(ptr: int):
    _check(load_library().tl_ipc_close_handle(ptr))


def tl_attn_host_workspace_bytes(B, Hq, Hkv, Sq, Skv, D, with_lse=True) -> int:
    return int(load_library().tl_attn_host_workspace_bytes(B, Hq, Hkv, Sq, Skv, D, int(with_lse)))


def tl_attn_fwd_host(q_h, k_h, v_h, o_h, lse_h, B, Hq, Hkv, Sq, Skv, D, causal, scale, dtype,
                     ws, ws_bytes, stream=None):
    """Direct mirror of the C host-buffer entry point."""
    _check(load_library().tl_attn_fwd_host(_ptr(q_h), _ptr(k_h), _ptr(v_h), _ptr(o_h), _ptr(lse_h),
                                           int(B), int(Hq), int(Hkv), int(Sq), int(Skv), int(D),
                                           int(causal), float(scale), int(dtype), _ptr(ws),
                                           int(ws_bytes), _stream_handle(stream)))


def _dims(q, k, v):
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4 or k.shape != v.shape:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "expected BSHD q[B,Sq,Hq,D], k/v[B,Skv,Hkv,D]")
    B, Sq, Hq, D = q.shape
    Bk, Skv, Hkv, Dk = k.shape
    if Bk != B or Dk != D or q.dtype != k.dtype or q.dtype != v.dtype:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "q/k/v batch, head_dim or dtype mismatch")
    for t in (q, k, v):
        if not t.is_contiguous():
            raise TlAttnError(TL_ERR_INVALID_VALUE, "q/k/v must be contiguous BSHD")
    return B, Hq, Hkv, Sq, Skv, D


def _check_out(t, shape, dtype, device, name):
    """A caller-provided output must match exactly: the kernels' tensor maps and raw
    stores are built from the problem sizes, so a smaller or strided buffer would be
    written out of bounds."""
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != device or \
            not t.is_contiguous():
        raise TlAttnError(TL_ERR_INVALID_VALUE,
                          f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)} "
                          f"on {device} (got {tuple(t.shape)} {t.dtype} on {t.device})")


def _same_device(device, *ts):
    for t in ts:
        if t is not None and t.device != device:
            raise TlAttnError(TL_ERR_INVALID_VALUE, f"all tensors must be on {device}")


def attention(q, k, v, causal=False, scale=None, return_lse=True, out=None, lse_out=None,
              stream=None):
    """o[, lse] = softmax(scale q k^T [+ causal mask]) v on the GPU (allocates outputs)."""
    B, Hq, Hkv, Sq, Skv, D = _dims(q, k, v)
    if not q.is_cuda:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "attention() takes CUDA tensors; use "
                          "attention_host() for host buffers")
    _same_device(q.device, k, v)
    scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
    if out is not None:
        _check_out(out, q.shape, q.dtype, q.device, "out")
    o = out if out is not None else torch.empty_like(q)
    lse = None
    if return_lse:
        if lse_out is not None:
            _check_out(lse_out, (B, Hq, Sq), torch.float32, q.device, "lse_out")
        lse = lse_out if lse_out is not None else torch.empty((B, Hq, Sq), dtype=torch.float32,
                                                              device=q.device)
    tl_attn_fwd(q, k, v, o, lse, B, Hq, Hkv, Sq, Skv, D, int(bool(causal)), scale,
                dtype_code(q.dtype), stream)
    return (o, lse) if return_lse else o


def tl_gemm(a, b, c, M, N, K, dtype, stream=None):
    """Direct mirror of the C entry point: C[M,N] = A[M,K] @ B[K,N]."""
    _check(load_library().tl_gemm(_ptr(a), _ptr(b), _ptr(c), int(M), int(N), int(K), int(dtype),
                                  _stream_handle(stream)))


def gemm(a, b, out=None, stream=None):
    """C = A @ B on the GPU for row-major fp16/bf16 A [M,K], B [K,N] (allocates C)."""
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0] or a.dtype != b.dtype:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "expected A[M,K], B[K,N] of one dtype")
    if not (a.is_contiguous() and b.is_contiguous() and a.is_cuda):
        raise TlAttnError(TL_ERR_INVALID_VALUE, "A and B must be contiguous CUDA tensors")
    M, K = a.shape
    N = b.shape[1]
    c = out if out is not None else torch.empty((M, N), dtype=a.dtype, device=a.device)
    tl_gemm(a, b, c, M, N, K, dtype_code(a.dtype), stream)
    return c


def tl_mla_decode(q, q_pe, kv, k_pe, o, lse, seqlens, B, H, Hkv, Skv, Dl, Dr, scale, dtype,
                  ws, ws_bytes, stream=None):
    """Direct mirror of the C entry point (Fig. 18 MLA decode)."""
    _check(load_library().tl_mla_decode(_ptr(q), _ptr(q_pe), _ptr(kv), _ptr(k_pe), _ptr(o),
                                        _ptr(lse), _ptr(seqlens), int(B), int(H), int(Hkv),
                                        int(Skv), int(Dl), int(Dr), float(scale), int(dtype),
                                        _ptr(ws), int(ws_bytes), _stream_handle(stream)))


def tl_mla_decode_workspace_bytes(B, H, Hkv) -> int:
    return int(load_library().tl_mla_decode_workspace_bytes(int(B), int(H), int(Hkv)))


def mla_decode(q, q_pe, kv, k_pe, seqlens=None, scale=None, return_lse=True, out=None,
               lse_out=None, workspace=None, stream=None):
    """MLA decode on the GPU: q[B,H,Dl], q_pe[B,H,Dr], kv[B,Skv,Hkv,Dl], k_pe[B,Skv,Hkv,Dr],
    optional int32 seqlens[B]. Returns o[B,H,Dl] (and lse[B,H]). ``workspace`` is a uint8
    CUDA tensor of >= tl_mla_decode_workspace_bytes(B, H, Hkv) bytes (allocated if None)."""
    if q.dim() != 3 or q_pe.dim() != 3 or kv.dim() != 4 or k_pe.dim() != 4:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "expected q[B,H,Dl], q_pe[B,H,Dr], "
                          "kv[B,Skv,Hkv,Dl], k_pe[B,Skv,Hkv,Dr]")
    B, H, Dl = q.shape
    _, Skv, Hkv, _ = kv.shape
    Dr = q_pe.shape[2]
    for t in (q, q_pe, kv, k_pe):
        if not (t.is_cuda and t.is_contiguous() and t.dtype == q.dtype):
            raise TlAttnError(TL_ERR_INVALID_VALUE, "inputs must be contiguous CUDA tensors of one dtype")
    _same_device(q.device, q_pe, kv, k_pe, seqlens)
    # every shape the kernel's tensor maps are built from (a shorter k_pe / kv would be read
    # out of bounds: ADVICE r1)
    if tuple(q_pe.shape) != (B, H, Dr) or tuple(kv.shape) != (B, Skv, Hkv, Dl) or \
            tuple(k_pe.shape) != (B, Skv, Hkv, Dr):
        raise TlAttnError(TL_ERR_INVALID_VALUE, "expected q[B,H,Dl], q_pe[B,H,Dr], "
                          "kv[B,Skv,Hkv,Dl], k_pe[B,Skv,Hkv,Dr] with one B, H, Skv, Hkv")
    if seqlens is not None and (seqlens.dtype != torch.int32 or not seqlens.is_cuda or
                                not seqlens.is_contiguous() or seqlens.numel() < B):
        raise TlAttnError(TL_ERR_INVALID_VALUE, "seqlens must be a contiguous CUDA int32 tensor "
                          "with >= B entries")
    scale = 1.0 / math.sqrt(Dl + Dr) if scale is None else float(scale)
    if out is not None:
        _check_out(out, (B, H, Dl), q.dtype, q.device, "out")
    o = out if out is not None else torch.empty((B, H, Dl), dtype=q.dtype, device=q.device)
    lse = None
    if return_lse:
        if lse_out is not None:
            _check_out(lse_out, (B, H), torch.float32, q.device, "lse_out")
        lse = lse_out if lse_out is not None else torch.empty((B, H), dtype=torch.float32,
                                                              device=q.device)
    nbytes = tl_mla_decode_workspace_bytes(B, H, Hkv)
    if workspace is not None and (workspace.dtype != torch.uint8 or
                                  workspace.device != q.device or not workspace.is_contiguous()):
        raise TlAttnError(TL_ERR_INVALID_VALUE, "workspace must be a contiguous uint8 tensor on "
                          f"{q.device}")
    if workspace is None:
        workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=q.device)
    tl_mla_decode(q, q_pe, kv, k_pe, o, lse, seqlens, B, H, Hkv, Skv, Dl, Dr, scale,
                  dtype_code(q.dtype), workspace, workspace.numel(), stream)
    return (o, lse) if return_lse else o


class HostAttention:
    """End-to-end entry on HOST (ideally pinned) tensors via tl_attn_fwd_host.

    Holds the device workspace for one problem shape (allocated by torch).
    """

    def __init__(self, B, Hq, Hkv, Sq, Skv, D, with_lse=True, device=None):
        self.shape = (B, Hq, Hkv, Sq, Skv, D)
        self.with_lse = with_lse
        nbytes = tl_attn_host_workspace_bytes(B, Hq, Hkv, Sq, Skv, D, with_lse)
        if nbytes == 0:
            raise TlAttnError(TL_ERR_INVALID_VALUE, "bad problem size")
        self.ws_bytes = nbytes
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=device or "cuda")

    def __call__(self, q_h, k_h, v_h, o_h, lse_h=None, causal=False, scale=None, stream=None):
        B, Hq, Hkv, Sq, Skv, D = self.shape
        if _dims(q_h, k_h, v_h) != self.shape:
            raise TlAttnError(TL_ERR_INVALID_VALUE, "shape differs from this HostAttention's")
        scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
        tl_attn_fwd_host(q_h, k_h, v_h, o_h, lse_h if self.with_lse else None, B, Hq, Hkv, Sq,
                         Skv, D, int(bool(causal)), scale, dtype_code(q_h.dtype), self.ws,
                         self.ws_bytes, stream)


# --------------------------------------------------------------------------- Mamba-2 SSD
def tl_ssd_chunk_state(x, Bm, dt, dA, states, batch, seqlen, nheads, ngroups, headdim, dstate,
                       chunk_size, dtype, stream=None):
    """Direct mirror of the C entry point (Table 4; include/tlattn.h)."""
    _check(load_library().tl_ssd_chunk_state(
        _ptr(x), _ptr(Bm), _ptr(dt), _ptr(dA), _ptr(states), int(batch), int(seqlen), int(nheads),
        int(ngroups), int(headdim), int(dstate), int(chunk_size), int(dtype), _stream_handle(stream)))


def tl_ssd_chunk_scan(cb, x, dt, dA, C, prev_states, D, out, batch, seqlen, nheads, ngroups,
                      headdim, dstate, chunk_size, dtype, stream=None):
    """Direct mirror of the C entry point (Table 4; include/tlattn.h)."""
    _check(load_library().tl_ssd_chunk_scan(
        _ptr(cb), _ptr(x), _ptr(dt), _ptr(dA), _ptr(C), _ptr(prev_states), _ptr(D), _ptr(out),
        int(batch), int(seqlen), int(nheads), int(ngroups), int(headdim), int(dstate),
        int(chunk_size), int(dtype), _stream_handle(stream)))


def _ssd_dims(x, BC, dt, dA, chunk_size):
    if x.dim() != 4 or BC.dim() != 4 or dt.dim() != 4 or dA.shape != dt.shape:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "expected x[B,L,H,P], B/C[B,L,G,N], "
                          "dt/dA[B,H,nchunks,Q]")
    Bn, L, H, P = x.shape
    G, N = BC.shape[2], BC.shape[3]
    nc = (L + chunk_size - 1) // chunk_size
    if tuple(BC.shape[:2]) != (Bn, L) or tuple(dt.shape) != (Bn, H, nc, chunk_size):
        raise TlAttnError(TL_ERR_INVALID_VALUE, "SSD input shapes disagree")
    if dt.dtype != torch.float32 or dA.dtype != torch.float32 or BC.dtype != x.dtype:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "dt / dA must be fp32, x / B / C one 16-bit dtype")
    for t in (x, BC, dt, dA):
        if not (t.is_cuda and t.is_contiguous() and t.device == x.device):
            raise TlAttnError(TL_ERR_INVALID_VALUE, "SSD inputs must be contiguous CUDA tensors "
                              "on one device")
    return Bn, L, H, G, P, N, nc


def ssd_chunk_state(x, Bm, dt, dA, chunk_size=256, out=None, stream=None):
    """states[B,nchunks,H,P,N] of Mamba-2's chunk_state on the GPU (allocates the output)."""
    Bn, L, H, G, P, N, nc = _ssd_dims(x, Bm, dt, dA, chunk_size)
    shape = (Bn, nc, H, P, N)
    if out is not None:
        _check_out(out, shape, x.dtype, x.device, "out")
    st = out if out is not None else torch.empty(shape, dtype=x.dtype, device=x.device)
    tl_ssd_chunk_state(x, Bm, dt, dA, st, Bn, L, H, G, P, N, chunk_size, dtype_code(x.dtype),
                       stream)
    return st


def ssd_chunk_scan(cb, x, dt, dA, C, prev_states, D=None, chunk_size=256, out=None, stream=None):
    """out[B,L,H,P] of Mamba-2's chunk_scan on the GPU (allocates the output)."""
    Bn, L, H, G, P, N, nc = _ssd_dims(x, C, dt, dA, chunk_size)
    if tuple(cb.shape) != (Bn, nc, G, chunk_size, chunk_size) or cb.dtype != x.dtype:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "cb must be [B,nchunks,G,Q,Q] in x's dtype")
    if tuple(prev_states.shape) != (Bn, nc, H, P, N) or prev_states.dtype != x.dtype:
        raise TlAttnError(TL_ERR_INVALID_VALUE, "prev_states must be [B,nchunks,H,P,N] in x's dtype")
    if D is not None and (tuple(D.shape) != (H,) or D.dtype != torch.float32):
        raise TlAttnError(TL_ERR_INVALID_VALUE, "D must be fp32 [H]")
    for t in (cb, prev_states, D):
        if t is not None and not (t.is_cuda and t.is_contiguous() and t.device == x.device):
            raise TlAttnError(TL_ERR_INVALID_VALUE, "SSD inputs must be contiguous CUDA tensors "
                              "on one device")
    if out is not None:
        _check_out(out, x.shape, x.dtype, x.device, "out")
    o = out if out is not None else torch.empty_like(x)
    tl_ssd_chunk_scan(cb, x, dt, dA, C, prev_states, D, o, Bn, L, H, G, P, N, chunk_size,
                      dtype_code(x.dtype), stream)
    return o
