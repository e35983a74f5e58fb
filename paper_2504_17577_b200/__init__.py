"""B200-native fused attention forward (the hot path of arXiv 2504.17577, TileLang §5.2).

The product is the C-ABI library ``libtlattn.so`` (include/tlattn.h) built from
``csrc/``; this package is its thin Python binding plus test/bench plumbing
(seeded input generator, configs, multi-GPU sharding helpers).
"""
from .tlattn import (  # noqa: F401
    TL_DTYPE_BF16,
    TL_DTYPE_F16,
    TL_ERR_CUDA,
    TL_ERR_INVALID_VALUE,
    TL_ERR_UNSUPPORTED,
    TL_OK,
    HostAttention,
    TlAttnError,
    attention,
    dtype_code,
    gemm,
    mla_decode,
    tl_mla_decode,
    tl_mla_decode_workspace_bytes,
    tl_gemm,
    ssd_chunk_state,
    ssd_chunk_scan,
    tl_ssd_chunk_state,
    tl_ssd_chunk_scan,
    load_library,
    tl_attn_fwd,
    tl_attn_fwd_host,
    tl_attn_host_workspace_bytes,
    tl_attn_last_launch_count,
    tl_attn_strerror,
    tl_attn_version,
    tl_attn_fwd_replicated,
    tl_peer_barrier,
    tl_peer_barrier_set_timeout_ns,
    tl_peer_barrier_check,
    TL_ERR_TIMEOUT,
    tl_ipc_get_handle,
    tl_ipc_open_handle,
    tl_ipc_close_handle,
)
