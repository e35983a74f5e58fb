"""C-ABI checks that need no GPU: the library builds/loads, exports every symbol
include/tlattn.h declares, and rejects bad arguments synchronously BEFORE any CUDA
call (include/tlattn.h "Errors")."""
import ctypes
import os
import re

import pytest
import torch

from paper_2504_17577_b200 import build as pkg_build
from paper_2504_17577_b200 import tlattn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tlattn.h")


@pytest.fixture(scope="module")
def lib():
    pkg_build.build()
    return tlattn.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tl_\w+)\s*\(", src)))


def test_header_declares_the_entry_points():
    names = declared_functions()
    for n in ("tl_attn_fwd", "tl_attn_fwd_host", "tl_attn_host_workspace_bytes",
              "tl_attn_strerror", "tl_attn_version", "tl_attn_last_launch_count", "tl_gemm",
              "tl_mla_decode", "tl_mla_decode_workspace_bytes"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(pkg_build.LIB)
    for name in declared_functions():
        assert hasattr(raw, name), f"libtlattn.so does not export {name}"


def test_version_and_strerror(lib):
    assert tlattn.tl_attn_version() == 0x000300
    for code in (0, 1, 2, 3, 4):
        assert tlattn.tl_attn_strerror(code).startswith(("TL_OK", "TL_ERR"))
    assert "unknown" in tlattn.tl_attn_strerror(99)


FAKE = 1 << 20  # a 16-byte-aligned non-null "device pointer" (never dereferenced)

GOOD = dict(q=FAKE, k=FAKE, v=FAKE, o=FAKE, lse=FAKE, B=1, Hq=2, Hkv=1, Sq=128, Skv=128, D=128,
            causal=0, scale=0.125, dtype=1)


def call(lib, **over):
    a = dict(GOOD, **over)
    return lib.tl_attn_fwd(a["q"], a["k"], a["v"], a["o"], a["lse"], a["B"], a["Hq"], a["Hkv"],
                           a["Sq"], a["Skv"], a["D"], a["causal"], a["scale"], a["dtype"], None)


@pytest.mark.parametrize("over,code", [
    (dict(q=None), 1), (dict(k=None), 1), (dict(v=None), 1), (dict(o=None), 1),
    (dict(B=0), 1), (dict(Hq=0), 1), (dict(Hkv=-1), 1), (dict(Sq=0), 1), (dict(Skv=0), 1),
    (dict(D=0), 1), (dict(causal=2), 1), (dict(scale=float("nan")), 1),
    (dict(scale=float("inf")), 1), (dict(dtype=5), 1),
    (dict(D=96), 2), (dict(D=256), 2), (dict(Hq=3, Hkv=2), 2), (dict(q=FAKE + 8), 2),
    (dict(o=FAKE + 2), 2), (dict(lse=FAKE + 2), 2),
    (dict(B=1 << 20, Hq=1 << 10, Hkv=1 << 10, Sq=1 << 12), 2),
])
def test_invalid_arguments_rejected(lib, over, code):
    assert call(lib, **over) == code


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_valid_arguments_without_device_is_cuda_error(lib):
    # Validation passes; the first CUDA call finds no device -> TL_ERR_CUDA, no fallback.
    assert call(lib) == 3
    assert call(lib, lse=None) == 3


def test_host_workspace_size(lib):
    n = tlattn.tl_attn_host_workspace_bytes(64, 32, 32, 2048, 2048, 128, True)
    per_b = 2048 * 32 * 128 * 2
    assert n >= 2 * (4 * per_b) * 8 and n % 256 == 0
    assert tlattn.tl_attn_host_workspace_bytes(0, 1, 1, 1, 1, 64, True) == 0


def test_host_entry_rejects_small_workspace(lib):
    rc = lib.tl_attn_fwd_host(FAKE, FAKE, FAKE, FAKE, None, 1, 1, 1, 128, 128, 64, 0, 0.1, 0,
                              FAKE, 16, None)
    assert rc == 1
    rc = lib.tl_attn_fwd_host(FAKE, FAKE, FAKE, FAKE, None, 1, 1, 1, 128, 128, 64, 0, 0.1, 0,
                              None, 1 << 30, None)
    assert rc == 1


def test_python_binding_fails_loudly_without_library(tmp_path):
    with pytest.raises(RuntimeError):
        saved = tlattn._lib
        tlattn._lib = None
        try:
            tlattn.load_library(str(tmp_path / "missing.so"))
        finally:
            tlattn._lib = saved


# ---------------------------------------------------------------- tl_mla_decode
MLA_GOOD = dict(q=FAKE, q_pe=FAKE, kv=FAKE, k_pe=FAKE, o=FAKE, lse=FAKE, seqlens=None, B=2, H=128,
                Hkv=1, Skv=1024, Dl=512, Dr=64, scale=0.04, dtype=1, ws=FAKE, ws_bytes=1 << 40)


def mla_call(lib, **over):
    a = dict(MLA_GOOD, **over)
    return lib.tl_mla_decode(a["q"], a["q_pe"], a["kv"], a["k_pe"], a["o"], a["lse"], a["seqlens"],
                             a["B"], a["H"], a["Hkv"], a["Skv"], a["Dl"], a["Dr"], a["scale"],
                             a["dtype"], a["ws"], a["ws_bytes"], None)


@pytest.mark.parametrize("over,code", [
    (dict(q=None), 1), (dict(q_pe=None), 1), (dict(kv=None), 1), (dict(k_pe=None), 1),
    (dict(o=None), 1), (dict(ws=None), 1), (dict(B=0), 1), (dict(H=0), 1), (dict(Hkv=0), 1),
    (dict(Skv=0), 1), (dict(Dr=0), 1), (dict(scale=float("nan")), 1), (dict(dtype=2), 1),
    (dict(Dl=256), 2), (dict(Dr=32), 2), (dict(H=6, Hkv=4), 2), (dict(kv=FAKE + 8), 2),
    (dict(lse=FAKE + 1), 2), (dict(seqlens=FAKE + 2), 2), (dict(ws=FAKE + 16), 2),
    (dict(B=1 << 16, Skv=1 << 16), 2),
])
def test_mla_invalid_arguments_rejected(lib, over, code):
    assert mla_call(lib, **over) == code


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_mla_without_device(lib):
    assert mla_call(lib) == 3  # arguments valid, no device -> TL_ERR_CUDA (no fallback)
    assert tlattn.tl_mla_decode_workspace_bytes(2, 128, 1) == 0  # needs the device's SM count
    assert tlattn.tl_mla_decode_workspace_bytes(0, 128, 1) == 0


# ------------------------------------------- replicated output / peer memory
def _ptrs(*xs):
    arr = (ctypes.c_void_p * len(xs))(*xs)
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))


REP_GOOD = dict(q=FAKE, k=FAKE, v=FAKE, outs=[FAKE, FAKE], lses=None, B_total=2, b_off=0,
                Hq_total=4, h_off=2, B=2, Hq=2, Hkv=1, Sq=128, Skv=128, D=128, causal=1,
                scale=0.1, dtype=1)


def rep_call(lib, **over):
    a = dict(REP_GOOD, **over)
    outs = _ptrs(*a["outs"]) if a["outs"] is not None else None
    lses = _ptrs(*a["lses"]) if a["lses"] is not None else None
    n = a.get("n", len(a["outs"]) if a["outs"] is not None else 1)
    return lib.tl_attn_fwd_replicated(a["q"], a["k"], a["v"], outs, lses, n, a["B_total"],
                                      a["b_off"], a["Hq_total"], a["h_off"], a["B"], a["Hq"],
                                      a["Hkv"], a["Sq"], a["Skv"], a["D"], a["causal"], a["scale"],
                                      a["dtype"], None)


@pytest.mark.parametrize("over,code", [
    (dict(outs=None), 1), (dict(n=0), 1), (dict(outs=[FAKE] * 9), 1), (dict(outs=[FAKE, 0]), 1),
    (dict(h_off=3), 1), (dict(b_off=1), 1), (dict(h_off=-1), 1), (dict(Hq_total=0), 1),
    (dict(q=None), 1), (dict(D=96), 2), (dict(outs=[FAKE, FAKE + 8]), 2),
    (dict(lses=[FAKE, FAKE + 2]), 2),
])
def test_replicated_invalid_arguments_rejected(lib, over, code):
    assert rep_call(lib, **over) == code


def test_peer_barrier_and_ipc_invalid_arguments_rejected(lib):
    assert lib.tl_peer_barrier(None, 2, 0, 1, None) == 1
    assert lib.tl_peer_barrier(_ptrs(FAKE, FAKE), 0, 0, 1, None) == 1
    assert lib.tl_peer_barrier(_ptrs(*([FAKE] * 9)), 9, 0, 1, None) == 1
    assert lib.tl_peer_barrier(_ptrs(FAKE, FAKE), 2, 2, 1, None) == 1
    assert lib.tl_peer_barrier(_ptrs(FAKE, FAKE + 2), 2, 0, 1, None) == 1
    assert lib.tl_peer_barrier_set_timeout_ns(0) == 1
    assert lib.tl_peer_barrier_check(None) == 1
    assert lib.tl_peer_barrier_check(FAKE + 2) == 1
    assert lib.tl_ipc_handle_bytes() >= 64
    buf = ctypes.create_string_buffer(lib.tl_ipc_handle_bytes())
    assert lib.tl_ipc_get_handle(None, buf) == 1
    assert lib.tl_ipc_open_handle(None, None) == 1
    assert lib.tl_ipc_close_handle(None) == 1


def test_options_set_get_without_a_device(lib):
    """Experiment options are process-wide values behind tl_attn_set_option (no getenv on
    production calls); unknown options are refused, -1 restores automatic."""
    from paper_2504_17577_b200.tlattn import TL_OPT_LPT, TL_OPT_UNIT_TILES, option
    assert lib.tl_attn_set_option(99, 1) == 1 and lib.tl_attn_get_option(99) == -2
    assert lib.tl_attn_set_option(-1, 1) == 1
    old = lib.tl_attn_get_option(TL_OPT_LPT)
    with option(TL_OPT_LPT, 1):
        assert lib.tl_attn_get_option(TL_OPT_LPT) == 1
        with option(TL_OPT_UNIT_TILES, 2):
            assert lib.tl_attn_get_option(TL_OPT_UNIT_TILES) == 2
    assert lib.tl_attn_get_option(TL_OPT_LPT) == old
    assert lib.tl_attn_set_option(TL_OPT_LPT, -7) == 0 and lib.tl_attn_get_option(TL_OPT_LPT) == -1
    lib.tl_attn_set_option(TL_OPT_LPT, old)


def test_ssd_argument_errors_before_any_cuda_call(lib):
    """tl_ssd_chunk_state / _scan validate their arguments before touching the device."""
    F = FAKE
    st = lambda **o: lib.tl_ssd_chunk_state(  # noqa: E731
        o.get("x", F), o.get("b", F), o.get("dt", F), o.get("dA", F), o.get("out", F),
        o.get("B", 1), o.get("L", 256), o.get("H", 2), o.get("G", 1), o.get("P", 64),
        o.get("N", 128), o.get("Q", 256), o.get("dtype", 1), None)
    sc = lambda **o: lib.tl_ssd_chunk_scan(  # noqa: E731
        o.get("cb", F), o.get("x", F), o.get("dt", F), o.get("dA", F), o.get("c", F),
        o.get("prev", F), o.get("D", None), o.get("out", F), o.get("B", 1), o.get("L", 256),
        o.get("H", 2), o.get("G", 1), o.get("P", 64), o.get("N", 128), o.get("Q", 256),
        o.get("dtype", 1), None)
    for call in (st, sc):
        assert call(x=None) == 1
        assert call(B=0) == 1
        assert call(H=3, G=2) == 1          # nheads % ngroups
        assert call(dtype=7) == 1
        assert call(P=32) == 2              # head_dim 64 only
        assert call(N=64) == 2              # d_state 128 only
        assert call(Q=128) == 2             # chunk length 256 only
        assert call(x=F + 8) == 2           # 16-byte alignment
    assert st(H=3, G=1) == 2                # chunk_state: head pairs
    assert st(H=4, G=4) == 2                # both heads of a pair in one group
    assert sc(dt=F + 2) == 2                # fp32 vectors: 4-byte alignment
