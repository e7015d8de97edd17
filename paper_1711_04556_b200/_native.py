"""Loader for the sm_100a library `_lib/libb200tabu.so` (C ABI in
include/rcpsp_tabu_b200.h).

There is no fallback: importing the package works without the library (so
host-only helpers stay usable), but every device entry point calls `lib()`,
which raises `NativeLibraryError` when the shared object is missing or no
CUDA device is visible.  Build it with `python -c "import __graft_entry__ as
g; g.build()"` (or `make -C paper_1711_04556_b200`).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / "libb200tabu.so"
# A/B measurements of kernel variants (tools/ab_bench.sh) point this at another build
if os.environ.get("RCPSP_B200_LIB"):
    LIB_PATH = Path(os.environ["RCPSP_B200_LIB"])
ABI_VERSION = 8

_lib = None

_vp = ctypes.c_void_p
_i = ctypes.c_int


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, stale, or cannot run here."""


class RcpspSolveArgs(ctypes.Structure):
    """ctypes mirror of `RcpspSolveArgs` (every field is 64-bit)."""

    _fields_ = [
        ("blob", _vp), ("blob_off", _vp), ("n_inst", ctypes.c_int64), ("n_max", ctypes.c_int64),
        ("workers", ctypes.c_int64), ("pool_size", ctypes.c_int64),
        ("tabu_size", ctypes.c_int64), ("delta", ctypes.c_int64), ("phi_steps", ctypes.c_int64),
        ("phi_max", ctypes.c_int64), ("total_iters", ctypes.c_int64),
        ("block_iters", ctypes.c_int64), ("epoch_limit", ctypes.c_int64),
        ("grant_cap", ctypes.c_int64), ("collect_trace", ctypes.c_int64),
        ("ws_lock", _vp), ("ws_hdr", _vp), ("ent_order", _vp), ("ent_cmax", _vp),
        ("ent_tabu", _vp), ("ent_head", _vp), ("ent_ic", _vp), ("ent_reads", _vp),
        ("ws_best_order", _vp),
        ("w_rng", _vp), ("w_stats", _vp), ("w_trace", _vp), ("trace_cap", ctypes.c_int64),
        ("w_chunks", _vp), ("chunk_cap", ctypes.c_int64),
        ("moves_buf", _vp), ("cmax_buf", _vp), ("nbhd_max", ctypes.c_int64), ("err", _vp),
        ("h_max", ctypes.c_int64), ("e_max", ctypes.c_int64), ("m_max", ctypes.c_int64),
        ("rmax_max", ctypes.c_int64), ("words", ctypes.c_int64), ("group", ctypes.c_int64),
        ("threads", ctypes.c_int64), ("steal", ctypes.c_int64), ("full_sgs", ctypes.c_int64),
        ("cluster", ctypes.c_int64), ("time_budget_ns", ctypes.c_int64), ("t0_ns", _vp),
        ("no_big", ctypes.c_int64),
        ("sumcap_max", ctypes.c_int64), ("prof_slots", ctypes.c_int64), ("ent_lock", _vp), ("outbox", _vp), ("peers", _vp), ("n_peers", ctypes.c_int64), ("peer_seen", _vp),
        ("poll_every", ctypes.c_int64), ("peer_stats", _vp),
    ]


class RcpspShape(ctypes.Structure):
    """ctypes mirror of `RcpspShape` (the packed blob's header fields)."""

    _fields_ = [(name, ctypes.c_int32) for name in
                ("n", "m", "horizon", "edges", "words", "lane_bits", "rmax", "cpm", "len", "big",
                 "sumcap")]


_SHP = ctypes.POINTER(RcpspShape)

_SIGNATURES = {
    "rcpsp_abi_version": ([], _i),
    "rcpsp_last_error": ([], ctypes.c_char_p),
    "rcpsp_pack_last_error": ([], ctypes.c_char_p),
    "rcpsp_blob_words": ([_vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, ctypes.c_int32],
                         ctypes.c_int64),
    "rcpsp_pack_instance": ([_vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, ctypes.c_int32, _vp,
                             ctypes.c_int64], _i),
    "rcpsp_blob_shape": ([_vp, _SHP], _i),
    "rcpsp_device_info": ([_vp, _vp, _vp, _vp], _i),
    "rcpsp_eval_batch": ([_vp, _SHP, _i, _vp, _i, _i, _vp, _vp, _i, _vp, _vp], _i),
    "rcpsp_filter_batch": ([_vp, _SHP, _vp, _i, _i, _vp, _i, _vp, _vp, _vp], _i),
    "rcpsp_run_chunk_batch": ([_vp, _SHP, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i,
                               _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _i, _vp, _vp], _i),
    "rcpsp_pool_init": ([ctypes.POINTER(RcpspSolveArgs), _vp, _i, _i, _vp, _vp], _i),
    "rcpsp_solve": ([ctypes.POINTER(RcpspSolveArgs), _vp, _i, _i, _vp], _i),
    "rcpsp_merge_elites": ([ctypes.POINTER(RcpspSolveArgs), _vp, _vp, _i, _vp], _i),
    "rcpsp_export_elites": ([ctypes.POINTER(RcpspSolveArgs), _vp, _vp, _vp], _i),
    "rcpsp_outbox_alloc": ([ctypes.c_int64, ctypes.POINTER(_vp), _vp], _i),
    "rcpsp_outbox_open": ([_vp, ctypes.POINTER(_vp)], _i),
    "rcpsp_outbox_close": ([_vp], _i),
    "rcpsp_outbox_free": ([_vp], _i),
    "rcpsp_outbox_reset": ([_vp, ctypes.c_int64, _vp], _i),
    "rcpsp_diversify_batch": ([_vp, _SHP, _vp, _i, _i, _vp, _vp, _vp], _i),
    "rcpsp_rng_probe": ([_vp, _vp, _i, _vp, _vp], _i),
    "rcpsp_eq8_probe": ([_vp, _i, _vp, _vp], _i),
    "rcpsp_smem_probe": ([_i, _i, _i, _vp, _vp], _i),
    "rcpsp_state_op": ([_vp, _SHP, _i, _vp, _i, _i, _vp, _vp, _vp], _i),
}

EXPORTED = tuple(_SIGNATURES)


def load_library(path: Path = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and declare every exported signature (no CUDA calls)."""
    if not path.exists():
        raise NativeLibraryError(
            f"{path} is missing: build the sm_100a library first (__graft_entry__.build())")
    L = ctypes.CDLL(str(path))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.rcpsp_abi_version() != ABI_VERSION:
        raise NativeLibraryError(f"{path}: ABI {L.rcpsp_abi_version()} != {ABI_VERSION}")
    return L


_host_lib = None


def host_lib() -> ctypes.CDLL:
    """The library for its host-only entry points (instance packing): needs
    the built .so but no GPU -- no kernel is launched through this handle."""
    global _host_lib
    if _host_lib is None:
        _host_lib = _lib if _lib is not None else load_library()
    return _host_lib


def lib() -> ctypes.CDLL:
    """The loaded library; raises unless a CUDA device can run it."""
    global _lib
    if _lib is None:
        import torch
        if not torch.cuda.is_available():
            raise NativeLibraryError("no CUDA device visible: the B200 kernels cannot run here "
                                     "(there is no CPU fallback)")
        torch.cuda.init()
        _lib = load_library()
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().rcpsp_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed: {msg}")


def ptr(t) -> int | None:
    """data_ptr of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
