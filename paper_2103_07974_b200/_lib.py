"""ctypes binding of libcrossover.so (the C-ABI declared in include/crossover.h).

This is the only door to the device path.  There is no fallback: if the
library is missing or fails to load, importing this module raises, and every
operator that needs it fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libcrossover.so"

CS_ERR_ARG = -1
CS_ERR_NCCL_BASE = 10000
CS_NCCL_UNIQUE_ID_BYTES = 128
CS_MAX_SOURCES = 8
CS_ROUND_REFERENCE = 0
CS_ROUND_TORCH = 1

# numpy mirrors of the C descriptor structs (layouts asserted below)
PACK_DESC = np.dtype([("src", "<u8"), ("dst", "<u8"), ("numel", "<i8")])
UPDATE_DESC = np.dtype([("param", "<u8"), ("momentum_buf", "<u8"), ("grad_offset", "<u8"),
                        ("snap_offset", "<u8"), ("numel", "<i8")])
# cs_p2p_desc as a table row (the p2p_gather chunk table)
P2P_DESC = np.dtype([("src", "<u8", (CS_MAX_SOURCES,)), ("dst", "<u8", (CS_MAX_SOURCES,)),
                     ("param", "<u8"), ("momentum_buf", "<u8"), ("numel", "<i8"),
                     ("nranks", "<i4"), ("max_ctas", "<i4")])


class SgdHyper(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("momentum", ctypes.c_float),
                ("dampening_complement", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("nesterov", ctypes.c_int32), ("first_step", ctypes.c_int32),
                ("divisor", ctypes.c_int32), ("rounding", ctypes.c_int32)]


CS_IPC_HANDLE_BYTES = 64


class P2PDesc(ctypes.Structure):
    _fields_ = [("src", ctypes.c_uint64 * CS_MAX_SOURCES), ("dst", ctypes.c_uint64 * CS_MAX_SOURCES),
                ("param", ctypes.c_void_p), ("momentum_buf", ctypes.c_void_p),
                ("numel", ctypes.c_int64), ("nranks", ctypes.c_int32), ("max_ctas", ctypes.c_int32)]


class NvlsDesc(ctypes.Structure):
    _fields_ = [("mc_bucket", ctypes.c_void_p), ("mc_param", ctypes.c_void_p), ("param", ctypes.c_void_p),
                ("momentum_buf", ctypes.c_void_p), ("numel", ctypes.c_int64), ("nranks", ctypes.c_int32),
                ("max_ctas", ctypes.c_int32)]


class CrossoverLibError(RuntimeError):
    """A libcrossover.so call returned a non-zero status."""

    def __init__(self, fn: str, code: int, message: str):
        self.fn = fn
        self.code = code
        super().__init__(f"{fn} failed (code {code}): {message}")


EXPORTS = {
    "cs_abi_version": ([], ctypes.c_int),
    "cs_last_error": ([], ctypes.c_char_p),
    "cs_tune": ([ctypes.c_char_p, ctypes.c_int], ctypes.c_int),
    "cs_stream_create": ([ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cs_stream_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "cs_stream_synchronize": ([ctypes.c_void_p], ctypes.c_int),
    "cs_event_create": ([ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cs_event_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "cs_event_record": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "cs_stream_wait_event": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "cs_event_query": ([ctypes.c_void_p], ctypes.c_int),
    "cs_event_elapsed_ns": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "cs_pack": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "cs_unpack_sgd": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                       ctypes.c_void_p, ctypes.POINTER(SgdHyper), ctypes.c_int, ctypes.c_void_p],
                      ctypes.c_int),
    "cs_spin_ns": ([ctypes.c_uint64, ctypes.c_void_p], ctypes.c_int),
    "cs_gradient_stats_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "cs_gradient_stats": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p], ctypes.c_int),
    "cs_p2p_reduce_sgd_bcast": ([ctypes.POINTER(P2PDesc), ctypes.POINTER(SgdHyper), ctypes.c_void_p],
                                ctypes.c_int),
    "cs_p2p_gather_chunk_elems": ([ctypes.c_int], ctypes.c_int64),
    "cs_p2p_gather_check": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "cs_p2p_gather_reduce_sgd_bcast": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(SgdHyper), ctypes.c_void_p], ctypes.c_int),
    "cs_nvls_reduce_sgd_bcast": ([ctypes.POINTER(NvlsDesc), ctypes.POINTER(SgdHyper), ctypes.c_void_p],
                                 ctypes.c_int),
    "cs_nvls_supported": ([ctypes.c_int], ctypes.c_int),
    "cs_nvls_granularity": ([ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "cs_nvls_create": ([ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint64),
                        ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cs_nvls_import": ([ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
    "cs_nvls_add_device": ([ctypes.c_uint64, ctypes.c_int], ctypes.c_int),
    "cs_nvls_alloc_bind": ([ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t,
                            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_void_p),
                            ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cs_nvls_free": ([ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_size_t], ctypes.c_int),
    "cs_nvls_release": ([ctypes.c_uint64], ctypes.c_int),
    "cs_device_alloc": ([ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cs_device_free": ([ctypes.c_void_p], ctypes.c_int),
    "cs_ipc_get_handle": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "cs_ipc_open_handle": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cs_ipc_close_handle": ([ctypes.c_void_p], ctypes.c_int),
    "cs_ipc_base_of": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)],
                       ctypes.c_int),
    "cs_copy_async": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "cs_stream_memops_supported": ([], ctypes.c_int),
    "cs_host_register": ([ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "cs_host_unregister": ([ctypes.c_void_p], ctypes.c_int),
    "cs_flag_barrier": ([ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p],
                        ctypes.c_int),
    "cs_bn_workspace_bytes": ([ctypes.c_int64, ctypes.c_int], ctypes.c_size_t),
    "cs_bn_forward": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float, ctypes.c_float,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "cs_bn_backward": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "cs_bn_backward2": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "cs_im2col_nhwc": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "cs_maxpool2d_forward": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p], ctypes.c_int),
    "cs_maxpool2d_backward": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_version": ([], ctypes.c_int),
    "cs_nccl_get_unique_id": ([ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_init": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int,
                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "cs_nccl_allreduce_sum_f32": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_reduce_scatter_sum_f32": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_all_gather_f32": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_async_error": ([ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_abort": ([ctypes.c_void_p], ctypes.c_int),
    "cs_nccl_destroy": ([ctypes.c_void_p], ctypes.c_int),
}


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2103_07974_b200._build` "
            "(there is no CPU fallback for the crossover step)")
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (argtypes, restype) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    return lib


lib = _load()
assert lib.cs_abi_version() == 3, "libcrossover.so ABI version mismatch"


def check(fn: str, rc: int) -> None:
    if rc != 0:
        msg = lib.cs_last_error()
        raise CrossoverLibError(fn, rc, msg.decode() if msg else "")


def pack(descs: np.ndarray, stream: int, max_ctas: int = 0) -> None:
    """K1 over a PACK_DESC array (host memory); max_ctas > 0 = persistent grid cap."""
    assert descs.dtype == PACK_DESC and descs.flags.c_contiguous
    check("cs_pack", lib.cs_pack(descs.ctypes.data, len(descs), max_ctas, stream))


def unpack_sgd(descs: np.ndarray, sources: np.ndarray, snapshot: int, hyper: SgdHyper,
               stream: int, max_ctas: int = 0) -> None:
    """K2 over an UPDATE_DESC array with `sources` (uint64 device addresses)."""
    assert descs.dtype == UPDATE_DESC and descs.flags.c_contiguous
    assert sources.dtype == np.uint64 and 1 <= len(sources) <= CS_MAX_SOURCES
    check("cs_unpack_sgd", lib.cs_unpack_sgd(descs.ctypes.data, len(descs), sources.ctypes.data,
                                             len(sources), snapshot or None,
                                             ctypes.byref(hyper), max_ctas, stream))


def gradient_stats_workspace_bytes(numel: int) -> int:
    return int(lib.cs_gradient_stats_workspace_bytes(numel))


def gradient_stats(data: int, numel: int, out: int, workspace: int, stream: int) -> None:
    check("cs_gradient_stats", lib.cs_gradient_stats(data, numel, out, workspace, stream))


def tune(key: str, value: int) -> None:
    """Launch-shape knob (see include/crossover.h cs_tune)."""
    check("cs_tune", lib.cs_tune(key.encode(), value))


def spin_ns(ns: int, stream: int) -> None:
    """Enqueue a compute phase of `ns` nanoseconds of device time (cs_spin_ns)."""
    check("cs_spin_ns", lib.cs_spin_ns(int(ns), stream))
