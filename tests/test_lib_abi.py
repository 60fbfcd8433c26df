"""libcrossover.so loads on a CPU-only host and exports exactly what include/crossover.h declares."""

import ctypes
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "crossover.h").read_text()
    return sorted(set(re.findall(r"CS_API\s+[\w\s\*]+?\b(cs_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("cs_pack", "cs_unpack_sgd", "cs_nccl_init", "cs_nccl_allreduce_sum_f32",
                 "cs_nccl_destroy", "cs_last_error", "cs_gradient_stats"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2103_07974_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cs_\w+)", out))
    assert set(_declared()) <= exported
    for name in _declared():
        assert hasattr(_lib.lib, name)
        assert name in _lib.EXPORTS, f"{name} not bound in _lib.EXPORTS"


def test_library_is_sm100a():
    from paper_2103_07974_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    from paper_2103_07974_b200 import _lib

    assert _lib.PACK_DESC.itemsize == 24
    assert ctypes.sizeof(_lib.P2PDesc) == 8 * 8 * 2 + 8 + 8 + 8 + 8
    assert _lib.UPDATE_DESC.itemsize == 40
    assert ctypes.sizeof(_lib.SgdHyper) == 32
    assert _lib.P2P_DESC.itemsize == ctypes.sizeof(_lib.P2PDesc)
    assert _lib.lib.cs_abi_version() == 3


def test_gather_table_validation_without_gpu():
    """cs_p2p_gather_check validates the p2p_gather chunk table on the host."""
    from paper_2103_07974_b200 import _lib

    assert [_lib.lib.cs_p2p_gather_chunk_elems(w) for w in (2, 4, 8)] == [4096, 2048, 1024]
    assert _lib.lib.cs_p2p_gather_chunk_elems(9) == 0
    t = np.zeros(3, dtype=_lib.P2P_DESC)
    for i in range(3):
        t[i]["src"][:2] = [0x100000 + 0x10000 * i, 0x200000 + 0x10000 * i]
        t[i]["dst"][:2] = [0x300000 + 0x10000 * i, 0x400000 + 0x10000 * i]
        t[i]["param"] = 0x300000 + 0x10000 * i
        t[i]["numel"] = 4096 if i < 2 else 17
        t[i]["nranks"] = 2

    def check(tab, momentum=0):
        return _lib.lib.cs_p2p_gather_check(tab.ctypes.data, len(tab), 2, momentum)

    assert check(t) == 0
    assert check(t, momentum=1) == _lib.CS_ERR_ARG                        # no momentum buffer
    bad = t.copy()
    bad[1]["src"][1] += 4
    assert check(bad) == _lib.CS_ERR_ARG and b"aligned" in _lib.lib.cs_last_error()
    big = t.copy()
    big[0]["numel"] = 4097                                                # longer than one chunk
    assert check(big) == _lib.CS_ERR_ARG and b"chunk 0" in _lib.lib.cs_last_error()
    w = t.copy()
    w[2]["nranks"] = 4
    assert check(w) == _lib.CS_ERR_ARG


def test_argument_errors_without_gpu():
    """Invalid calls fail in host validation with a message; nothing reaches CUDA."""
    from paper_2103_07974_b200 import _lib

    assert _lib.lib.cs_pack(None, -1, 0, None) == _lib.CS_ERR_ARG
    assert b"invalid descriptor" in _lib.lib.cs_last_error()
    d = np.zeros(1, dtype=_lib.PACK_DESC)
    d["numel"] = 5
    with pytest.raises(_lib.CrossoverLibError, match="null pointer"):
        _lib.pack(d, 0)
    u = np.zeros(1, dtype=_lib.UPDATE_DESC)
    h = _lib.SgdHyper(lr=0.1, divisor=0, rounding=0)
    with pytest.raises(_lib.CrossoverLibError, match="divisor"):
        _lib.unpack_sgd(u, np.zeros(1, dtype=np.uint64), 0, h, 0)
    h = _lib.SgdHyper(lr=0.1, momentum=0.9, divisor=1, rounding=_lib.CS_ROUND_REFERENCE)
    with pytest.raises(_lib.CrossoverLibError, match="reference rounding"):
        _lib.unpack_sgd(u, np.zeros(1, dtype=np.uint64), 0, h, 0)
    assert _lib.lib.cs_unpack_sgd(u.ctypes.data, 1, np.zeros(9, dtype=np.uint64).ctypes.data, 9,
                                  None, ctypes.byref(_lib.SgdHyper(lr=0.1, divisor=1)), 0, None) == _lib.CS_ERR_ARG
    assert _lib.lib.cs_nccl_init(None, 0, 0, None, 0, 0) == _lib.CS_ERR_ARG
    # BN: channel counts the kernels do not support are rejected before any launch
    assert _lib.lib.cs_bn_workspace_bytes(100, 7) == 0
    assert _lib.lib.cs_bn_forward(16, None, 100, 7, None, None, None, None, 0.1, 1e-5, 16, 16, 16, 16,
                                  16, 0, None) == _lib.CS_ERR_ARG
    assert b"cs_bn_forward" in _lib.lib.cs_last_error()
    # copy-engine transport and the SM-free flag barrier validate before touching CUDA
    assert _lib.lib.cs_copy_async(None, None, 0, None) == 0
    assert _lib.lib.cs_copy_async(None, None, 16, None) == _lib.CS_ERR_ARG
    assert _lib.lib.cs_flag_barrier(None, 0, 0, 2, None) == _lib.CS_ERR_ARG
    peers = np.zeros(2, dtype=np.uint64)
    assert _lib.lib.cs_flag_barrier(peers.ctypes.data, 64, 2, 2, None) == _lib.CS_ERR_ARG   # rank out of range
    assert _lib.lib.cs_stream_memops_supported() in (0, 1)
    p2p = _lib.P2PDesc()
    p2p.nranks = 9
    assert _lib.lib.cs_p2p_reduce_sgd_bcast(ctypes.byref(p2p), ctypes.byref(_lib.SgdHyper(lr=0.1, divisor=9)),
                                            None) == _lib.CS_ERR_ARG
    p2p.nranks, p2p.max_ctas = 2, -1
    assert _lib.lib.cs_p2p_reduce_sgd_bcast(ctypes.byref(p2p), ctypes.byref(_lib.SgdHyper(lr=0.1, divisor=2)),
                                            None) == _lib.CS_ERR_ARG


def test_nccl_version_is_torchs():
    import torch

    from paper_2103_07974_b200 import _lib

    v = _lib.lib.cs_nccl_version()
    major, minor, patch = torch.cuda.nccl.version()
    assert v == major * 10000 + minor * 100 + patch


def test_product_has_no_oracle_dependency():
    """The product package never imports the CPU oracle (no fallback path)."""
    for path in (ROOT / "paper_2103_07974_b200").rglob("*.py"):
        src = path.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), path
