"""Builds libcrossover.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Run as ``python -m paper_2103_07974_b200._build`` or via ``__graft_entry__.build()``.
The library links the NCCL that torch itself loads (site-packages/nvidia/nccl),
so one copy of libnccl.so.2 is mapped per process.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libcrossover.so"
SOURCES = ["crossover_im2col.cu", "crossover_kernels.cu", "crossover_p2p.cu", "crossover_nvls.cu", "crossover_bn.cu",
           "crossover_pool.cu", "crossover_abi.cu", "crossover_nccl.cu"]
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_home() -> Path:
    import nvidia  # namespace package shipped with the torch wheels

    for root in nvidia.__path__:
        cand = Path(root) / "nccl"
        if (cand / "include" / "nccl.h").exists():
            return cand
    raise FileNotFoundError("nccl.h not found under site-packages/nvidia/nccl")


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(path).exists():
        raise FileNotFoundError("nvcc not found")
    return path


def needs_rebuild() -> bool:
    if not LIB_PATH.exists():
        return True
    mtime = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [REPO_DIR / "include" / "crossover.h"]
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_rebuild():
        return LIB_PATH
    nccl = nccl_home()
    cmd = [
        nvcc(), *ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17", "--shared",
        "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
        f"-I{REPO_DIR / 'include'}", f"-I{CSRC}", f"-I{nccl / 'include'}",
        *[str(CSRC / s) for s in SOURCES],
        f"-L{nccl / 'lib'}", "-l:libnccl.so.2", f"-Xlinker=-rpath,{nccl / 'lib'}",
        "-o", str(LIB_PATH) + ".tmp",
    ]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (PKG_DIR / "build.log").write_text(" ".join(cmd) + "\n" + log)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{log[-6000:]}")
    os.replace(str(LIB_PATH) + ".tmp", LIB_PATH)
    if verbose:
        print(log)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB_PATH)
