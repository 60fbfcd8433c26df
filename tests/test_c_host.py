"""A torch-free C host drives the crossover step through the C-ABI alone (include/crossover.h)."""

import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = ROOT / "tests" / "c" / "abi_pipeline.c"
LIBDIR = ROOT / "paper_2103_07974_b200"


def _compile(out):
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-I", str(ROOT / "include"), "-I/usr/local/cuda/include",
           str(SRC), "-L", str(LIBDIR), "-l:libcrossover.so", f"-Wl,-rpath,{LIBDIR}",
           "-L/usr/local/cuda/lib64", "-lcudart", "-o", str(out)]
    return subprocess.run(cmd, capture_output=True, text=True)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc missing")
def test_c_host_compiles_against_the_header(tmp_path):
    r = _compile(tmp_path / "abi_pipeline")
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_c_host_pipeline_runs_bit_exact(tmp_path, cuda_device):
    exe = tmp_path / "abi_pipeline"
    r = _compile(exe)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "bit-exact" in run.stdout
