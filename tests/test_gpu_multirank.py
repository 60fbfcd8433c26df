"""NCCL path over NVLink: one process per GPU (needs >= 2 GPUs; `gpurun --gpus 2`)."""

import json
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multirank_crossover_parity(tmp_path, world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + world}",
           str(ROOT / "tests" / "mp_crossover_check.py"), str(out)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    checks = [ln for ln in proc.stdout.splitlines() if ln.startswith("MPCHECK ")]
    assert proc.returncode == 0, (checks or [proc.stdout[-3000:]])[-1] + proc.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res


@pytest.mark.parametrize("world", [2, 4])
def test_nvls_transport(tmp_path, world):
    """The NVSwitch-multicast transport (multimem.ld_reduce / multimem.st) on `world` GPUs: linear
    momentum vs the fp64 oracle, MLP close to the rank-order p2p transport, ranks identical."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    out = tmp_path / "nvls.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29640 + world}",
           str(ROOT / "tests" / "mp_nvls_check.py"), str(out)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    assert json.loads(out.read_text())["ok"]
