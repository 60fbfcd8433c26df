"""The W > 1 data plane (p2p / ce transports, flag barriers, failure path) with W processes on ONE GPU.

NCCL refuses two ranks on one device, but the peer-memory transports do not use NCCL: CUDA IPC
mappings and stream memory operations work between processes on the same device, so W ranks on a
single B200 run the same code path as W GPUs over NVLink (tests/mp_peer_check.py).  The NCCL
transports (bucket / sharded / unfused) keep their >= 2-GPU test in test_gpu_multirank.py.
"""

import json
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _launch(tmp_path, world: int, case: str, port: int, timeout: int = 900):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / f"{case}_{world}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           str(ROOT / "tests" / "mp_peer_check.py"), str(out), case]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("PEERCHECK ")]
    assert proc.returncode == 0, (lines or [proc.stdout[-3000:]])[-1] + proc.stderr[-4000:]
    res = json.loads(out.read_text())
    bad = [c for c in res["checks"] if not c["ok"]]
    assert res["ok"] and not bad, bad or res
    return res


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_transports_parity_one_gpu(tmp_path, world):
    """p2p / ce / adaptive at W ranks: reference golden within 1e-5 + 1e-4|w|, bitwise == W
    simulated workers (rank-order sum), bitwise across transports, ranks identical."""
    res = _launch(tmp_path, world, "parity", 29710 + world)
    assert res["golden_worst_ratio"] <= 1.0
    names = {c["name"] for c in res["checks"]}
    assert f"mlp_momentum_p2p_bitwise_eq_simulated_w{world}" in names


def test_flag_barrier_failure_releases_device(tmp_path):
    """A rank that stops issuing work: the watchdog raises DeadlockError(job, iteration) and the
    host-written final epoch releases every pending flag wait, so the device drains."""
    _launch(tmp_path, 2, "fail", 29730, timeout=300)


def test_resnet50_update_parity_ce_two_ranks(tmp_path):
    """Config-2 update path (161 tensors, graphed, channels_last, IPC flat params) over the
    copy-engine transport at W = 2: bitwise torch.optim.SGD(foreach=False) on the rank-order
    average of both ranks' gradients, 3 iterations x 2 apps."""
    _launch(tmp_path, 2, "resnet", 29740)


@pytest.mark.parametrize("world", [2, 4])
def test_rotation_graph_over_peer_transports(tmp_path, world):
    """graphs.RotationGraph with ce / p2p: barriers, CE pulls and the P2P kernel captured into one
    graph per rotation -- bitwise equal to eager, ranks identical."""
    _launch(tmp_path, world, "graph", 29750 + world)


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_gather_resnet50_update_parity(tmp_path, world):
    """The K1-free p2p_gather transport: one kernel per sync reads every rank's CUDA-graph static
    gradient tensors in place (161 ResNet-50 tensors cut at the W shard boundaries); bitwise
    torch.optim.SGD(foreach=False) on the rank-order average, 3 iterations x 2 apps."""
    _launch(tmp_path, world, "gather", 29760 + world)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p2p_gather_graphed_mlp(tmp_path, world):
    """p2p_gather at W = 2 / 4 / 8 (every chunk-table width of the kernel) on two CUDA-graphed MLP
    apps: per-iteration weights bitwise equal to the p2p transport (graphed and eager), ranks
    identical, one kernel launch per sync."""
    _launch(tmp_path, world, "gather_mlp", 29770 + world)
