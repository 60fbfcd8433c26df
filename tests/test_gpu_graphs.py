"""Whole-rotation CUDA graphs (graphs.RotationGraph): same arithmetic, same schedule, one launch.

The graph replays the crossover (or sequential) rotation with the same kernels in the same order
as eager ``step()``; only K1's stream moves (compute stream, right after the backward).  So the
weights after T iterations must equal the eager run's bit for bit, and stay within the stated fp32
tolerance of the reference's own fp64 trajectories (equivalence.py:150-232, golden vectors).
"""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _flat(app):
    return torch.cat([p.detach().reshape(-1) for p in app.params]).cpu()


def _run(make_apps, policy, T, graph, warm=2, per=1):
    from paper_2103_07974_b200.graphs import RotationGraph
    from paper_2103_07974_b200.scheduler import CrossoverScheduler

    apps = make_apps(T)
    s = CrossoverScheduler(policy, sync_mode="bucket")
    for a in apps:
        s.register(a)
    if not graph:
        s.run()
        return [_flat(a) for a in apps], None
    for _ in range(warm * len(apps)):
        s.step()
    rg = RotationGraph(s, rotations=per)
    rg.begin()
    while rg.t < T:
        rg.replay()
    rg.end()
    s.drain()
    return [_flat(a) for a in apps], rg


@pytest.mark.parametrize("policy_name", ["crossover", "sequential"])
def test_rotation_graph_bitwise_eq_eager_mlp(cuda_device, policy_name):
    """Config 1 shape: 2 x MLP 784-256-10, two simulated workers each, batch 64."""
    from paper_2103_07974_b200.apps import MlpConfig, mlp_app
    from paper_2103_07974_b200.scheduler import Policy

    torch.backends.cuda.matmul.allow_tf32 = False
    pol = Policy(policy_name)

    def make(T):
        return [mlp_app(MlpConfig(dataset_seed=11 + k, workers=2, momentum=0.9), f"m{k}", k, T,
                        cuda_device) for k in range(2)]

    eager, _ = _run(make, pol, 10, graph=False)
    graphed, rg = _run(make, pol, 10, graph=True)
    assert rg.replays == 10 - 3
    unrolled, rg = _run(make, pol, 11, graph=True, per=4)      # 2 launches of 4 rotations
    assert rg.replays == 2
    eager11, _ = _run(make, pol, 11, graph=False)
    for a, b in zip(eager11, unrolled):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    for a, b in zip(eager, graphed):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_rotation_graph_matches_reference_golden(cuda_device):
    """The reference's own 2-job, W = 2 and W = 4 trajectories (fp64 golden) at T = 30."""
    from paper_2103_07974_b200.apps import LossKind, SgdConfig, linear_app
    from paper_2103_07974_b200.scheduler import Policy

    meta = json.loads((GOLDEN / "equivalence_meta.json").read_text())
    arrays = dict(np.load(GOLDEN / "equivalence.npz"))
    done = 0
    for m in meta:
        if not m["key"].startswith("j2_w") or m["key"].startswith("j2_w1") or "perturb" in m:
            continue
        cfgs = [SgdConfig(c["learning_rate"], c["workers"], LossKind(c["loss"]), c["dataset_seed"])
                for c in m["configs"]]

        def make(T, cfgs=cfgs, m=m):
            return [linear_app(c, f"job{j}", m["rng_seeds"][j], T, cuda_device) for j, c in enumerate(cfgs)]

        got, _ = _run(make, Policy.CROSSOVER, m["iterations"], graph=True)
        ref = arrays[m["key"]][:, -1, :]             # [jobs, dim] after the last iteration
        for j in range(len(cfgs)):
            w = got[j][:8].numpy().astype(np.float64)
            assert np.all(np.abs(w - ref[j]) <= 1e-5 + 1e-4 * np.abs(ref[j])), (m["key"], j)
        done += 1
    assert done >= 4


def test_rotation_graph_overlaps_like_alg1(cuda_device):
    """Fixed-time apps (spin compute 2 units, K2 sync ~1 unit): the replayed crossover rotation
    takes N*max(comp, comm) = 2*comp per rotation, the sequential one 2*(comp+comm)."""
    from paper_2103_07974_b200 import graphs
    from paper_2103_07974_b200.apps import fixed_time_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    nbytes = 600_000_000
    rot = {}
    for pol in (Policy.CROSSOVER, Policy.SEQUENTIAL):
        s = CrossoverScheduler(pol, sync_mode="bucket", sync_ctas=-1)
        for j in range(2):
            s.register(fixed_time_app(f"f{j}", 300_000, 700_000, nbytes, 16, cuda_device, seed=j))
        for _ in range(4):
            s.step()
        rg = graphs.RotationGraph(s)
        rg.begin()
        rg.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s.compute_stream)
        for _ in range(10):
            rg.replay()
        b.record(s.compute_stream)
        torch.cuda.synchronize()
        rot[pol] = a.elapsed_time(b) / 10
        comps, comms = rg.phase_times(reps=5)
        rg.end()
        s.drain()
        rot[(pol, "phases")] = (comps, comms)
    comps, comms = rot[(Policy.SEQUENTIAL, "phases")]
    assert max(comms) < min(comps)                      # rho < 1: the sync hides under compute
    assert rot[Policy.CROSSOVER] <= 1.05 * sum(comps)
    assert rot[Policy.SEQUENTIAL] >= 0.95 * (sum(comps) + sum(comms))
