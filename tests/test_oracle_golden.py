"""Pin the CPU oracle against the reference's golden vectors (no GPU needed)."""

import numpy as np
import pytest

from oracle import schedule as osched
from oracle import sgd as osgd

# literal KAT of the reference (tests/test_scheduler.py:42-55)
GOLDEN_CROSSOVER = [
    ("gpu0", "j1", "forward", 1, 0, 1), ("gpu0", "j1", "backward", 1, 1, 2),
    ("nic0", "j1", "sync", 1, 2, 3),
    ("gpu0", "j2", "forward", 1, 2, 3), ("gpu0", "j2", "backward", 1, 3, 4),
    ("nic0", "j2", "sync", 1, 4, 5),
    ("gpu0", "j1", "forward", 2, 4, 5), ("gpu0", "j1", "backward", 2, 5, 6),
    ("nic0", "j1", "sync", 2, 6, 7),
    ("gpu0", "j2", "forward", 2, 6, 7), ("gpu0", "j2", "backward", 2, 7, 8),
    ("nic0", "j2", "sync", 2, 8, 9),
    ("gpu0", "j1", "forward", 3, 8, 9), ("gpu0", "j1", "backward", 3, 9, 10),
    ("nic0", "j1", "sync", 3, 10, 11),
    ("gpu0", "j2", "forward", 3, 10, 11), ("gpu0", "j2", "backward", 3, 11, 12),
    ("nic0", "j2", "sync", 3, 12, 13),
]


def test_literal_golden_crossover():
    spans, makespan = osched.crossover([("j1", 1, 1, 1, 3), ("j2", 1, 1, 1, 3)])
    assert spans == GOLDEN_CROSSOVER
    assert makespan == 13
    assert osched.sequential([("j1", 1, 1, 1, 3), ("j2", 1, 1, 1, 3)])[1] == 18


def test_schedule_matches_reference_emission_order(schedule_golden):
    assert len(schedule_golden) >= 300
    for case in schedule_golden:
        jobs = [tuple(j) for j in case["jobs"]]
        for policy, fn in (("crossover", osched.crossover), ("sequential", osched.sequential)):
            spans, makespan = fn(jobs)
            ref = [tuple(s) for s in case[policy]["spans"]]
            assert spans == ref, (case["name"], policy)
            assert makespan == case[policy]["makespan"], (case["name"], policy)


def test_head_of_line_blocking_case(schedule_golden):
    # B's and C's zero-length syncs queue behind A's long one
    case = next(c for c in schedule_golden if c["name"] == "hol_block")
    spans = case["crossover"]["spans"]
    syncs = [(s[1], s[4], s[5]) for s in spans if s[2] == "sync" and s[3] == 1]
    assert syncs == [("A", 1, 11), ("B", 11, 11), ("C", 11, 11)]


def test_crossover_period_bound(schedule_golden):
    for case in schedule_golden[:120]:
        jobs = [tuple(j) for j in case["jobs"]]
        if len(jobs) < 2:
            continue
        cyc = osched.crossover_period(jobs)
        bound = max(sum(f + b for _, f, b, _, _ in jobs), sum(c for *_, c, _ in jobs),
                    max(f + b + c for _, f, b, c, _ in jobs))
        assert cyc >= bound


def _jobs_from_meta(m, dtype=np.float64):
    return [osgd.LinearJob(c["learning_rate"], c["workers"], c["loss"], c["dataset_seed"], s,
                           c["dim"], c["dataset_size"], c["batch_size"], dtype)
            for c, s in zip(m["configs"], m["rng_seeds"])]


def test_sgd_oracle_bitwise_vs_reference(equivalence_golden):
    meta, arrays = equivalence_golden
    for m in meta:
        jobs = _jobs_from_meta(m)
        traj = osgd.run_crossover(jobs, m["iterations"],
                                  perturb=tuple(m["perturb"]) if "perturb" in m else None)
        got = np.stack([np.stack(t) for t in traj])
        assert np.array_equal(got, arrays[m["key"]]), m["key"]
        if "perturb" not in m:
            iso = np.stack(osgd.run_isolated(jobs[0], m["iterations"]))
            assert np.array_equal(iso, arrays[m["key"] + "_isolated0"]), m["key"]


def test_fp32_drift_bound(equivalence_golden):
    """The same sequence in fp32 stays within the tolerance the GPU tests use."""
    meta, arrays = equivalence_golden
    worst = 0.0
    for m in meta:
        if "perturb" in m:
            continue
        traj = osgd.run_crossover(_jobs_from_meta(m, np.float32), m["iterations"])
        got = np.stack([np.stack(t) for t in traj]).astype(np.float64)
        ref = arrays[m["key"]]
        worst = max(worst, float(np.max(np.abs(got - ref) / (1e-5 + 1e-4 * np.abs(ref)))))
    assert worst < 1.0, worst


def test_average_gradients_basis():
    basis = [np.eye(4)[k] for k in range(4)]
    assert np.array_equal(osgd.average_gradients(basis), np.full(4, 0.25))


def test_sgd_step_exact():
    assert np.array_equal(osgd.sgd_step(np.array([1.0, 1.0]), np.array([1.0, -1.0]), 0.1),
                          np.array([0.9, 1.1]))


@pytest.mark.parametrize("loss", [osgd.LEAST_SQUARES, osgd.LOGISTIC])
def test_gradient_finite_differences(loss):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((30, 6))
    y = x @ rng.standard_normal(6) if loss == osgd.LEAST_SQUARES else (rng.standard_normal(30) > 0) * 1.0

    def f(p):
        z = x @ p
        if loss == osgd.LEAST_SQUARES:
            return 0.5 * np.mean((z - y) ** 2)
        return np.mean(np.logaddexp(0.0, z) - y * z)

    for _ in range(5):
        p = rng.standard_normal(6)
        num = np.array([(f(p + e) - f(p - e)) / 2e-5 for e in np.eye(6) * 1e-5])
        ana = osgd.loss_gradient(loss, p, x, y)
        assert np.linalg.norm(num - ana) / np.linalg.norm(ana) < 1e-6


def test_mlp_gradient_finite_differences():
    rng = np.random.default_rng(5)
    params = [rng.standard_normal((7, 5)) * 0.4, rng.standard_normal(7) * 0.4,
              rng.standard_normal((3, 7)) * 0.4, rng.standard_normal(3) * 0.4]
    x = rng.standard_normal((6, 5))
    y = rng.integers(0, 3, 6)

    def loss(ps):
        w1, b1, w2, b2 = ps
        h = np.maximum(x @ w1.T + b1, 0)
        lg = h @ w2.T + b2
        lg = lg - lg.max(1, keepdims=True)
        return np.mean(np.log(np.exp(lg).sum(1)) - lg[np.arange(6), y])

    grads = osgd.mlp_gradient([p.copy() for p in params], x, y)
    for i in range(4):
        flat = params[i].reshape(-1)
        for k in range(0, flat.size, max(1, flat.size // 7)):
            up = [p.copy() for p in params]
            dn = [p.copy() for p in params]
            up[i].reshape(-1)[k] += 1e-6
            dn[i].reshape(-1)[k] -= 1e-6
            num = (loss(up) - loss(dn)) / 2e-6
            assert abs(num - grads[i].reshape(-1)[k]) < 1e-6


def test_fixture_inventories_match_torchvision(fixtures_golden):
    """The reference's bucket fixtures are torchvision's parameter lists."""
    torchvision = pytest.importorskip("torchvision")
    r = torchvision.models.resnet50()
    sizes = [p.numel() * 4 for p in r.parameters()]
    assert sizes == fixtures_golden["resnet50"]["sizes"]
    assert [n for n, _ in r.named_parameters()] == fixtures_golden["resnet50"]["names"]
    assert sum(sizes) == fixtures_golden["resnet50"]["grad_bytes"] == 102_228_128
    v = torchvision.models.vgg16()
    vs = [p.numel() * 4 for p in v.parameters()]
    assert vs == fixtures_golden["vgg16"]["sizes"]
    assert sum(vs) == 553_430_176 and len(vs) == 32


@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_mlp_trajectory_vs_torch_fp64(momentum):
    """The config-1 MLP oracle has no reference counterpart (SURVEY §8 c), so cross-check the whole
    trajectory against an independent implementation: torch autograd + torch.optim.SGD in fp64,
    the W workers' gradients averaged in worker order (equivalence.py:150-160's structure)."""
    import torch

    T, W, B, size, lr = 4, 2, 16, 256, 0.05
    specs = [(11, 0), (12, 1)]
    traj = osgd.run_mlp_crossover(specs, T, W, batch=B, lr=lr, dataset_size=size, momentum=momentum)
    for k, (ds, rs) in enumerate(specs):
        x, y = osgd.mlp_dataset(ds, size)
        ps = [torch.tensor(p, dtype=torch.float64, requires_grad=True) for p in osgd.mlp_init(rs)]
        opt = torch.optim.SGD(ps, lr=lr, momentum=momentum, foreach=False)
        for t in range(1, T + 1):
            acc = [torch.zeros_like(p) for p in ps]
            for w in range(W):
                idx = osgd.batch_indices(rs, t, w, size, B)
                xb, yb = torch.tensor(x[idx]), torch.tensor(y[idx])
                h = torch.relu(xb @ ps[0].T + ps[1])
                loss = torch.nn.functional.cross_entropy(h @ ps[2].T + ps[3], yb)
                gs = torch.autograd.grad(loss, ps)
                acc = [a + g for a, g in zip(acc, gs)]
            for p, a in zip(ps, acc):
                p.grad = a / W
            opt.step()
            for got, want in zip(traj[k][t - 1], ps):
                np.testing.assert_allclose(got, want.detach().numpy(), rtol=1e-12, atol=1e-14)
