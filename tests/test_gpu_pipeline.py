"""Parity of the device crossover pipeline -- ladder L3 (weights) and L4 (neutrality),
plus the bit-exact phase schedule and legality of measured traces."""

import numpy as np
import pytest
import torch

from oracle import sgd as osgd

pytestmark = pytest.mark.gpu

# stated fp32 tolerance vs the fp64 reference: |w_gpu - w_ref| <= ATOL + RTOL * |w_ref|
ATOL, RTOL = 1e-5, 1e-4


def _cfgs(m):
    from paper_2103_07974_b200.apps import LossKind, SgdConfig

    return [SgdConfig(c["learning_rate"], c["workers"], LossKind(c["loss"]), c["dataset_seed"],
                      c["dim"], c["dataset_size"], c["batch_size"]) for c in m["configs"]]


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False


def test_weights_match_reference_golden(cuda_device, equivalence_golden):
    """Per-iteration weights of every job vs the reference's fp64 trajectories."""
    from paper_2103_07974_b200 import equivalence as deq

    meta, arrays = equivalence_golden
    worst = 0.0
    for m in meta:
        pert = tuple(m["perturb"]) if "perturb" in m else None
        traj = deq.run_crossover(_cfgs(m), m["iterations"], m["rng_seeds"], perturb=pert)
        got = np.stack([np.stack([s.parameters for s in t]) for t in traj]).astype(np.float64)
        ref = arrays[m["key"]]
        ratio = np.abs(got - ref) / (ATOL + RTOL * np.abs(ref))
        worst = max(worst, float(ratio.max()))
        assert ratio.max() <= 1.0, (m["key"], float(ratio.max()))
    print(f"worst |dw| / (atol + rtol|w|) = {worst:.3f}")


def test_neutrality_bitwise_on_device(cuda_device):
    from paper_2103_07974_b200 import equivalence as deq

    cfgs = [deq.SgdConfig(0.05, 4, deq.LossKind.LEAST_SQUARES, 21),
            deq.SgdConfig(0.05, 4, deq.LossKind.LOGISTIC, 22)]
    rep = deq.check_neutrality(cfgs, 100, [1, 2])
    assert rep.equal and rep.max_abs_deviation == 0.0


def test_perturbation_is_detected_on_device(cuda_device):
    from paper_2103_07974_b200 import equivalence as deq

    cfgs = [deq.SgdConfig(0.05, 2, deq.LossKind.LEAST_SQUARES, 41),
            deq.SgdConfig(0.05, 2, deq.LossKind.LEAST_SQUARES, 42)]
    rep = deq.check_neutrality(cfgs, 10, [0, 1], perturb=(1, 4))
    assert not rep.equal and rep.first_divergence[:2] == (1, 4)


def test_job_order_irrelevant_on_device(cuda_device):
    from paper_2103_07974_b200 import equivalence as deq

    a = deq.SgdConfig(0.05, 2, deq.LossKind.LEAST_SQUARES, 31)
    b = deq.SgdConfig(0.05, 2, deq.LossKind.LOGISTIC, 32)
    fwd = deq.run_crossover([a, b], 30, [5, 6])
    rev = deq.run_crossover([b, a], 30, [6, 5])
    for x, y in zip(fwd[0], rev[1]):
        assert np.array_equal(x.parameters, y.parameters)


def _linear_sched(policy, budgets, ids, record_weights=False):
    from paper_2103_07974_b200.apps import LossKind, SgdConfig, linear_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler

    s = CrossoverScheduler(policy, record_weights=record_weights)
    dev = torch.device("cuda", 0)
    for k, (j, t) in enumerate(zip(ids, budgets)):
        cfg = SgdConfig(0.05, 2, LossKind.LEAST_SQUARES if k % 2 == 0 else LossKind.LOGISTIC, 100 + k)
        s.register(linear_app(cfg, j, k, t, dev))
    return s


@pytest.mark.parametrize("case_name", ["golden_2jobs", "solo", "hol_block", "unequal_budgets",
                                       "random_0", "random_7", "random_42"])
def test_measured_schedule_bitexact_and_legal(cuda_device, schedule_golden, case_name):
    from paper_2103_07974_b200.engine import schedule_key, validate_trace
    from paper_2103_07974_b200.scheduler import Policy

    case = next(c for c in schedule_golden if c["name"] == case_name)
    ids = [j[0] for j in case["jobs"]]
    budgets = [j[4] for j in case["jobs"]]
    for policy in (Policy.CROSSOVER, Policy.SEQUENTIAL):
        trace = _linear_sched(policy, budgets, ids).run()
        ref = [tuple(s[:4]) for s in case[policy.value]["spans"]]
        assert schedule_key(trace) == ref
        assert validate_trace(trace) == []


def test_sequential_and_crossover_weights_identical(cuda_device):
    from paper_2103_07974_b200.scheduler import Policy

    a = _linear_sched(Policy.CROSSOVER, [7, 5], ["a", "b"], record_weights=True)
    b = _linear_sched(Policy.SEQUENTIAL, [7, 5], ["a", "b"], record_weights=True)
    a.run()
    b.run()
    for j in ("a", "b"):
        assert torch.equal(a.weights(j), b.weights(j))


def test_sequential_gpu_idles_during_sync(cuda_device):
    from paper_2103_07974_b200.engine import Phase
    from paper_2103_07974_b200.scheduler import Policy

    tr = _linear_sched(Policy.SEQUENTIAL, [4, 4], ["a", "b"]).run()
    comp = [(s.start, s.end) for s in tr.spans if s.phase is not Phase.SYNC]
    for s in tr.spans:
        if s.phase is Phase.SYNC:
            assert all(ce <= s.start or cs >= s.end for cs, ce in comp)


def test_mlp_config1_matches_oracle(cuda_device):
    """Config 1: two MLP 784-256-10 jobs, W=2 (simulated workers), batch 64, lr 0.05."""
    from paper_2103_07974_b200.apps import MlpConfig, mlp_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    T = 15
    specs = [(11, 0), (12, 1)]
    sched = CrossoverScheduler(Policy.CROSSOVER, record_weights=True)
    for k, (ds, rs) in enumerate(specs):
        sched.register(mlp_app(MlpConfig(dataset_seed=ds), f"mlp{k}", rs, T, cuda_device))
    sched.run()
    ref = osgd.run_mlp_crossover(specs, T, workers=2)
    from paper_2103_07974_b200.workload import BucketLayout

    lay = BucketLayout.build([256 * 784, 256, 10 * 256, 10], 32)
    worst = 0.0
    for k in range(2):
        w = sched.weights(f"mlp{k}").cpu().numpy().astype(np.float64)
        for t in range(T):
            for i, o in enumerate(lay.offsets):
                r = ref[k][t][i].reshape(-1)
                g = w[t, o:o + r.size]
                ratio = np.abs(g - r) / (1e-5 + 1e-4 * np.abs(r))   # the L3 bar
                worst = max(worst, float(ratio.max()))
    assert worst <= 1.0, worst


def test_direct_vs_bucket_pipeline_identical(cuda_device):
    from paper_2103_07974_b200.apps import MlpConfig, mlp_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    out = []
    for mode in ("direct", "bucket"):
        s = CrossoverScheduler(Policy.CROSSOVER, record_weights=True, sync_mode=mode)
        s.register(mlp_app(MlpConfig(workers=1, dataset_seed=3), "m", 0, 5, cuda_device))
        s.run()
        out.append(s.weights("m").clone())
    assert torch.equal(out[0], out[1])


def test_resnet50_two_jobs_smoke(cuda_device):
    from paper_2103_07974_b200.apps import resnet50_app
    from paper_2103_07974_b200.engine import schedule_key, validate_trace
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy, rotation_schedule

    s = CrossoverScheduler(Policy.CROSSOVER)
    for k in range(2):
        s.register(resnet50_app(f"r{k}", 8, 3, cuda_device, seed=k))
    before = [p.detach().clone() for p in s.states[0].app.params[:3]]
    tr = s.run()
    assert schedule_key(tr) == rotation_schedule(["r0", "r1"], [3, 3])
    assert validate_trace(tr) == []
    assert all(torch.isfinite(l).all() for st in s.states for l in st.losses)
    assert any(not torch.equal(a, b) for a, b in zip(before, s.states[0].app.params[:3]))


def test_resnet50_graphed_two_jobs(cuda_device):
    """Forward/backward replayed as CUDA graphs: same pipeline, legal trace, finite losses."""
    from paper_2103_07974_b200.apps import resnet50_app
    from paper_2103_07974_b200.engine import schedule_key, validate_trace
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy, rotation_schedule

    s = CrossoverScheduler(Policy.CROSSOVER)
    for k in range(2):
        s.register(resnet50_app(f"g{k}", 8, 4, cuda_device, seed=k, graphed=True))
    before = s.states[1].app.params[0].detach().clone()
    tr = s.run()
    assert schedule_key(tr) == rotation_schedule(["g0", "g1"], [4, 4])
    assert validate_trace(tr) == []
    assert all(torch.isfinite(l).all() for st in s.states for l in st.losses)
    assert not torch.equal(before, s.states[1].app.params[0])


def test_mixed_models_bert_vgg(cuda_device):
    """Config 5 shape: heterogeneous apps (VGG-16, BERT-base) co-located on one GPU."""
    from paper_2103_07974_b200.apps import bert_app, vgg16_app
    from paper_2103_07974_b200.engine import validate_trace
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    s = CrossoverScheduler(Policy.CROSSOVER)
    s.register(vgg16_app("vgg", 4, 2, cuda_device))
    s.register(bert_app("bert", 2, 32, 2, cuda_device))
    tr = s.run()
    assert validate_trace(tr) == []
    assert [st.sync.layout.payload_bytes for st in s.states][0] == 553_430_176
    assert all(torch.isfinite(l).all() for st in s.states for l in st.losses)


@pytest.mark.parametrize("workers", [1, 3, 4])
def test_momentum_linear_matches_oracle(cuda_device, workers):
    """torch-SGD momentum through K2 (W simulated workers) vs the fp64 momentum oracle."""
    from paper_2103_07974_b200.apps import LossKind, SgdConfig, linear_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    cfgs = [SgdConfig(0.05, workers, LossKind.LEAST_SQUARES, 51), SgdConfig(0.05, workers, LossKind.LOGISTIC, 52)]
    s = CrossoverScheduler(Policy.CROSSOVER, record_weights=True)
    for k, c in enumerate(cfgs):
        s.register(linear_app(c, f"j{k}", 7 + k, 25, cuda_device, momentum=0.9))
    s.run()
    for k, c in enumerate(cfgs):
        ref = np.stack(osgd.run_isolated_momentum(
            osgd.LinearJob(0.05, workers, c.loss.value, c.dataset_seed, 7 + k), 25, 0.9))
        got = s.weights(f"j{k}")[:, :8].cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= ATOL + RTOL * np.abs(ref))


def test_simulate_measure_compare_on_device(cuda_device):
    """Reference-shaped API end to end: SchedulePlan -> simulate (on the GPU) -> measure -> compare."""
    from paper_2103_07974_b200.apps import MlpConfig, mlp_app
    from paper_2103_07974_b200.metrics import compare, measure, report
    from paper_2103_07974_b200.scheduler import Policy, SchedulePlan, simulate

    mk = lambda: [mlp_app(MlpConfig(workers=1, dataset_seed=k), f"m{k}", k, 6, cuda_device)  # noqa: E731
                  for k in range(2)]
    px = SchedulePlan(Policy.CROSSOVER, mk())
    ps = SchedulePlan(Policy.SEQUENTIAL, mk())
    mx = measure(simulate(px), px, "mlp")
    ms = measure(simulate(ps), ps, "mlp")
    c = compare(mx, ms)
    assert c.per_job_iterations == {"m0": 6, "m1": 6}
    assert c.speedup_vs_baseline > 0 and 0 < c.gpu_utilization <= 1
    assert "speedup" in report(c, "table")


def test_e2e_host_batches_resnet(cuda_device):
    """Pinned-host uint8 batches are copied on the H2D stream and normalised on the device."""
    from paper_2103_07974_b200.apps import resnet50_app
    from paper_2103_07974_b200.engine import validate_trace
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    s = CrossoverScheduler(Policy.CROSSOVER)
    for k in range(2):
        s.register(resnet50_app(f"h{k}", 8, 2, cuda_device, seed=k, host_data=True))
    tr = s.run()
    assert validate_trace(tr) == []
    assert all(torch.isfinite(l).all() for st in s.states for l in st.losses)


def test_watchdog_raises_deadlock_error(cuda_device):
    """No completion within the watchdog limit -> DeadlockError naming the pending (job, iteration)."""
    from paper_2103_07974_b200.apps import MlpConfig, mlp_app
    from paper_2103_07974_b200.errors import DeadlockError
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    app = mlp_app(MlpConfig(workers=1), "slow", 0, 1, cuda_device)
    inner = app.loss_fn

    def slow_loss(model, batch):
        torch.cuda._sleep(2_000_000_000)          # ~1 s of device time
        return inner(model, batch)

    app.loss_fn = slow_loss
    s = CrossoverScheduler(Policy.CROSSOVER, watchdog_s=0.05)
    s.register(app)
    s.step()
    with pytest.raises(DeadlockError) as ei:
        s.drain()
    assert ei.value.job_id == "slow" and ei.value.iteration == 1
    torch.cuda.synchronize()
