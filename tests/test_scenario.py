"""Scenario files: the reference's config surface parsed identically, priced identically, and
turned into device plans.

Golden: tests/golden/scenarios.json, made by gen_golden.py from the reference's own parser on its
five bundled scenario files and on ~40 malformed documents (exact error texts)."""

import json
import math

import pytest

from conftest import GOLDEN
from oracle import schedule as osched
from paper_2103_07974_b200.comm import SyncRequest, comm_time
from paper_2103_07974_b200.errors import ConfigError
from paper_2103_07974_b200.scenario import load_config, parse_scenario, scaled_int
from paper_2103_07974_b200.scheduler import Policy
from paper_2103_07974_b200.workload import fuse_gradients


@pytest.fixture(scope="module")
def golden():
    return json.loads((GOLDEN / "scenarios.json").read_text())


def _parsed(sc):
    c = sc.cluster
    return {"name": sc.name, "policy": sc.policy.value, "override": sc.iterations_override,
            "cluster": [c.workers, c.gpus_per_worker, c.bandwidth_bytes_per_sec,
                        c.latency_per_message, c.architecture.value, c.ps_servers],
            "jobs": [[j.job_id, j.forward_time, j.backward_time, j.iterations,
                      [[t.name, t.size_bytes] for t in j.tensors]] for j in sc.jobs],
            "comm_ns": [comm_time(SyncRequest(j.job_id, 1, fuse_gradients(j, 1)), c)
                        for j in sc.jobs]}


def _unmark(x):
    if x == "__inf__":
        return math.inf
    if x == "__nan__":
        return math.nan
    if isinstance(x, dict):
        return {k: _unmark(v) for k, v in x.items()}
    if isinstance(x, list):
        return [_unmark(v) for v in x]
    return x


def test_reference_scenario_files_parse_identically(golden, tmp_path):
    assert len(golden["files"]) == 5
    for fname, g in golden["files"].items():
        sc = parse_scenario(g["doc"], origin=fname)
        got = _parsed(sc)
        want = {k: v for k, v in g["parsed"].items() if not k.startswith(("makespan", "spans"))}
        assert got == want, fname
        # the same file through load_config
        p = tmp_path / fname
        p.write_text(json.dumps(g["doc"]))
        assert _parsed(load_config(p)) == want


def test_reference_scenarios_schedule_identically(golden):
    """Parsed jobs + the comm predictor through the oracle recurrence give the reference's
    simulated makespan and span count (default budgets and a 3-iteration override)."""
    for fname, g in golden["files"].items():
        sc = parse_scenario(g["doc"], origin=fname)
        for iters in (None, 3):
            plan = sc.plan(iters)
            jobs = [(j.job_id, j.forward_time, j.backward_time,
                     comm_time(SyncRequest(j.job_id, 1, fuse_gradients(j, 1)), sc.cluster),
                     j.iterations) for j in plan.jobs]
            run = osched.crossover if plan.policy is Policy.CROSSOVER else osched.sequential
            spans, makespan = run(jobs)
            assert makespan == g["parsed"][f"makespan_iters_{iters}"], (fname, iters)
            assert len(spans) == g["parsed"][f"spans_iters_{iters}"], (fname, iters)


def test_malformed_documents_fail_with_the_reference_message(golden):
    assert len(golden["errors"]) >= 40
    for case in golden["errors"]:
        doc = _unmark(case["doc"])
        if case["error"] is None:
            parse_scenario(doc, origin="bad.json")
            continue
        with pytest.raises(ConfigError) as exc:
            parse_scenario(doc, origin="bad.json")
        assert str(exc.value) == case["error"], case["name"]


def test_profile_job_with_budget_override(golden):
    for case in golden["ok"]:
        sc = parse_scenario(case["doc"], origin="ok.json")
        want = {k: v for k, v in case["parsed"].items() if k != "comm_ns"}
        got = {k: v for k, v in _parsed(sc).items() if k != "comm_ns"}
        assert got == want
        assert sc.profiles[0] == "resnet50"


def test_load_config_file_errors(tmp_path):
    with pytest.raises(ConfigError, match="cannot read config"):
        load_config(tmp_path / "absent.json")
    p = tmp_path / "broken.json"
    p.write_text('{\n  "name": "x",\n  "policy": crossover\n}')
    with pytest.raises(ConfigError, match=r"parse error at line 3 column 13"):
        load_config(p)


def test_scaled_int_units():
    assert scaled_int(30, 10**6, 1, "f") == 30_000_000
    assert scaled_int(1e-6, 10**6, 1, "f") == 1
    assert scaled_int(100, 10**9, 8, "f") == 12_500_000_000
    assert scaled_int(124.75, 10**6, 1, "f") == 124_750_000
    with pytest.raises(ConfigError, match="whole internal unit"):
        scaled_int(0.1, 1, 1, "f")


def test_iterations_override_layering(golden):
    sc = parse_scenario(golden["files"]["speedup_band.json"]["doc"])
    assert {j.iterations for j in sc.plan().jobs} == {1000}
    assert {j.iterations for j in sc.plan(7).jobs} == {7}
    with pytest.raises(ConfigError, match="override must be >= 1"):
        sc.plan(0)


def test_device_plan_rejects_unspreadable_workers(golden):
    """Without a process group the world is 1: up to 8 simulated workers, not 0 and not 16."""
    sc = parse_scenario(golden["files"]["golden_2jobs.json"]["doc"])
    with pytest.raises(ConfigError, match="cannot be spread"):
        sc.device_plan("cpu", workers=0)
    big = parse_scenario(golden["files"]["resnet50_2jobs_100g.json"]["doc"])
    with pytest.raises(ConfigError, match="16 workers cannot be spread over 1 rank"):
        big.device_plan("cpu")


# -- device runs of scenario files (B200) ---------------------------------------------------

@pytest.mark.gpu
def test_golden_scenario_runs_on_device(cuda_device, golden):
    """golden_2jobs.json (W = 2 workers emulated on one GPU) through the device pipeline: the
    measured trace has the reference's phase schedule (bit-exact) and is legal."""
    from paper_2103_07974_b200.engine import schedule_key, validate_trace
    from paper_2103_07974_b200.metrics import measure
    from paper_2103_07974_b200.scheduler import simulate

    sc = parse_scenario(golden["files"]["golden_2jobs.json"]["doc"])
    for policy in (Policy.CROSSOVER, Policy.SEQUENTIAL):
        plan = sc.device_plan(cuda_device, policy=policy)
        assert [a.local_workers for a in plan.jobs] == [2, 2]
        trace = simulate(plan)
        spans, _ = (osched.crossover if policy is Policy.CROSSOVER else osched.sequential)(
            [(j.job_id, 1, 1, 1, j.iterations) for j in sc.jobs])
        assert schedule_key(trace) == osched.schedule_order(spans)
        assert len(trace.spans) == golden["files"]["golden_2jobs.json"]["parsed"]["spans_iters_None"]
        assert validate_trace(trace) == []
        m = measure(trace, plan, scenario=sc.name)
        assert dict(m.per_job_iterations) == {"j1": 3, "j2": 3}


@pytest.mark.gpu
def test_inline_jobs_calibrated_compute_and_exact_split(cuda_device, golden):
    """speedup_band.json scaled to ~2 ms of compute per iteration: the synthetic apps carry the
    job's exact tensor split and their measured compute lands near the calibrated target."""
    from paper_2103_07974_b200.engine import Phase, validate_trace
    from paper_2103_07974_b200.scheduler import simulate

    sc = parse_scenario(golden["files"]["speedup_band.json"]["doc"])
    plan = sc.device_plan(cuda_device, iterations=6, time_scale=0.02, workers=1)
    for app, job in zip(plan.jobs, sc.jobs):
        assert [p.numel() * 4 for p in app.params] == [t.size_bytes for t in job.tensors]
    trace = simulate(plan)
    assert validate_trace(trace) == []
    comp: dict = {}
    for s in trace.spans:
        if s.phase is not Phase.SYNC and s.iteration > 2:
            comp[(s.job_id, s.iteration)] = comp.get((s.job_id, s.iteration), 0) + s.end - s.start
    target = 100e6 * 0.02          # forward 30 ms + backward 70 ms, scaled: 2 ms
    med = sorted(comp.values())[len(comp) // 2]
    assert 0.6 * target < med < 1.6 * target, med
