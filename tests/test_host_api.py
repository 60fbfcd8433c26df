"""Host-side logic of the product package (no GPU): schedule emitter, traces, metrics, layout."""

from fractions import Fraction

import pytest

import paper_2103_07974_b200 as cx
from paper_2103_07974_b200 import engine, metrics, workload
from paper_2103_07974_b200.comm import ClusterSpec, comm_time_allreduce, allreduce_bus_bytes
from paper_2103_07974_b200.engine import Phase, Span, Trace
from paper_2103_07974_b200.errors import InvalidTraceError, ComparisonError, DeadlockError
from paper_2103_07974_b200.scheduler import (Policy, SchedulePlan, overlap_roofline,
                                             predicted_speedup, rotation_schedule,
                                             steady_state_period)


def _trace(spans):
    sp = tuple(Span(l, j, Phase(p), t, a, b) for l, j, p, t, a, b in spans)
    return Trace(sp, max((s.end for s in sp), default=0))


def test_rotation_schedule_is_reference_order(schedule_golden):
    """The device pipeline's emission order == the reference's span order, every case."""
    for case in schedule_golden:
        order = [j[0] for j in case["jobs"]]
        budgets = [j[4] for j in case["jobs"]]
        got = rotation_schedule(order, budgets)
        for policy in ("crossover", "sequential"):
            ref = [tuple(s[:4]) for s in case[policy]["spans"]]
            assert got == ref, (case["name"], policy)


def test_validate_trace_accepts_reference_traces(schedule_golden):
    for case in schedule_golden[:100]:
        for policy in ("crossover", "sequential"):
            tr = _trace(case[policy]["spans"])
            assert engine.validate_trace(tr) == []


def test_validate_trace_rejects_violations(schedule_golden):
    spans = [list(s) for s in schedule_golden[0]["crossover"]["spans"]]
    # next forward of j1 starts before its sync completes
    bad = [s[:] for s in spans]
    bad[6][4] -= 2
    out = engine.validate_trace(_trace(bad))
    assert any("compute starts before" in v for v in out)
    # lane overlap on nic0
    bad = [s[:] for s in spans]
    bad[5][4] = 2
    assert any("overlaps" in v for v in engine.validate_trace(_trace(bad)))
    # missing sync for a non-final iteration
    bad = [s for s in spans if not (s[2] == "sync" and s[1] == "j1" and s[3] == 1)]
    assert any("missing sync" in v for v in engine.validate_trace(_trace(bad)))
    # makespan mismatch
    tr = _trace(spans)
    assert engine.validate_trace(Trace(tr.spans, tr.makespan + 1))


def test_metrics_golden(schedule_golden):
    case = schedule_golden[0]
    jobs = [workload.JobProfile(j, f, b, (workload.TensorSpec("g", c),), t)
            for j, f, b, c, t in case["jobs"]]
    px = SchedulePlan(Policy.CROSSOVER, jobs)
    ps = SchedulePlan(Policy.SEQUENTIAL, jobs)
    mx = metrics.measure(_trace(case["crossover"]["spans"]), px, "golden")
    ms = metrics.measure(_trace(case["sequential"]["spans"]), ps, "golden")
    assert mx.makespan == 13
    assert mx.gpu_utilization == Fraction(12, 13)
    assert mx.nic_utilization == Fraction(6, 13)
    assert mx.aggregate_throughput == Fraction(6 * 10**9, 13)
    assert mx.per_job_iteration_period == {"j1": 4, "j2": 4}
    c = metrics.compare(mx, ms)
    assert c.speedup_vs_baseline == Fraction(18, 13)
    assert metrics.metrics_from_json(metrics.report(c, "json")) == c
    csv = metrics.report(c, "csv").splitlines()
    assert csv[0] == metrics.METRICS_CSV_HEADER
    assert csv[-1].startswith("golden,crossover,aggregate,6,,13,")
    assert "speedup: 1.3846" in metrics.report(c, "table")
    assert metrics.samples_per_second(mx, {"j1": 64, "j2": 64}) == pytest.approx(6 * 64 * 1e9 / 13)
    with pytest.raises(ValueError):
        metrics.report(c, "xml")
    with pytest.raises(InvalidTraceError):
        metrics.measure(Trace(_trace(case["crossover"]["spans"]).spans, 99), px)
    other = SchedulePlan(Policy.SEQUENTIAL, jobs[:1])
    with pytest.raises(ComparisonError):
        metrics.compare(mx, metrics.measure(_trace(schedule_golden[1]["sequential"]["spans"]),
                                            SchedulePlan(Policy.SEQUENTIAL, [workload.JobProfile(
                                                "solo", 1, 1, (workload.TensorSpec("g", 1),), 2)])))
    assert other.jobs[0].job_id == "j1"


def test_closed_forms():
    assert steady_state_period(Policy.CROSSOVER, [2, 2], [1, 1]) == 4
    assert steady_state_period(Policy.CROSSOVER, [1, 1], [2, 2]) == 4
    assert steady_state_period(Policy.SEQUENTIAL, [2, 2], [1, 1]) == 6
    assert predicted_speedup([1_000_000] * 2, [150_000] * 2) == Fraction(23, 20)
    assert predicted_speedup([1, 1], [1, 1]) == 2
    assert predicted_speedup([1, 1], [2, 2]) == Fraction(3, 2)
    with pytest.raises(ValueError, match="homogeneous"):
        predicted_speedup([1, 2], [1, 1])
    r = overlap_roofline([1, 1], [0.1, 3])
    assert r["north_star"] == 3.1 and r["tight"] == 4 and r["sequential"] == 5.1


def test_plan_validation():
    with pytest.raises(ValueError):
        SchedulePlan(Policy.CROSSOVER, [])
    j = workload.JobProfile("a", 1, 1, (workload.TensorSpec("g", 4),), 1)
    with pytest.raises(ValueError):
        SchedulePlan(Policy.CROSSOVER, [j, j])


def test_workload_invariants():
    with pytest.raises(ValueError):
        workload.TensorSpec("t", -1)
    with pytest.raises(ValueError):
        workload.JobProfile("a", 0, 0, (workload.TensorSpec("g", 1),), 1)
    with pytest.raises(ValueError):
        workload.JobProfile("a", 1, 0, (), 1)
    with pytest.raises(ValueError):
        workload.JobProfile("a", 1, 0, (workload.TensorSpec("g", 1), workload.TensorSpec("g", 2)), 1)
    j = workload.JobProfile("a", 1, 2, tuple(workload.TensorSpec(f"t{i}", s)
                                            for i, s in enumerate([3, 1000, 481, 77, 0])), 2)
    assert workload.fuse_gradients(j, 1).size_bytes == 1561
    assert len(workload.unfused_messages(j, 2)) == 5
    with pytest.raises(ValueError):
        workload.fuse_gradients(j, 3)
    assert workload.comp_time(j) == 3


@pytest.mark.parametrize("align", [1, 4, 32])
def test_bucket_layout(align):
    numels = [200704, 256, 2560, 10, 0, 7]
    lay = workload.BucketLayout.build(numels, align)
    assert lay.payload_bytes == 4 * sum(numels)
    assert all(o % align == 0 for o in lay.offsets)
    assert lay.total % align == 0 and lay.total >= lay.offsets[-1] + numels[-1]
    for a, b, n in zip(lay.offsets, lay.offsets[1:], numels):
        assert b >= a + n and b - (a + n) < align
    if align == 1:
        assert lay.total == sum(numels)


def test_comm_predictor_kats():
    mb = 10**6
    ring = lambda w, lat=0: ClusterSpec(w, 12_500_000_000, lat)  # noqa: E731
    assert comm_time_allreduce(400 * mb, ring(1)) == 0
    assert comm_time_allreduce(0, ring(4, 10_000)) == 60_000
    assert comm_time_allreduce(400 * mb, ring(4, 5_000)) == 48_030_000
    assert allreduce_bus_bytes(102_228_128, 8) == pytest.approx(178_899_224)
    fused = comm_time_allreduce(1561, ClusterSpec(2, 10**9, 5_000))
    unfused = sum(comm_time_allreduce(s, ClusterSpec(2, 10**9, 5_000)) for s in [3, 1000, 481, 77, 0])
    assert unfused - fused == 2 * 5_000 * 4


def test_errors_semantics():
    e = DeadlockError("a", 3, "policy=crossover")
    assert e.job_id == "a" and e.iteration == 3 and "policy=crossover" in str(e)
    e = InvalidTraceError([str(i) for i in range(7)])
    assert "(+2 more)" in str(e) and len(e.violations) == 7
    assert issubclass(cx.ConfigError, ValueError)


def test_chrome_and_json_exports(schedule_golden):
    tr = _trace(schedule_golden[0]["crossover"]["spans"])
    import json
    doc = json.loads(engine.trace_to_chrome_json(tr))
    assert {e["args"]["name"] for e in doc["traceEvents"] if e["ph"] == "M"} == {"gpu0", "nic0"}
    rows = json.loads(engine.trace_to_json(tr))
    assert rows[0] == {"lane_id": "gpu0", "job_id": "j1", "phase": "forward", "iteration": 1,
                       "start_ns": 0, "end_ns": 1}
    assert engine.schedule_key(tr)[:3] == [("gpu0", "j1", "forward", 1), ("gpu0", "j1", "backward", 1),
                                           ("nic0", "j1", "sync", 1)]


def test_bucket_layout_multiple_for_shards():
    lay = workload.BucketLayout.build([10, 33, 7], 32, multiple=32 * 4)
    assert lay.total % 128 == 0 and lay.total >= lay.offsets[-1] + 7
    with pytest.raises(ValueError):
        workload.BucketLayout.build([1], 32, multiple=48)


def test_flatten_parameters_keeps_values_and_strides():
    import torch

    from paper_2103_07974_b200.fusion import flatten_parameters

    torch.manual_seed(0)
    conv = torch.nn.Conv2d(3, 8, 3).to(memory_format=torch.channels_last)
    lin = torch.nn.Linear(5, 3)
    params = list(conv.parameters()) + list(lin.parameters())
    before = [p.detach().clone() for p in params]
    strides = [p.stride() for p in params]
    flat, lay = flatten_parameters(params, 32, shards=4)
    assert flat.numel() == lay.total and lay.total % 128 == 0
    for p, b, st, off in zip(params, before, strides, lay.offsets):
        assert torch.equal(p, b) and p.stride() == st
        assert p.data_ptr() == flat.data_ptr() + 4 * off
    y = conv(torch.randn(1, 3, 6, 6).contiguous(memory_format=torch.channels_last))
    assert y.shape == (1, 8, 4, 4)
