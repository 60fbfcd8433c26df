"""Property-based and report-level parity of the host logic (CPU), in the reference's style
(derandomised hypothesis, tests/conftest.py; the reference's own strategy: SURVEY §4).

* metrics: the package's `measure` / `compare` / `report` on the reference's own spans give the
  reference's reports byte for byte (json, csv, table; tests/golden/metrics.json);
* the device pipeline's emission order (`rotation_schedule`) equals the oracle recurrence for
  any plan, and measured-style traces built from it are legal;
* the bucket layout, the comm predictor and the scenario unit conversion keep their invariants.
"""

import json

from hypothesis import given
from hypothesis import strategies as st

from conftest import GOLDEN
from oracle import schedule as osched
from paper_2103_07974_b200.comm import (Architecture, ClusterSpec, SyncRequest, comm_time,
                                        comm_time_unfused)
from paper_2103_07974_b200.engine import (Phase, Span, Trace, trace_to_chrome_json, trace_to_json,
                                          validate_trace)
from paper_2103_07974_b200.metrics import compare, measure, report
from paper_2103_07974_b200.scenario import scaled_int
from paper_2103_07974_b200.scheduler import (Policy, SchedulePlan, rotation_schedule,
                                             steady_state_period)
from paper_2103_07974_b200.workload import (BucketLayout, JobProfile, TensorSpec,
                                            fuse_gradients, unfused_messages)


def _trace(spans):
    ss = tuple(Span(l, j, Phase(p), t, a, b) for l, j, p, t, a, b in spans)
    return Trace(ss, max((s.end for s in ss), default=0))


def _plan(policy, jobs):
    return SchedulePlan(policy, tuple(JobProfile(j, f, b, (TensorSpec("g", c),), t)
                                      for j, f, b, c, t in jobs))


def test_metrics_reports_match_reference_byte_for_byte():
    cases = {c["name"]: c for c in json.loads((GOLDEN / "schedule.json").read_text())["cases"]}
    golden = json.loads((GOLDEN / "metrics.json").read_text())
    assert len(golden) == 60
    for g in golden:
        c = cases[g["name"]]
        mx = measure(_trace(c["crossover"]["spans"]), _plan(Policy.CROSSOVER, c["jobs"]),
                     scenario=c["name"])
        ms = measure(_trace(c["sequential"]["spans"]), _plan(Policy.SEQUENTIAL, c["jobs"]),
                     scenario=c["name"])
        for fmt in ("json", "csv", "table"):
            assert report(mx, fmt) == g["crossover"][fmt], (g["name"], fmt)
            assert report(ms, fmt) == g["sequential"][fmt], (g["name"], fmt)
            assert report(compare(mx, ms), fmt) == g["compare"][fmt], (g["name"], fmt)
        # span exports (engine.py:245-289): JSON and Chrome trace-event documents
        assert trace_to_json(_trace(c["crossover"]["spans"])) == g["trace_json"], g["name"]
        assert trace_to_chrome_json(_trace(c["crossover"]["spans"])) == g["trace_chrome"], g["name"]


plans = st.lists(st.tuples(st.integers(0, 12), st.integers(1, 12), st.integers(0, 15),
                           st.integers(1, 7)), min_size=1, max_size=4)


@given(plans)
def test_emission_order_is_the_oracle_recurrence(specs):
    jobs = [(f"j{i}", f, b, c, t) for i, (f, b, c, t) in enumerate(specs)]
    order = rotation_schedule([j[0] for j in jobs], [j[4] for j in jobs])
    for run in (osched.crossover, osched.sequential):
        spans, _ = run(jobs)
        assert order == osched.schedule_order(spans)
        assert validate_trace(_trace(spans)) == []


@given(plans)
def test_crossover_never_slower_than_sequential(specs):
    jobs = [(f"j{i}", f, b, c, t) for i, (f, b, c, t) in enumerate(specs)]
    assert osched.crossover(jobs)[1] <= osched.sequential(jobs)[1]


@given(st.integers(1, 20), st.integers(0, 20), st.integers(2, 4))
def test_hiding_condition_period(comp, comm, n):
    """N >= 2 co-located jobs, rho <= 1 => the crossover period is N*comp (SPEC.md:545,
    tests/test_acceptance.py:71-93); the closed form agrees with the recurrence."""
    jobs = [(f"j{i}", comp, 0, comm, 50) for i in range(n)]
    if comm <= comp:
        assert osched.crossover_period(jobs) == n * comp
    assert steady_state_period(Policy.CROSSOVER, [comp] * n, [comm] * n) == n * max(comp, comm)
    assert steady_state_period(Policy.SEQUENTIAL, [comp] * n, [comm] * n) == n * (comp + comm)


@given(st.lists(st.integers(0, 5000), min_size=1, max_size=40), st.sampled_from([1, 4, 32]),
       st.integers(1, 8))
def test_bucket_layout_invariants(numels, align, world):
    lay = BucketLayout.build(numels, align, multiple=align * world)
    assert lay.payload_elems == sum(numels)
    assert all(o % align == 0 for o in lay.offsets)
    ends = [o + n for o, n in zip(lay.offsets, numels)]
    assert all(e <= o2 for e, o2 in zip(ends, lay.offsets[1:]))          # no overlap, in order
    assert lay.total >= ends[-1] and lay.total % (align * world) == 0
    assert lay.total - ends[-1] < align * world                           # minimal padding
    if align == 1 and world == 1:
        assert lay.total == sum(numels)                                   # the reference's prefix sum


sizes = st.lists(st.integers(0, 10**8), min_size=1, max_size=12)


@given(sizes, st.integers(1, 16), st.integers(1, 10**4), st.sampled_from(list(Architecture)))
def test_fusion_never_loses_and_gap_is_latency(sz, w, latency, arch):
    cl = ClusterSpec(w, 12_500_000_000, latency, arch)
    job = JobProfile("j", 1, 1, tuple(TensorSpec(f"t{i}", s) for i, s in enumerate(sz)), 1)
    fused = comm_time(SyncRequest("j", 1, fuse_gradients(job, 1)), cl)
    unfused = comm_time_unfused(unfused_messages(job, 1), cl)
    assert fused <= unfused
    per_msg = (2 * (w - 1) if arch is Architecture.RING_ALLREDUCE else 2) * latency
    if arch is Architecture.RING_ALLREDUCE and w == 1:
        per_msg = 0
    # ceiling rounding can save at most one ns per extra message
    assert (len(sz) - 1) * per_msg <= unfused - fused <= (len(sz) - 1) * (per_msg + 1)


@given(st.integers(-10**12, 10**12), st.integers(0, 6))
def test_scaled_int_exact_decimal(n, k):
    value = n / 10**k
    assert scaled_int(value, 10**6, 1, "f") == n * 10**(6 - k)
