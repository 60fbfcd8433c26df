"""Generate the golden fixtures by running the REFERENCE itself (colosim).

Run in the build container, where /root/reference exists:

    python tests/golden/gen_golden.py

Outputs (committed, small):
  schedule.json      reference span lists (emission order) + makespans for the
                     golden 2-job plan and 300 seeded random plans, both policies
  equivalence.npz    reference fp64 trajectories of run_crossover / run_isolated for a
                     grid of (jobs, workers, loss, T) plus one perturbed run
  fixtures.json      reference fixture bucket inventories (resnet50, vgg16 sizes)
  metrics.json       the reference's metrics reports (json / csv / table, both policies + the
                     crossover-vs-sequential comparison) for the first 60 schedule cases
  scenarios.json     the reference's scenario files (pkg/scenarios/*.json) with the reference
                     parser's result and simulated makespan for each, plus ~30 malformed
                     documents with the reference parser's exact error message

The GPU box has no /root/reference: tests there read only these files.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main() -> None:
    sys.path.insert(0, str(REF))
    from colosim.comm import Architecture, ClusterSpec
    from colosim.equivalence import LossKind, SgdConfig, run_crossover, run_isolated
    from colosim.scheduler import Policy, SchedulePlan, schedule_crossover, schedule_sequential
    from colosim.workload import JobProfile, TensorSpec, fixture_profile

    # PS at 2e9 B/s with zero latency prices S bytes at exactly S ns (tests/test_scheduler.py:21-25)
    ns = ClusterSpec(workers=2, bandwidth_bytes_per_sec=2_000_000_000, latency_per_message=0,
                     architecture=Architecture.PARAMETER_SERVER)

    def plan(policy, specs):
        return SchedulePlan(policy, tuple(JobProfile(j, f, b, (TensorSpec("g", c),), t)
                                          for j, f, b, c, t in specs), ns)

    def spans(trace):
        return [[s.lane_id, s.job_id, s.phase.value, s.iteration, s.start, s.end]
                for s in trace.spans]

    cases = [{"name": "golden_2jobs", "jobs": [["j1", 1, 1, 1, 3], ["j2", 1, 1, 1, 3]]},
             {"name": "solo", "jobs": [["solo", 1, 1, 1, 2]]},
             {"name": "hol_block", "jobs": [["A", 1, 0, 10, 2], ["B", 1, 0, 0, 2], ["C", 1, 0, 0, 2]]},
             {"name": "unequal_budgets", "jobs": [["a", 2, 1, 2, 5], ["b", 1, 1, 4, 2], ["c", 1, 2, 1, 3]]}]
    rng = random.Random(20260810)
    for k in range(300):
        specs = []
        for i in range(rng.randint(1, 4)):
            fwd = rng.randint(0, 12)
            bwd = rng.randint(1, 12) if fwd == 0 else rng.randint(0, 12)
            specs.append([f"j{i}", fwd, bwd, rng.randint(0, 15), rng.randint(1, 7)])
        cases.append({"name": f"random_{k}", "jobs": specs})
    for c in cases:
        cross = schedule_crossover(plan(Policy.CROSSOVER, c["jobs"]))
        seq = schedule_sequential(plan(Policy.SEQUENTIAL, c["jobs"]))
        c["crossover"] = {"spans": spans(cross), "makespan": cross.makespan}
        c["sequential"] = {"spans": spans(seq), "makespan": seq.makespan}
    (OUT / "schedule.json").write_text(json.dumps({"generator": "colosim (reference) 0.1.0",
                                                   "cases": cases}, separators=(",", ":")) + "\n")

    from colosim.engine import trace_to_chrome_json, trace_to_json
    from colosim.metrics import compare, measure, report
    mcases = []
    for c in cases[:60]:
        px, ps = plan(Policy.CROSSOVER, c["jobs"]), plan(Policy.SEQUENTIAL, c["jobs"])
        mx = measure(schedule_crossover(px), px, scenario=c["name"])
        ms = measure(schedule_sequential(ps), ps, scenario=c["name"])
        cmp = compare(mx, ms)
        mcases.append({"name": c["name"],
                       "crossover": {f: report(mx, f) for f in ("json", "csv", "table")},
                       "sequential": {f: report(ms, f) for f in ("json", "csv", "table")},
                       "compare": {f: report(cmp, f) for f in ("json", "csv", "table")},
                       "trace_json": trace_to_json(schedule_crossover(px)),
                       "trace_chrome": trace_to_chrome_json(schedule_crossover(px))})
    (OUT / "metrics.json").write_text(json.dumps(mcases, separators=(",", ":")) + "\n")

    losses = (LossKind.LEAST_SQUARES, LossKind.LOGISTIC)
    arrays = {}
    meta = []
    for n_jobs in (1, 2, 3):
        for workers in (1, 2, 4, 8):
            for seed in (0, 3):
                iters = 30
                cfgs = [SgdConfig(learning_rate=0.05, workers=workers, loss=losses[j % 2],
                                  dataset_seed=1000 * seed + 10 * n_jobs + j) for j in range(n_jobs)]
                rng_seeds = [seed * 31 + j for j in range(n_jobs)]
                cross = run_crossover(cfgs, iters, rng_seeds)
                key = f"j{n_jobs}_w{workers}_s{seed}"
                arrays[key] = np.stack([np.stack([s.parameters for s in tr]) for tr in cross])
                arrays[key + "_isolated0"] = np.stack(
                    [s.parameters for s in run_isolated(cfgs[0], iters, rng_seeds[0])])
                meta.append({"key": key, "iterations": iters, "rng_seeds": rng_seeds,
                             "configs": [{"learning_rate": c.learning_rate, "workers": c.workers,
                                          "loss": c.loss.value, "dataset_seed": c.dataset_seed,
                                          "dim": c.dim, "dataset_size": c.dataset_size,
                                          "batch_size": c.batch_size} for c in cfgs]})
    pert_cfgs = [SgdConfig(0.05, 2, LossKind.LEAST_SQUARES, 41), SgdConfig(0.05, 2, LossKind.LEAST_SQUARES, 42)]
    pert = run_crossover(pert_cfgs, 10, [0, 1], perturb=(1, 4))
    arrays["perturb"] = np.stack([np.stack([s.parameters for s in tr]) for tr in pert])
    meta.append({"key": "perturb", "iterations": 10, "rng_seeds": [0, 1], "perturb": [1, 4],
                 "configs": [{"learning_rate": 0.05, "workers": 2, "loss": "least_squares",
                              "dataset_seed": s, "dim": 8, "dataset_size": 128, "batch_size": 16}
                             for s in (41, 42)]})
    np.savez_compressed(OUT / "equivalence.npz", **arrays)
    (OUT / "equivalence_meta.json").write_text(json.dumps(meta, indent=1) + "\n")

    fixtures = {}
    for name in ("resnet50", "vgg16"):
        prof = fixture_profile(name)
        fixtures[name] = {"tensors": len(prof.tensors), "grad_bytes": prof.grad_bytes,
                          "sizes": [t.size_bytes for t in prof.tensors],
                          "names": [t.name for t in prof.tensors]}
    (OUT / "fixtures.json").write_text(json.dumps(fixtures, separators=(",", ":")) + "\n")
    scenario_golden()
    print("wrote", sorted(p.name for p in OUT.iterdir()))


def scenario_golden() -> None:
    import copy
    import math

    from colosim.comm import SyncRequest, comm_time
    from colosim.errors import ConfigError
    from colosim.scenario import parse_scenario
    from colosim.workload import fuse_gradients
    from colosim.scheduler import simulate

    def parsed(sc):
        c = sc.cluster
        return {"name": sc.name, "policy": sc.policy.value, "override": sc.iterations_override,
                "cluster": [c.workers, c.gpus_per_worker, c.bandwidth_bytes_per_sec,
                            c.latency_per_message, c.architecture.value, c.ps_servers],
                "jobs": [[j.job_id, j.forward_time, j.backward_time, j.iterations,
                          [[t.name, t.size_bytes] for t in j.tensors]] for j in sc.jobs],
                "comm_ns": [comm_time(SyncRequest(j.job_id, 1, fuse_gradients(j, 1)), c)
                            for j in sc.jobs]}

    files = {}
    for f in sorted((REF.parent / "scenarios").glob("*.json")):
        doc = json.loads(f.read_text())
        sc = parse_scenario(doc, origin=f.name)
        out = parsed(sc)
        for iters in (None, 3):
            plan = sc.plan(iters)
            tr = simulate(plan)
            out[f"makespan_iters_{iters}"] = tr.makespan
            out[f"spans_iters_{iters}"] = len(tr.spans)
        files[f.name] = {"doc": doc, "parsed": out}

    base = files["speedup_band.json"]["doc"]
    ps = files["vgg16_2jobs_10g.json"]["doc"]

    def mut(fn, src=None):
        d = copy.deepcopy(base if src is None else src)
        fn(d)
        return d

    def setk(path, value):
        def f(d):
            o = d
            for k in path[:-1]:
                o = o[k]
            o[path[-1]] = value
        return f

    def delk(path):
        def f(d):
            o = d
            for k in path[:-1]:
                o = o[k]
            del o[path[-1]]
        return f

    bad = [
        ("top_level_array", [1, 2]),
        ("missing_name", mut(delk(["name"]))),
        ("empty_name", mut(setk(["name"], ""))),
        ("unknown_policy", mut(setk(["policy"], "fifo"))),
        ("missing_policy", mut(delk(["policy"]))),
        ("jobs_not_list", mut(setk(["jobs"], {}))),
        ("empty_jobs", mut(setk(["jobs"], []))),
        ("job_not_object", mut(setk(["jobs", 0], 7))),
        ("job_missing_id", mut(delk(["jobs", 0, "job_id"]))),
        ("job_empty_id", mut(setk(["jobs", 0, "job_id"], ""))),
        ("duplicate_ids", mut(setk(["jobs", 1, "job_id"], "band-a"))),
        ("unknown_profile", mut(setk(["jobs", 0], {"job_id": "x", "profile": "alexnet"}))),
        ("profile_bad_iterations", mut(setk(["jobs", 0], {"job_id": "x", "profile": "vgg16", "iterations": 0}))),
        ("inline_missing_iterations", mut(delk(["jobs", 0, "iterations"]))),
        ("inline_bool_iterations", mut(setk(["jobs", 0, "iterations"], True))),
        ("inline_float_iterations", mut(setk(["jobs", 0, "iterations"], 2.0))),
        ("missing_forward", mut(delk(["jobs", 0, "forward_ms"]))),
        ("missing_grad", mut(delk(["jobs", 1, "grad_mb"]))),
        ("tensor_count_zero", mut(setk(["jobs", 0, "tensor_count"], 0))),
        ("tensor_count_huge", mut(setk(["jobs", 0, "tensor_count"], 10001))),
        ("negative_grad", mut(setk(["jobs", 0, "grad_mb"], -1))),
        ("sub_unit_forward", mut(setk(["jobs", 0, "forward_ms"], 1e-7))),
        ("sub_unit_grad", mut(setk(["jobs", 0, "grad_mb"], 0.0000005))),
        ("negative_backward", mut(setk(["jobs", 0, "backward_ms"], -1))),
        ("zero_compute", mut(lambda d: d["jobs"][0].update(forward_ms=0, backward_ms=0))),
        ("string_number", mut(setk(["jobs", 0, "forward_ms"], "30"))),
        ("bool_number", mut(setk(["jobs", 0, "backward_ms"], False))),
        ("overflow", mut(setk(["jobs", 0, "grad_mb"], 1e30))),
        ("infinite", mut(setk(["jobs", 0, "forward_ms"], math.inf))),
        ("nan", mut(setk(["jobs", 0, "forward_ms"], math.nan))),
        ("override_zero", mut(setk(["iterations_override"], 0))),
        ("missing_cluster", mut(delk(["cluster"]))),
        ("cluster_not_object", mut(setk(["cluster"], [4]))),
        ("unknown_architecture", mut(setk(["cluster", "architecture"], "mesh"))),
        ("missing_architecture", mut(delk(["cluster", "architecture"]))),
        ("zero_bandwidth", mut(setk(["cluster", "bandwidth_gbps"], 0))),
        ("sub_unit_bandwidth", mut(setk(["cluster", "bandwidth_gbps"], 1e-10))),
        ("zero_workers", mut(setk(["cluster", "workers"], 0))),
        ("missing_workers", mut(delk(["cluster", "workers"]))),
        ("zero_gpus_per_worker", mut(setk(["cluster", "gpus_per_worker"], 0))),
        ("negative_latency", mut(setk(["cluster", "latency_us"], -1))),
        ("sub_unit_latency", mut(setk(["cluster", "latency_us"], 0.0001))),
        ("zero_ps_servers", mut(setk(["cluster", "ps_servers"], 0), ps)),
    ]
    errors = []
    for name, doc in bad:
        try:
            parse_scenario(doc, origin="bad.json")
            msg = None
        except ConfigError as exc:
            msg = str(exc)
        # json cannot carry inf / nan: keep them as markers the test turns back into floats
        text = json.dumps(doc).replace("Infinity", '"__inf__"').replace("NaN", '"__nan__"')
        errors.append({"name": name, "doc": json.loads(text), "error": msg})
    ok = [{"name": "layered_override", "doc": mut(lambda d: d["jobs"].__setitem__(
        0, {"job_id": "r", "profile": "resnet50", "iterations": 7}))}]
    for o in ok:
        o["parsed"] = parsed(parse_scenario(o["doc"], origin="ok.json"))
    (OUT / "scenarios.json").write_text(json.dumps({"files": files, "errors": errors, "ok": ok},
                                                   separators=(",", ":")) + "\n")


if __name__ == "__main__":
    main()
