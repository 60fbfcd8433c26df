"""Generate the golden fixtures by running the REFERENCE itself (colosim).

Run in the build container, where /root/reference exists:

    python tests/golden/gen_golden.py

Outputs (committed, small):
  schedule.json      reference span lists (emission order) + makespans for the
                     golden 2-job plan and 300 seeded random plans, both policies
  equivalence.npz    reference fp64 trajectories of run_crossover / run_isolated for a
                     grid of (jobs, workers, loss, T) plus one perturbed run
  fixtures.json      reference fixture bucket inventories (resnet50, vgg16 sizes)

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

    losses = (LossKind.LEAST_SQUARES, LossKind.LOGISTIC)
    arrays = {}
    meta = []
    for n_jobs in (1, 2, 3):
        for workers in (1, 2, 4):
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
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
