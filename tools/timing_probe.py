"""Print measured vs predicted spans of the timing-level schedule tests (diagnostics).

    python tools/timing_probe.py [sync_ctas ...]
"""
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import schedule as osched  # noqa: E402
from paper_2103_07974_b200.apps import fixed_time_app  # noqa: E402
from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy  # noqa: E402

BYTES = 1_200_000_000


def run(policy, specs, T, sync_ctas):
    s = CrossoverScheduler(policy, sync_ctas=sync_ctas)
    for k, (job, fwd, bwd, nbytes) in enumerate(specs):
        s.register(fixed_time_app(job, fwd, bwd, nbytes, T, torch.device("cuda", 0), seed=k))
    tr = s.run()
    t0 = min(sp.start for sp in tr.spans if sp.phase.value == "forward")
    return [(sp.lane_id, sp.job_id, sp.phase.value, sp.iteration, sp.start - t0, sp.end - t0) for sp in tr.spans]


def main():
    caps = [int(x) for x in sys.argv[1:]] or [0, -1]
    for cap in caps:
        probe = [("j1", 200_000, 200_000, BYTES), ("j2", 200_000, 200_000, BYTES)]
        run(Policy.SEQUENTIAL, probe, 3, cap)
        cal = run(Policy.SEQUENTIAL, probe, 3, cap)
        unit = statistics.median(e - s for *_, ph, t, s, e in cal if ph == "sync")
        specs = [(j, unit // 2, 3 * unit // 2, BYTES) for j in ("j1", "j2")]
        for pol, rec in ((Policy.CROSSOVER, osched.crossover), (Policy.SEQUENTIAL, osched.sequential)):
            sp = run(pol, specs, 3, cap)
            jobs = [(j, unit // 2, 3 * unit // 2, unit, 3) for j in ("j1", "j2")]
            pred, ms = rec(jobs)
            print(f"cap={cap} {pol.value} unit={unit/1e6:.3f} ms makespan={max(s[5] for s in sp)/unit:.2f} "
                  f"(pred {ms/unit:.2f})")
            for m, p in zip(sp, pred):
                print(f"   {m[0]} {m[1]} {m[2]:8s} t{m[3]}  {m[4]/unit:6.2f}-{m[5]/unit:6.2f}   pred {p[4]/unit:6.2f}-{p[5]/unit:6.2f}")


if __name__ == "__main__":
    main()
