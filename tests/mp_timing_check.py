"""Timing-level Alg. 1 check with a real NVLink sync (W ranks, one per GPU; launched by
tests/test_gpu_schedule_timing.py when >= 2 GPUs are visible).

Same golden plan as the single-GPU test (reference tests/test_scheduler.py:42-97: N = 2, comp = 2,
comm = 1, T = 3 -> makespans 13 / 18), but the sync is the copy-engine transport over NVLink
(K1, flag barriers, CE pulls, shard K2, CE all-gather) between W processes on W GPUs.  The unit is
calibrated as the slowest rank's median sync time; every rank then sizes its compute from it.
"""

import json
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2103_07974_b200.apps import fixed_time_app  # noqa: E402
from paper_2103_07974_b200.comm import PeerGroup  # noqa: E402
from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy  # noqa: E402

BYTES = 400_000_000


def run(policy, comm, dev, specs, T):
    s = CrossoverScheduler(policy, comm=comm, sync_mode="ce", sync_ctas=-1)
    for k, (job, fwd, bwd, nbytes) in enumerate(specs):
        s.register(fixed_time_app(job, fwd, bwd, nbytes, T, dev, seed=k, flat="ipc"))
    # start every rank's device timeline together: under crossover the computes never wait for a
    # sync while there is slack, so a start skew between ranks would persist (absorbed by the early
    # rank's barrier waits) and show up in its makespan
    torch.cuda.synchronize()
    dist.barrier()
    while s.step():
        pass
    s.drain()
    tr = s.recorder.resolve()
    s.close()
    t0 = min(sp.start for sp in tr.spans if sp.phase.value == "forward")
    return [(sp.lane_id, sp.job_id, sp.phase.value, sp.iteration, sp.start - t0, sp.end - t0)
            for sp in tr.spans]


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = PeerGroup(rank, world)
    T = 3
    probe = [("j1", 200_000, 200_000, BYTES), ("j2", 200_000, 200_000, BYTES)]
    run(Policy.SEQUENTIAL, comm, dev, probe, T)                      # warm-up
    cal = run(Policy.SEQUENTIAL, comm, dev, probe, T)
    unit = statistics.median(e - s for *_, ph, t, s, e in cal if ph == "sync")
    t = torch.tensor([unit], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    unit = int(t.item())
    specs = [(j, unit // 2, 3 * unit // 2, BYTES) for j in ("j1", "j2")]
    cross = run(Policy.CROSSOVER, comm, dev, specs, T)
    seq = run(Policy.SEQUENTIAL, comm, dev, specs, T)
    mk = lambda sp: max(x[5] for x in sp)  # noqa: E731
    res = {"world": world, "unit_ms": unit / 1e6, "crossover_units": mk(cross) / unit,
           "sequential_units": mk(seq) / unit, "ratio": mk(seq) / mk(cross)}
    res["ok"] = (abs(res["ratio"] / (18 / 13) - 1) <= 0.05 and abs(res["crossover_units"] - 13) <= 0.65
                 and abs(res["sequential_units"] - 18) <= 0.9)
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        Path(out_path).write_text(json.dumps(allres, indent=1))
        print("TIMINGCHECK " + json.dumps(allres), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not all(r["ok"] for r in allres):
        sys.exit(1)


if __name__ == "__main__":
    main()
