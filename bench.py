"""Benchmark of the crossover step: two co-located ResNet-50 jobs (BASELINE.json config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

A *step* is one rotation: every co-located job does one iteration (forward,
backward, fused-gradient sync: K1 pack -> NCCL all-reduce -> K2 average + SGD).
Rank 0 prints ONE JSON line:

  value       combined images/s of both jobs under crossover, all ranks, inputs
              resident in HBM (device-timed with CUDA events, max over ranks)
  e2e         the same through the public API with pinned-host uint8 batches
              copied H2D every step and every loss read back D2H
  sequential  the back-to-back baseline with the same kernels -> speedup
  roofline    K2 (fused average + SGD update) achieved HBM GB/s vs the measured peak
  cpu_baseline the reference CPU path (oracle port) on a bounded sample
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "combined samples/sec of co-located jobs; crossover-vs-sequential speedup"
UNIT = "images/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--jobs", type=int, default=2)
    ap.add_argument("--model", default="resnet50", choices=["resnet50", "vgg16"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-batch", type=int, default=2)
    ap.add_argument("--nccl-max-ctas", type=int, default=0)
    ap.add_argument("--trace-out", default="")
    ap.add_argument("--no-graphs", action="store_true", help="eager forward/backward (no CUDA graphs)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# reference CPU path (oracle port): rotation + torch-CPU fwd/bwd + numpy fusion/average/SGD
# ---------------------------------------------------------------------------
def cpu_crossover(model_name: str, jobs: int, batch: int, steps: int, warmup: int):
    """The reference's crossover step on the host: the oracle's rotation order
    (oracle/schedule.py), per job a PyTorch-CPU forward/backward of the same
    model (the reference has no model compute of its own), then the oracle's
    fusion (numpy pack into one bucket), fixed-order average over W (= 1 here)
    and the torch-SGD momentum update in numpy fp32.  Returns (samples/s, cores, wall)."""
    import numpy as np
    import torch
    import torchvision

    from oracle import fusion as ofusion
    from oracle import schedule as osched
    from oracle import sgd as osgd

    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    models, bufs = [], []
    for j in range(jobs):
        torch.manual_seed(j)
        m = getattr(torchvision.models, model_name)()
        models.append(m)
        bufs.append([None] * len(list(m.parameters())))
    g = torch.Generator().manual_seed(0)
    x = torch.randn(batch, 3, 224, 224, generator=g)
    y = torch.randint(0, 1000, (batch,), generator=g)
    order = osched.schedule_order(osched.crossover(
        [(f"j{j}", 1, 1, 1, warmup + steps) for j in range(jobs)])[0])
    computes = [(int(job[1:]), t) for lane, job, ph, t in order if ph == "backward"]
    t0 = None
    for n, (j, t) in enumerate(computes):
        if n == warmup * jobs:
            t0 = time.perf_counter()
        m = models[j]
        params = list(m.parameters())
        loss = torch.nn.functional.cross_entropy(m(x), y)
        grads = torch.autograd.grad(loss, params)
        bucket = ofusion.pack([gr.numpy() for gr in grads], 1)           # fuse_gradients
        avg = osgd.average_gradients([bucket])                           # W = 1 worker
        off = 0
        with torch.no_grad():
            for i, p in enumerate(params):
                k = p.numel()
                pn = p.numpy().reshape(-1)
                new, bufs[j][i] = osgd.torch_sgd_step(pn, avg[off:off + k], bufs[j][i], 0.1,
                                                      momentum=0.9, weight_decay=1e-4,
                                                      first=bufs[j][i] is None)
                pn[:] = new
                off += k
    wall = time.perf_counter() - t0
    return jobs * batch * steps / wall, cores, wall


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    val, cores, wall = cpu_crossover(args.model, args.jobs, args.cpu_batch, args.steps, args.warmup)
    sample = (f"{args.jobs} x {args.model} jobs, batch {args.cpu_batch}/job (bounded sample of "
              f"batch {args.batch}), {args.steps} timed rotations, torch-CPU fwd/bwd + oracle "
              f"numpy fusion/average/SGD-momentum, {wall:.1f} s")
    line = {"metric": METRIC, "value": round(val, 3), "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.jobs}x {args.model} crossover, batch {args.batch}/GPU",
                       "jobs": args.jobs, "batch_per_gpu": args.batch, "cpu_batch": args.cpu_batch},
            "cpu_baseline": {"value": round(val, 3), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(val, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        if not sm:
            return None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, name in enumerate(names):
                if len(r) >= 9 and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(name)
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(sm)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2103_07974_b200 import apps
    from paper_2103_07974_b200.comm import NcclCommunicator
    from paper_2103_07974_b200.engine import Phase, schedule_key, trace_to_chrome_json, validate_trace
    from paper_2103_07974_b200.scheduler import (CrossoverScheduler, Policy, overlap_roofline,
                                                 rotation_schedule)

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.backends.cudnn.benchmark = True
    comm = NcclCommunicator(rank, world, max_ctas=args.nccl_max_ctas) if world > 1 else None

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    K, W = args.steps, args.warmup
    build = apps.resnet50_app if args.model == "resnet50" else apps.vgg16_app
    base = [build(f"{args.model}_{j}", args.batch, 1, dev, seed=1000 * j + rank,
                  graphed=not args.no_graphs) for j in range(args.jobs)]
    host_data = None if args.no_e2e else [
        apps._CycleData(apps.synthetic_image_batches(args.batch, 2, 7 + j, dev, host_uint8=True))
        for j in range(args.jobs)]
    samples_per_rot = args.jobs * args.batch * world

    def timed(policy: Policy, e2e: bool, clocks: bool = False):
        sched = CrossoverScheduler(policy, comm=comm, time_kernels=not e2e)
        for j, a in enumerate(base):
            app = dataclasses.replace(a, iterations=W + K,
                                      data=host_data[j] if e2e else a.data)
            sched.register(app)
        loss_host = torch.zeros(len(base), dtype=torch.float32).pin_memory()
        cs, ms = sched.compute_stream, sched.comm_stream

        def one_rotation():
            for j in range(len(base)):
                sched.step()
                if e2e:  # D2H of this step's result
                    st = sched.states[j]
                    with torch.cuda.stream(cs):
                        loss_host[j:j + 1].copy_(st.losses[-1].float().view(1), non_blocking=True)

        for _ in range(W):
            one_rotation()
        sched.drain()
        barrier()
        if sched.timer is not None:
            sched.timer.clear()
        launches0 = sched.kernel_launches
        n_spans0 = len(sched.recorder._pending)
        clk = Clocks(local) if clocks else None
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(cs)
        for _ in range(K):
            one_rotation()
        join = torch.cuda.Event()
        join.record(ms)
        cs.wait_event(join)
        end.record(cs)
        end.synchronize()
        clk_info = clk.stop() if clk else None
        ms_total = max_over_ranks(start.elapsed_time(end))
        launches = sched.kernel_launches - launches0
        trace = sched.recorder.resolve()
        timed_spans = trace.spans[n_spans0:]
        kern = sched.timer.summary() if sched.timer is not None else {}
        sched.drain()
        return {"ms": ms_total, "trace": trace, "timed_spans": timed_spans, "kernels": kern,
                "launches": launches, "clocks": clk_info, "sched": sched}

    cross = timed(Policy.CROSSOVER, e2e=False, clocks=True)
    seq = timed(Policy.SEQUENTIAL, e2e=False)
    e2e = None if args.no_e2e else timed(Policy.CROSSOVER, e2e=True)

    # legality + bit-exact schedule of the measured runs
    order = [a.job_id for a in base]
    for r in (cross, seq):
        assert validate_trace(r["trace"]) == [], validate_trace(r["trace"])[:3]
        assert schedule_key(r["trace"]) == rotation_schedule(order, [W + K] * len(order))

    def per_job(spans, job, phases):
        vals = [s.end - s.start for s in spans if s.job_id == job and s.phase in phases]
        return statistics.median(vals) / 1e6 if vals else 0.0

    # per-job compute / sync medians of the sequential run (no overlap -> isolated costs)
    comp = [per_job(seq["timed_spans"], j, (Phase.FORWARD,)) + per_job(seq["timed_spans"], j, (Phase.BACKWARD,))
            for j in order]
    comm_t = [per_job(seq["timed_spans"], j, (Phase.SYNC,)) for j in order]
    roof = overlap_roofline(comp, comm_t)
    rot_cross = cross["ms"] / K
    rot_seq = seq["ms"] / K
    value = samples_per_rot * K / (cross["ms"] / 1e3)
    seq_value = samples_per_rot * K / (seq["ms"] / 1e3)

    hbm_peak, peak_kind = peaks()
    sync0 = cross["sched"].states[0].sync
    k2_ms = statistics.mean(cross["kernels"].get("k2_update", [0.0]))
    k2_bytes = sync0.k2_bytes()
    k2_gbs = k2_bytes / (k2_ms / 1e3) / 1e9 if k2_ms else 0.0
    kernels = {"k2_update": {"ms": round(k2_ms, 4), "bytes": k2_bytes, "GB/s": round(k2_gbs, 1)}}
    if "k1_pack" in cross["kernels"]:
        k1_ms = statistics.mean(cross["kernels"]["k1_pack"])
        kernels["k1_pack"] = {"ms": round(k1_ms, 4), "bytes": sync0.k1_bytes(),
                              "GB/s": round(sync0.k1_bytes() / (k1_ms / 1e3) / 1e9, 1)}
    if "c1_allreduce" in cross["kernels"]:
        c1_ms = statistics.mean(cross["kernels"]["c1_allreduce"])
        kernels["c1_allreduce"] = {"ms": round(c1_ms, 4), "bus_bytes": sync0.c1_bus_bytes(),
                                   "busbw_GB/s": round(sync0.c1_bus_bytes() / (c1_ms / 1e3) / 1e9, 1),
                                   "peak_GB/s": 900.0}

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cv, cores, wall = cpu_crossover(args.model, args.jobs, args.cpu_batch, 2, 1)
            cpu = {"value": round(cv, 3), "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"{args.jobs} x {args.model}, batch {args.cpu_batch}/job, 2 rotations "
                             f"after 1 warm-up, torch-CPU fwd/bwd + oracle fusion/average/SGD "
                             f"({wall:.1f} s)"}
        e2e_line = None
        if e2e is not None:
            ev = samples_per_rot * K / (e2e["ms"] / 1e3)
            h2d = args.jobs * (args.batch * 224 * 224 * 3 + args.batch * 8)
            e2e_line = {"value": round(ev, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": args.jobs * 4}
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": round(rot_cross, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, N(0,1) images / random labels)",
            "config": {"workload": f"{args.jobs}x {args.model} co-located, crossover, batch "
                                   f"{args.batch}/GPU, bf16 autocast, fp32 params/grads, "
                                   f"SGD momentum 0.9 wd 1e-4"
                                   + ("" if args.no_graphs else ", fwd/bwd as CUDA graphs"),
                       "jobs": args.jobs, "model": args.model, "batch_per_gpu": args.batch,
                       "parallelism": f"dp{world}", "l2": "inputs + activations >> 126 MB L2",
                       "sync_mode": sync0.mode},
            "speedup_vs_sequential": round(rot_seq / rot_cross, 4),
            "sequential": {"value": round(seq_value, 2), "ms_per_step": round(rot_seq, 3)},
            "rho": round(sum(comm_t) / sum(comp), 5) if sum(comp) else None,
            "overlap_roofline": {"per_rotation_ms": {k: round(v, 4) for k, v in roof.items()},
                                 "measured_ms": round(rot_cross, 4),
                                 "frac": round(roof["north_star"] / rot_cross, 4),
                                 "frac_tight": round(roof["tight"] / rot_cross, 4),
                                 "comp_ms": [round(c, 4) for c in comp],
                                 "comm_ms": [round(c, 4) for c in comm_t]},
            "roofline": {"kernel": "k2_update (fused 1/W average + SGD-momentum)", "bound": "hbm",
                         "achieved": round(k2_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(k2_gbs / hbm_peak, 4), "traffic": None,
                         "peak_kind": peak_kind, "bytes_per_launch": k2_bytes},
            "kernels": kernels,
            "gpu_launches": cross["launches"],
            "clocks": cross["clocks"],
            "e2e": e2e_line,
            "cpu_baseline": cpu,
        }
        if args.trace_out:
            Path(args.trace_out).write_text(trace_to_chrome_json(cross["trace"]))
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
