"""Benchmark of the crossover step (BASELINE.json config 2 by default; --config mlp = config 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config resnet50|mlp]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

A *step* is one rotation: every co-located job does one iteration (forward,
backward, fused-gradient sync: K1 pack -> bucket exchange -> K2 average + SGD).
Rank 0 prints ONE JSON line:

  value       combined samples/s of the jobs under crossover, all ranks, inputs
              resident in HBM (device-timed with CUDA events, max over ranks)
  e2e         the same through the public API with pinned-host batches copied H2D
              every step and every loss read back D2H
  sequential  the back-to-back baseline with the same sync transport -> speedup_vs_sequential
  roofline    the dominant sync kernel (K2 / fused P2P kernel) vs the measured peak
  cpu_baseline the reference's CPU path on the host cores (oracle port) on a bounded sample
              of the same workload; --impl reference prints that arm alone with the same config
"""

from __future__ import annotations

import argparse
import dataclasses
import gc
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


def _grid_arg(v: str):
    return v if v == "auto" else int(v)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50", choices=["resnet50", "mlp"],
                    help="resnet50: BASELINE config 2 (default); mlp: config 1 (2 x MLP 784-256-10, "
                         "W = 2 workers, batch 64; at N = 1 the two workers are simulated on one GPU)")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--jobs", type=int, default=2)
    ap.add_argument("--model", default="resnet50", choices=["resnet50", "vgg16"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-batch", type=int, default=2)
    ap.add_argument("--nccl-max-ctas", type=int, default=0)
    ap.add_argument("--scenario", default="", help="run a reference scenario JSON file's jobs")
    ap.add_argument("--scenario-time-scale", type=float, default=0.02,
                    help="multiplier on inline scenario jobs' forward/backward ms")
    ap.add_argument("--barrier", default="auto", choices=["auto", "flags", "nccl"],
                    help="cross-rank barrier of the p2p / ce transports: SM-free stream-memory-op "
                         "flags (auto when supported) or a 1-element NCCL all-reduce")
    ap.add_argument("--p2p-ctas", type=int, default=0, help="persistent grid cap of the fused P2P kernel")
    ap.add_argument("--reg-shape", type=int, default=None,
                    help="K1/K2 launch shape (cs_tune reg_shape: 0..4 = unroll x CTAs/SM)")
    ap.add_argument("--p2p-registers", action="store_true",
                    help="capped P2P launches use the register kernel instead of the cp.async.bulk (TMA) one")
    ap.add_argument("--rotation-graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each rotation as one CUDA graph (graphs.RotationGraph); auto = on for "
                         "--config mlp (launch-bound), off for the image models")
    ap.add_argument("--sync-ctas", type=_grid_arg, default=None,
                    help="persistent grid cap of K1/K2 (-1 = 2 CTAs per SM, 0 = one CTA per chunk, "
                         "auto = measured in the untimed probe; default: the scheduler's)")
    ap.add_argument("--comm-priority", default="high", choices=["high", "low"],
                    help="comm stream priority (low: the sync fills gaps left by the compute)")
    ap.add_argument("--mix", default="", help="co-located mix, e.g. resnet50:256,vgg16:32,bert:16 "
                                              "(configs 3/5); overrides --model/--jobs/--batch")
    ap.add_argument("--trace-out", default="", help="Chrome trace (JSON) of the measured crossover run")
    ap.add_argument("--metrics-out", default="", help="colosim.metrics/v1 JSON + CSV of the measured runs")
    ap.add_argument("--no-graphs", action="store_true", help="eager forward/backward (no CUDA graphs)")
    ap.add_argument("--aten-bn", action="store_true", help="ATen BatchNorm instead of the NHWC BN kernels")
    ap.add_argument("--cudnn-stem", action="store_true",
                    help="cuDNN for the RGB stem convolution instead of im2col + tensor-core GEMMs")
    ap.add_argument("--side-grads", action="store_true",
                    help="hand each bottleneck's identity gradient to the producing BN's backward "
                         "(cs_bn_backward2) instead of an autograd add kernel")
    ap.add_argument("--bn-no-pdl", action="store_true",
                    help="launch the BN finalize / apply kernels without programmatic dependent launch")
    ap.add_argument("--sync-mode", default="auto", choices=["auto", "bucket", "sharded", "p2p", "p2p_gather",
                                                            "ce", "unfused", "nvls"],
                    help="W>1 sync: all-reduce bucket, reduce-scatter/all-gather (sharded) or "
                         "the fused NVLink P2P kernel; ce = copy-engine pulls + shard K2; auto = ce "
                         "under crossover and p2p for the sequential arm (bucket if peers cannot "
                         "be mapped)")
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


NVLINK_P2P_GBS = 770.0   # measured peer copy per direction (B200_PROFILING.md)
# NVLS ceiling: multimem.ld_reduce + multimem.st of every rank's 102 MB shard with nothing else in
# the kernel (no update, no barriers), 64 CTAs, all ranks at once, as all-reduce bus GB/s
# (tools/nvls_ceiling.cu, profiles/r02_nvls_ceiling/w{2,4}_102.json)
NVLS_CEILING_BUSBW = {2: 391.8, 4: 672.6}


def roofline_line(kernels: dict, sync, hbm_peak: float, peak_kind: str, model: str,
                  isolated: dict | None = None, sync_seq=None) -> dict:
    """Roofline of the path's dominant kernel: K2 (HBM), or in p2p mode the fused NVLink kernel,
    or in ce mode the shard K2 with the copy-engine transport beside it.

    Under crossover the P2P kernel is launched on a deliberately small grid (it overlaps the
    other app's compute and only has to finish inside it), so its live fraction is low by
    design; ``isolated`` is the same kernel at the full grid in the sequential arm."""
    if "k2_nvls_fused" in kernels:
        k = kernels["k2_nvls_fused"]
        ach = k["nvlink_GB/s"]
        return {"kernel": "k2_nvls_fused (multimem.ld_reduce of every rank's bucket shard through the "
                          "NVSwitch, /W, SGD-momentum, multimem.st of the new shard to every rank)",
                "bound": "nvlink", "achieved": ach, "peak": NVLINK_P2P_GBS, "unit": "GB/s",
                "frac": round(ach / NVLINK_P2P_GBS, 4), "traffic": None,
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                "bytes_per_launch": k["nvlink_bytes"], "grid_cap_ctas": int(sync._nvls.max_ctas) or "2 per SM",
                "bytes_convention": "all-reduce bus bytes 2(W-1)/W*S (NCCL busbw)",
                "link_bytes_per_direction": k["link_bytes_per_direction"],
                "link_frac": round(k["link_GB/s"] / NVLINK_P2P_GBS, 4),
                "nvls_ceiling": ({"busbw_GBps": NVLS_CEILING_BUSBW[sync.ranks],
                                  "frac": round(ach / NVLS_CEILING_BUSBW[sync.ranks], 4),
                                  "source": "tools/nvls_ceiling.cu, 102 MB, 64 CTAs"}
                                 if sync.ranks in NVLS_CEILING_BUSBW else None)}
    if "k2_p2p_gather" in kernels:
        k = kernels["k2_p2p_gather"]
        per_dir = sync.c1_bus_bytes()
        ach = per_dir / (k["ms"] / 1e3) / 1e9
        return {"kernel": "k2_p2p_gather (no K1: NVLink reads of every rank's gradient tensors in place, "
                          "rank-order sum, /W, SGD-momentum, NVLink writes of the new shard to every rank)",
                "bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_P2P_GBS, "unit": "GB/s",
                "frac": round(ach / NVLINK_P2P_GBS, 4), "traffic": None,
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                "bytes_per_launch": per_dir, "grid_cap_ctas": int(sync._gather_ctas) or "2 per SM"}
    if "k2_p2p_fused" in kernels:
        k = kernels["k2_p2p_fused"]
        per_dir = sync.c1_bus_bytes()          # 2(W-1)/W * S through each GPU's links per direction
        ach = per_dir / (k["ms"] / 1e3) / 1e9
        out = {"kernel": "k2_p2p_fused (NVLink reads of every rank's bucket shard, rank-order sum, "
                         "/W, SGD-momentum, NVLink writes of the new shard to every rank)",
               "bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_P2P_GBS, "unit": "GB/s",
               "frac": round(ach / NVLINK_P2P_GBS, 4),
               "traffic": ncu_traffic(f"k2_p2p_fused/{model}/emulated_w{sync.ranks}/momentum"),
               "traffic_note": "DRAM bytes of the same kernel with the W ranks' buffers local "
                               "(ncu cannot replay a multi-rank run)",
               "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
               "bytes_per_launch": per_dir,
               "grid_cap_ctas": int(sync._p2p.max_ctas) or "2 per SM"}
        ki = (isolated or {}).get("k2_p2p_fused")
        if ki:
            ach_i = per_dir / (ki["ms"] / 1e3) / 1e9
            out["isolated"] = {"achieved": round(ach_i, 1), "frac": round(ach_i / NVLINK_P2P_GBS, 4),
                               "grid_cap_ctas": "2 per SM", "arm": "sequential"}
        if "k1_pack" in kernels:
            k1 = kernels["k1_pack"]
            out["hbm_kernel"] = {"kernel": "k1_pack", "achieved": k1["GB/s"], "peak": hbm_peak,
                                 "frac": round(k1["GB/s"] / hbm_peak, 4), "bytes_per_launch": k1["bytes"]}
        return out
    k2 = kernels.get("k2_update", {"GB/s": 0.0})
    if "c1_ce_reduce_scatter" in kernels:
        # copy-engine transport: K2 (on the shard, W sources) is the dominant kernel of ours;
        # the two CE copy phases are reported against the NVLink peer-copy peak beside it
        t = kernels["c1_ce_reduce_scatter"]["ms"] + kernels["c1_ce_all_gather"]["ms"]
        ach = sync.c1_bus_bytes() / (t / 1e3) / 1e9
        out = {"kernel": "k2_update (W-source shard reduce, /W, SGD-momentum) beside copy-engine "
                         "reduce-scatter / all-gather pulls", "bound": "hbm",
                "achieved": k2["GB/s"], "peak": hbm_peak, "unit": "GB/s",
                "frac": round(k2["GB/s"] / hbm_peak, 4),
                "traffic": ncu_traffic(f"k2_update/{model}/ce_w{sync.ranks}/momentum"),
                "note": ("live: the shard K2 waits for SM slots held by the other app's "
                         "convolutions; alone the same kernel runs at 0.91 (W = 2) / 0.86 (W = 4) "
                         "of the measured peak (profiles/r01_shard_kernels_ncu.md)"),
                "peak_kind": peak_kind, "bytes_per_launch": sync.k2_bytes("ce"),
                "transport": {"engine": "copy engines (cudaMemcpyAsync peer pulls, no SM)",
                              "achieved": round(ach, 1), "peak": NVLINK_P2P_GBS, "unit": "GB/s",
                              "frac": round(ach / NVLINK_P2P_GBS, 4),
                              "bytes_per_sync": sync.c1_bus_bytes()}}
        if isolated and sync_seq is not None and sync_seq.mode == "p2p":
            seq_line = roofline_line(isolated, sync_seq, hbm_peak, peak_kind, model)
            out["sequential_arm"] = {k: seq_line[k] for k in ("kernel", "bound", "achieved", "peak",
                                                               "unit", "frac", "grid_cap_ctas")}
        return out
    if "c1_allreduce" in kernels and "k2_update" not in kernels:
        c1 = kernels["c1_allreduce"]
        return {"kernel": "sync graph (NCCL all-reduce + K2) of the rotation graph", "bound": "nvlink",
                "achieved": c1["busbw_GB/s"], "peak": NVLINK_P2P_GBS, "unit": "GB/s",
                "frac": round(c1["busbw_GB/s"] / NVLINK_P2P_GBS, 4), "traffic": None,
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                "bytes_per_launch": c1["bus_bytes"],
                "note": "a 0.8 MB bucket: latency-bound, the fraction says so"}
    return {"kernel": "k2_update (fused 1/W average + SGD-momentum)", "bound": "hbm",
            "achieved": k2["GB/s"], "peak": hbm_peak, "unit": "GB/s",
            "frac": round(k2["GB/s"] / hbm_peak, 4),
            "traffic": ncu_traffic(f"k2_update/{model}/{sync.mode}/momentum"),
            "peak_kind": peak_kind, "bytes_per_launch": sync.k2_bytes()}


def ncu_traffic(key: str):
    """dram read + write bytes per launch from a committed ncu --set full capture (or None)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(key)
    return None if d is None else d["dram_read_bytes"] + d["dram_write_bytes"]


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


def cpu_mlp(workers: int, steps: int, warmup: int):
    """Config 1 on the host: the oracle's MLP restatement of run_crossover (fp64 numpy, the
    reference's seeding / fixed-order averaging / sgd_step, equivalence.py:129-232) for 2 jobs x
    `workers` workers x batch 64.  Returns (samples/s, wall s)."""
    from oracle import sgd as osgd

    specs = [(11, 0), (12, 1)]
    osgd.run_mlp_crossover(specs, warmup, workers=workers)         # untimed (BLAS warm-up)
    t0 = time.perf_counter()
    osgd.run_mlp_crossover(specs, steps, workers=workers)
    wall = time.perf_counter() - t0
    return len(specs) * workers * 64 * steps / wall, wall


def reference_paths() -> dict:
    """The reference's own CPU algorithms (restated in oracle/, the GPU box has no /root/reference)
    timed on this host at the sizes BASELINE.md §3 quotes: the schedule recurrence of
    scheduler.schedule_crossover / schedule_sequential (N = 2, T = 1000 -> 6,000 spans) and the
    numeric run_crossover (2 linear jobs x W = 2 x T = 1000, dim 8, batch 16)."""
    from oracle import schedule as osched
    from oracle import sgd as osgd

    jobs = [(f"j{k}", 1, 1, 1, 1000) for k in range(2)]
    t0 = time.perf_counter()
    spans, _ = osched.crossover(jobs)
    spans2, _ = osched.sequential(jobs)
    t_sched = time.perf_counter() - t0
    lj = [osgd.LinearJob(0.05, 2, osgd.LEAST_SQUARES, 20, 0), osgd.LinearJob(0.05, 2, osgd.LOGISTIC, 21, 1)]
    t0 = time.perf_counter()
    osgd.run_crossover(lj, 1000)
    t_num = time.perf_counter() - t0
    return {"schedule_spans_per_s": round((len(spans) + len(spans2)) / t_sched),
            "run_crossover_job_iterations_per_s": round(2 * 1000 / t_num),
            "run_crossover_samples_per_s": round(2 * 2 * 16 * 1000 / t_num),
            "note": "oracle restatements of scheduler.py:209-218 / equivalence.py:190-232 "
                    "(BASELINE.md §3: 197 k spans/s, 6.4 k job-iterations/s on the survey host)"}


def host_threads() -> dict:
    import torch

    info = {"cores": len(os.sched_getaffinity(0)), "torch_threads": torch.get_num_threads()}
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [{"api": d.get("internal_api"), "threads": d.get("num_threads")}
                        for d in threadpool_info()]
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        pass
    return info


def workload_config(args, world: int) -> dict:
    """The `config` object of the bench line -- identical for both arms (ours / reference)."""
    if args.config == "mlp":
        w = max(2, world)
        return {"workload": f"2x MLP 784-256-10 co-located, crossover, {w} data-parallel workers, "
                            "batch 64/worker, SGD lr 0.05 (BASELINE config 1)",
                "jobs": 2, "model": "mlp784-256-10", "workers": w, "batch_per_worker": 64,
                "parallelism": f"dp{world}"}
    if args.mix or args.scenario:
        return {"workload": f"{args.scenario or args.mix} co-located, crossover",
                "jobs": len((args.mix or "").split(",")) if args.mix and not args.scenario else None,
                "model": args.mix or args.scenario, "parallelism": f"dp{world}",
                "l2": "inputs + activations >> 126 MB L2"}
    return {"workload": (f"{args.jobs}x {args.model} co-located, crossover, batch {args.batch}/GPU, "
                         "SGD momentum 0.9 (BASELINE config 2; arithmetic type in `dtype`)"),
            "jobs": args.jobs, "model": args.model, "batch_per_gpu": args.batch,
            "parallelism": f"dp{world}", "l2": "inputs + activations >> 126 MB L2"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    host = host_threads()
    if args.config == "mlp":
        w = max(2, world)
        val, wall = cpu_mlp(w, args.steps, args.warmup)
        sample = (f"the whole workload: 2 MLP jobs x {w} workers (simulated serially, "
                  f"equivalence.py:171-174) x batch 64 x {args.steps} rotations after {args.warmup} "
                  f"warm-up, oracle fp64 numpy ({wall:.2f} s)")
        dtype = "f64"
    else:
        val, _, wall = cpu_crossover(args.model, args.jobs, args.cpu_batch, args.steps, args.warmup)
        sample = (f"{args.jobs} x {args.model} jobs, batch {args.cpu_batch}/job per rotation (bounded "
                  f"sample of batch {args.batch}), {args.steps} timed rotations after {args.warmup} "
                  f"warm-up, torch-CPU fwd/bwd + oracle numpy fusion/average/SGD-momentum ({wall:.1f} s)")
        dtype = "f32"
    line = {"metric": METRIC, "value": round(val, 3), "unit": unit_of(args), "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": workload_config(args, world),
            "cpu_baseline": {"value": round(val, 3), "unit": unit_of(args), "cores": host["cores"],
                             "kind": "port", "sample": sample, "threads": host,
                             "reference_paths": reference_paths()},
            "e2e": {"value": round(val, 3), "unit": unit_of(args), "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def unit_of(args) -> str:
    return "samples/s" if args.config == "mlp" else UNIT


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


class Energy:
    """The GPU's cumulative energy counter (NVML, mJ) around a timed region: average board power over
    it, against the enforced power limit (tools/band.py's power accounting)."""

    def __init__(self, device):
        import pynvml
        import torch

        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda._get_nvml_device_index(device))
        self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0

    def read(self) -> tuple[float, float]:
        return time.perf_counter(), self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) / 1000.0

    @staticmethod
    def between(a, b) -> dict:
        dt = b[0] - a[0]
        return {"joules": round(b[1] - a[1], 4), "seconds": round(dt, 5),
                "watts": round((b[1] - a[1]) / dt, 1) if dt > 0 else None}


class Harness:
    """Per-process plumbing shared by bench.py and the tools (band, c1bench, cebench): device, comm,
    barrier, max over ranks."""

    def __init__(self, nccl_max_ctas: int = 0):
        import torch
        import torch.distributed as dist

        from paper_2103_07974_b200.comm import NcclCommunicator

        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = dist_env()
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1 and not dist.is_initialized():
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
        torch.backends.cudnn.benchmark = True
        self.comm = NcclCommunicator(self.rank, self.world, max_ctas=nccl_max_ctas) if self.world > 1 else None

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def mean_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64)
        self.dist.all_reduce(t)
        return float(t.item()) / self.world

    def close(self):
        if self.comm is not None:
            self.comm.close()
        if self.world > 1:
            self.dist.destroy_process_group()


P2P_CTAS: int | None = None   # --p2p-ctas; None = the scheduler's per-policy default
SYNC_CTAS: int | None = None  # --sync-ctas; None = the scheduler's default K1 / K2 grid
PACK_ENGINE = "sm"            # --pack-engine: K1 by a kernel (sm) or by the copy engines (ce)
BARRIER = "auto"              # --barrier: cross-rank barrier of the p2p / ce transports
ENERGY: Energy | None = None  # set by tools/band.py: NVML energy counter around timed regions


def timed_run(h: Harness, base, policy, W: int, K: int, host_data=None, clocks: bool = False,
              time_kernels: bool = True, sync_mode: str = "auto", comm_priority: int = -1,
              p2p_ctas: int | None = None, graph: bool = False):
    """W untimed rotations, drain + barrier, then K timed rotations (CUDA events, max over ranks).

    A rotation = every app in `base` steps once.  With `host_data` every step's batch is copied
    H2D from pinned host memory and every loss is read back D2H (the e2e measurement).
    """
    import torch

    from paper_2103_07974_b200.scheduler import CrossoverScheduler

    if graph:
        return timed_run_graph(h, base, policy, W, K, host_data, clocks, sync_mode, comm_priority,
                               p2p_ctas)
    mode = sync_mode if h.world > 1 else "auto"
    sched = CrossoverScheduler(policy, comm=h.comm, time_kernels=time_kernels, sync_mode=mode,
                               comm_priority=comm_priority,
                               p2p_ctas=P2P_CTAS if p2p_ctas is None else p2p_ctas,
                               barrier=BARRIER, sync_ctas=SYNC_CTAS, pack_engine=PACK_ENGINE)
    for j, a in enumerate(base):
        sched.register(dataclasses.replace(a, iterations=W + K,
                                           data=host_data[j] if host_data else a.data))
    loss_host = torch.zeros(len(base), dtype=torch.float32).pin_memory()
    cs, ms = sched.compute_stream, sched.comm_stream

    def one_rotation():
        for j in range(len(base)):
            sched.step()
            if host_data:  # D2H of this step's result
                with torch.cuda.stream(cs):
                    loss_host[j:j + 1].copy_(sched.states[j].losses[-1].float().view(1), non_blocking=True)

    for _ in range(W):
        one_rotation()
    sched.drain()
    h.barrier()
    if sched.timer is not None:
        sched.timer.clear()
    launches0 = sched.kernel_launches
    n_spans0 = len(sched.recorder._pending)
    # Python's cyclic GC can pause the host for tens of ms (the previous runs' autograd / span
    # objects); a paused host lets the GPU queue drain.  Collect now, keep it off while timing.
    gc.collect()
    gc.disable()
    clk = Clocks(h.local) if clocks else None
    e0 = ENERGY.read() if ENERGY is not None else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(cs)
    for _ in range(K):
        one_rotation()
    join = torch.cuda.Event()
    join.record(ms)
    cs.wait_event(join)
    end.record(cs)
    end.synchronize()
    energy = Energy.between(e0, ENERGY.read()) if e0 is not None else None
    gc.enable()
    clk_info = clk.stop() if clk else None
    ms_total = h.max_over_ranks(start.elapsed_time(end))
    trace = sched.recorder.resolve()
    sched.drain()
    sched.close()
    out = {"ms": ms_total, "trace": trace, "timed_spans": trace.spans[n_spans0:],
           "replicas_identical": replicas_identical(h, base),
           "kernels": sched.timer.summary() if sched.timer is not None else {},
           "launches": sched.kernel_launches - launches0, "clocks": clk_info, "energy": energy,
           "sched": sched}
    return out


def timed_run_graph(h: Harness, base, policy, W: int, K: int, host_data=None, clocks: bool = False,
                    sync_mode: str = "bucket", comm_priority: int = -1, p2p_ctas: int | None = None):
    """timed_run in graph mode (paper_2103_07974_b200.graphs): W eager rotations, the graph-layout
    rotation + capture, two untimed replays, then K timed replays (one launch per rotation).
    With `host_data` every replay is preceded by the H2D copies of that rotation's batches into the
    graph's static inputs (pinned host -> device) and followed by the D2H of every loss."""
    import torch

    from paper_2103_07974_b200.graphs import RotationGraph
    from paper_2103_07974_b200.scheduler import CrossoverScheduler

    mode = "bucket" if h.world == 1 or sync_mode == "auto" else sync_mode
    sched = CrossoverScheduler(policy, comm=h.comm, sync_mode=mode, comm_priority=comm_priority,
                               sync_ctas=SYNC_CTAS, barrier=BARRIER,
                               p2p_ctas=P2P_CTAS if p2p_ctas is None else p2p_ctas)
    total = W + 1 + 2 * 8 + K
    static = {}
    regs = []
    for j, a in enumerate(base):
        app = dataclasses.replace(a, iterations=total)
        if host_data:
            workers = [h.rank * a.local_workers + w for w in range(a.local_workers)]
            for w in workers:
                static[(j, w)] = tuple(torch.empty_like(x, device=h.dev) for x in host_data[j](1, w))
            app = dataclasses.replace(app, data=host_data[j],
                                      data_graph=(lambda jj: (lambda t_dev, w: static[(jj, w)]))(j))
        regs.append(app)
        sched.register(app)
    cs, ms = sched.compute_stream, sched.comm_stream
    loss_host = torch.zeros(len(base), dtype=torch.float32).pin_memory()
    for _ in range(W):
        for _j in range(len(base)):
            sched.step()
    # several rotations per graph launch (fewer launches; the e2e path feeds every rotation's
    # batches from the host, so it replays one rotation per launch)
    per = 1 if host_data else next(k for k in (8, 4, 2, 1) if K % k == 0)
    rg = RotationGraph(sched, rotations=per)

    def feed(t):
        if host_data:
            with torch.cuda.stream(cs):
                for (j, w), bufs in static.items():
                    for dst, src in zip(bufs, host_data[j](t, w)):
                        dst.copy_(src, non_blocking=True)

    feed(W + 1)
    rg.begin()
    for _ in range(2):
        feed(rg.t + 1)
        rg.replay()
    K_launches = K // per
    sched.drain()
    h.barrier()
    gc.collect()
    gc.disable()
    clk = Clocks(h.local) if clocks else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(cs)
    for _ in range(K_launches):
        feed(rg.t + 1)
        rg.replay()
        if host_data:   # D2H of every app's loss of this rotation
            with torch.cuda.stream(cs):
                for j, st in enumerate(sched.states):
                    loss_host[j:j + 1].copy_(st.graph_loss.float().view(1), non_blocking=True)
    join = torch.cuda.Event()
    join.record(ms)
    cs.wait_event(join)
    end.record(cs)
    end.synchronize()
    gc.enable()
    clk_info = clk.stop() if clk else None
    ms_total = h.max_over_ranks(start.elapsed_time(end))
    rg.end()
    sched.drain()
    phases = rg.phase_times() if policy.value == "crossover" and not host_data else None
    rg.release()            # before the NCCL communicator goes away (graphs hold NCCL work)
    trace = sched.recorder.resolve()
    out = {"ms": ms_total, "trace": trace, "timed_spans": [], "phases": phases,
           "replicas_identical": replicas_identical(h, regs), "kernels": {},
           "launches": K, "clocks": clk_info, "sched": sched}
    return out


def replicas_identical(h: Harness, base) -> bool | None:
    """Data-parallel replicas must hold bitwise the same weights after every sync: compare a
    hash of every app's parameter bits across the ranks (None at world 1)."""
    if h.world == 1:
        return None
    import hashlib

    import torch

    dig = hashlib.sha256()
    for a in base:
        for p in a.params:
            dig.update(p.detach().contiguous().view(torch.int32).cpu().numpy().tobytes())
    allh = [None] * h.world
    h.dist.all_gather_object(allh, dig.hexdigest())
    return len(set(allh)) == 1


def calibrate_transport(h: Harness, base, sm: str, prio: int = -1):
    """Peer-mapping probe and (sync_mode auto, W > 1) transport calibration before any timed run.

    Collective: if any rank cannot map its peers, every rank falls back to the bucket all-reduce.
    In auto mode the probe is an untimed adaptive crossover run (like cudnn.benchmark) whose
    tuner measures the copy-engine and the P2P-kernel transports (scheduler._TransportTuner);
    the timed crossover arm then runs the chosen one and the sequential arm the full-grid P2P
    kernel.  Returns (crossover mode, sequential mode, tuner summary or None)."""
    from paper_2103_07974_b200.errors import ConfigError
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    global SYNC_CTAS
    grid = None
    if SYNC_CTAS == "auto":
        # measured K1 / K2 grid cap (CrossoverScheduler.calibrate_grid) in an untimed probe; both
        # timed arms then use the chosen cap (same kernels)
        probe = CrossoverScheduler(Policy.CROSSOVER, comm=h.comm, sync_mode=sm if h.world > 1 else "auto",
                                   comm_priority=prio, p2p_ctas=P2P_CTAS, barrier=BARRIER,
                                   record_spans=False, sync_ctas="auto")
        for a in base:
            probe.register(dataclasses.replace(a, iterations=17))
        grid = probe.calibrate_grid(3)
        probe.drain()
        probe.close()
        h.barrier()
        SYNC_CTAS = grid["choice"] if grid else 0
    from paper_2103_07974_b200.nvls import nvls_buffer_of

    if sm == "auto" and base[0].flat_params is not None and nvls_buffer_of(base[0].flat_params) is not None:
        sm = "nvls"
    if h.world < 2 or sm not in ("p2p", "ce", "auto"):
        return sm, sm, ({"grid": grid} if grid else None)
    try:
        sched = CrossoverScheduler(Policy.CROSSOVER, comm=h.comm, sync_mode=sm, comm_priority=prio,
                                   p2p_ctas=P2P_CTAS, barrier=BARRIER, record_spans=False,
                                   sync_ctas=SYNC_CTAS)
        for a in base:
            sched.register(dataclasses.replace(a, iterations=9))
        summary = sched.calibrate(4) if sm == "auto" else None
        while sched.step():
            pass
        sched.drain()
        sched.close()
        h.barrier()
        if summary is not None and summary["active"]:
            return summary["choice"], "p2p", dict(summary, grid=grid)
        return sm, sm, ({"grid": grid} if grid else None)
    except ConfigError as exc:
        if h.rank == 0:
            print(f"{sm} sync unavailable ({exc}); using the bucket all-reduce", file=sys.stderr)
        return "bucket", "bucket", None


def phase_medians(spans, order):
    """Per-job median compute (fwd + bwd) and sync durations in ms."""
    from paper_2103_07974_b200.engine import Phase

    def med(job, phase):
        vals = [s.end - s.start for s in spans if s.job_id == job and s.phase is phase]
        return statistics.median(vals) / 1e6 if vals else 0.0

    comp = [med(j, Phase.FORWARD) + med(j, Phase.BACKWARD) for j in order]
    comm = [med(j, Phase.SYNC) for j in order]
    return comp, comm


def kernel_summary(kern: dict, sync) -> dict:
    out = {}
    if "k2_update" in kern:
        t = statistics.mean(kern["k2_update"])
        kb = sync.k2_bytes("ce" if sync.mode in ("ce", "adaptive") else None)
        out["k2_update"] = {"ms": round(t, 4), "bytes": kb, "GB/s": round(kb / (t / 1e3) / 1e9, 1)}
    if "k1_pack" in kern:
        t = statistics.mean(kern["k1_pack"])
        out["k1_pack"] = {"ms": round(t, 4), "bytes": sync.k1_bytes(),
                          "GB/s": round(sync.k1_bytes() / (t / 1e3) / 1e9, 1)}
    for name in ("c1_reduce_scatter", "c1_all_gather", "c1_ce_reduce_scatter", "c1_ce_all_gather"):
        if name in kern:
            t = statistics.mean(kern[name])
            out[name] = {"ms": round(t, 4), "bus_bytes": sync.c1_bus_bytes() / 2,
                         "busbw_GB/s": round(sync.c1_bus_bytes() / 2 / (t / 1e3) / 1e9, 1)}
    if "c1_unfused" in kern:
        t = statistics.mean(kern["c1_unfused"])
        out["c1_unfused"] = {"ms": round(t, 4), "messages": len(sync.params),
                             "busbw_GB/s": round(sync.c1_bus_bytes() / (t / 1e3) / 1e9, 1)}
    if "k2_p2p_fused" in kern:
        t = statistics.mean(kern["k2_p2p_fused"])
        nv = sync.c1_bus_bytes()
        out["k2_p2p_fused"] = {"ms": round(t, 4), "bytes": sync.k2_bytes("p2p"),
                               "GB/s": round(sync.k2_bytes("p2p") / (t / 1e3) / 1e9, 1),
                               "nvlink_bytes": nv, "nvlink_GB/s": round(nv / (t / 1e3) / 1e9, 1)}
    if "k2_p2p_gather" in kern:
        t = statistics.mean(kern["k2_p2p_gather"])
        nv = sync.c1_bus_bytes()
        out["k2_p2p_gather"] = {"ms": round(t, 4), "bytes": sync.k2_bytes("p2p_gather"),
                                "GB/s": round(sync.k2_bytes("p2p_gather") / (t / 1e3) / 1e9, 1),
                                "nvlink_bytes": nv, "nvlink_GB/s": round(nv / (t / 1e3) / 1e9, 1)}
    if "k2_nvls_fused" in kern:
        t = statistics.mean(kern["k2_nvls_fused"])
        nv = sync.c1_bus_bytes()
        link = sync.nvls_link_bytes()
        out["k2_nvls_fused"] = {"ms": round(t, 4), "bytes": sync.k2_bytes("nvls"),
                                "nvlink_bytes": nv, "nvlink_GB/s": round(nv / (t / 1e3) / 1e9, 1),
                                "link_bytes_per_direction": link,
                                "link_GB/s": round(link / (t / 1e3) / 1e9, 1)}
    if "c1_allreduce" in kern:
        t = statistics.mean(kern["c1_allreduce"])
        out["c1_allreduce"] = {"ms": round(t, 4), "bus_bytes": sync.c1_bus_bytes(),
                               "busbw_GB/s": round(sync.c1_bus_bytes() / (t / 1e3) / 1e9, 1),
                               "peak_GB/s": 900.0}
    return out


class _HostBatches:
    """data(t, worker) -> pinned host copies of the app's device batches (the e2e path copies
    them H2D every step through the scheduler's H2D stream)."""

    def __init__(self, device_data, iterations: int, workers):
        self.b = {(t, w): tuple(x.cpu().pin_memory() for x in device_data(t, w))
                  for t in range(1, iterations + 1) for w in workers}

    def __call__(self, t: int, worker: int):
        return self.b[(t, worker)]


def _graphed_models(args) -> bool:
    """Per-app CUDA graphs for the image models' forward / backward -- not when the whole rotation
    is captured (that graph contains the eager forward / backward itself)."""
    return not args.no_graphs and args.rotation_graph != "on"


def build_apps(args, h):
    """(apps, host-data callables for e2e or None, h2d bytes per step, per-app kernel launches
    per iteration that replay inside CUDA graphs) for the selected workload."""
    import torch

    from paper_2103_07974_b200 import apps

    rank, world, dev = h.rank, h.world, h.dev
    # auto at W >= 4: multicast-bound flat parameters (the nvls transport) when every rank's GPU
    # supports NVSwitch multicast, else IPC flat parameters and the adaptive ce / p2p choice.  Per
    # rank and link direction nvls moves S(1 + 1/W) bytes (the switch reads every member's shard,
    # the local one included, and fans the stores out to every member) against 2S(W-1)/W for the
    # peer-to-peer transports, so it only pays from W = 4 up (W = 2: 1.5S vs S, and the fused sync
    # measured 0.33 vs 0.20 ms, profiles/r02_nvls/c1_w2.json; W = 4: 1.25S vs 1.5S).
    flat = ({"sharded": True, "p2p": "ipc", "p2p_gather": "ipc", "ce": "ipc", "auto": "ipc",
             "nvls": "nvls"}.get(args.sync_mode, False)
            if world > 1 else False)
    if (flat == "ipc" and args.sync_mode == "auto" and args.config != "mlp" and not args.mix
            and not args.scenario and world >= 4):
        from paper_2103_07974_b200.nvls import nvls_available
        from paper_2103_07974_b200.p2p import all_ranks_agree

        if all_ranks_agree(nvls_available(dev)):
            flat = "nvls"
    if args.config == "mlp":
        w = max(2, world)
        local = w // world
        iters = max(args.warmup + args.steps + 24, 17)  # >= calibration / graph-mode prologue
        base = [apps.mlp_app(apps.MlpConfig(dataset_seed=11 + k, workers=w), f"mlp{k}", k, iters, dev,
                             local_workers=local, worker_count=w, flat=flat) for k in range(2)]
        host = None
        h2d = 0
        if not args.no_e2e:
            workers = [rank * local + i for i in range(local)]
            host = [_HostBatches(a.data, iters, workers) for a in base]
            h2d = 2 * local * (64 * 784 * 4 + 64 * 8)
        return base, host, h2d, 0
    if args.scenario:
        # a reference scenario file (colosim JSON) as device apps: profile jobs -> the model,
        # inline jobs -> exact tensor split + calibrated GEMM compute (paper_2103_07974_b200.scenario)
        from paper_2103_07974_b200.scenario import load_config
        sc = load_config(args.scenario)
        base = list(sc.device_plan(dev, 1, batch={"resnet50": args.batch, "vgg16": args.batch},
                                   time_scale=args.scenario_time_scale, workers=world, flat=flat,
                                   graphed=_graphed_models(args), fast_bn=not args.aten_bn,
                                   seed=0, data_seed=1000 * rank).jobs)
        args.mix = f"scenario {sc.name}"
        args.no_e2e, args.no_cpu_baseline = True, True
    elif args.mix:
        base = []
        for j, item in enumerate(args.mix.split(",")):
            name, b = item.split(":")
            if name == "bert":
                base.append(apps.bert_app(f"bert_{j}", int(b), 128, 1, dev, seed=1000 * j,
                                          data_seed=1000 * j + rank, flat=flat))
            else:
                fn = apps.resnet50_app if name == "resnet50" else apps.vgg16_app
                base.append(fn(f"{name}_{j}", int(b), 1, dev, seed=1000 * j, data_seed=1000 * j + rank,
                               graphed=_graphed_models(args), flat=flat, fast_bn=not args.aten_bn,
                               stem="cudnn" if args.cudnn_stem else "gemm"))
        args.no_e2e, args.no_cpu_baseline = True, True
    else:
        from paper_2103_07974_b200.errors import ConfigError

        build = apps.resnet50_app if args.model == "resnet50" else apps.vgg16_app

        def make(fl):
            return [build(f"{args.model}_{j}", args.batch, 1, dev, seed=1000 * j, data_seed=1000 * j + rank,
                          graphed=_graphed_models(args), flat=fl, fast_bn=not args.aten_bn,
                          stem="cudnn" if args.cudnn_stem else "gemm")
                    for j in range(args.jobs)]
        try:
            base = make(flat)
        except ConfigError as exc:            # multicast setup failed on some rank (all agree)
            if flat != "nvls" or args.sync_mode != "auto":
                raise
            if rank == 0:
                print(f"nvls unavailable ({exc}); using IPC flat parameters", file=sys.stderr)
            base = make("ipc")
    host = None if args.no_e2e else [
        apps._CycleData(apps.synthetic_image_batches(args.batch, 2, 7 + 1000 * j + rank, dev,
                                                     host_uint8=True))
        for j in range(args.jobs)]
    h2d = args.jobs * (args.batch * 224 * 224 * 3 + args.batch * 8)
    # NHWC BN kernels: 3 forward + 3 backward launches per BN layer per iteration, 2 per max-pool,
    # one im2col per RGB stem (they replay inside the CUDA graphs, so they are counted from the
    # model structure, not from Python calls)
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d, CrossoverMaxPool2d
    n_bn = sum(sum(1 for m in a.model.modules() if isinstance(m, CrossoverBatchNorm2d)) for a in base)
    n_pool = sum(sum(1 for m in a.model.modules() if isinstance(m, CrossoverMaxPool2d)) for a in base)
    n_stem = 0 if args.cudnn_stem else sum(
        sum(1 for m in a.model.modules() if isinstance(m, torch.nn.Conv2d) and m.in_channels == 3)
        for a in base)
    return base, host, h2d, 6 * n_bn + 2 * n_pool + n_stem


def run_ours(args):
    from paper_2103_07974_b200 import _lib
    from paper_2103_07974_b200.engine import schedule_key, trace_to_chrome_json, validate_trace
    from paper_2103_07974_b200.scheduler import Policy, overlap_roofline, rotation_schedule

    h = Harness(args.nccl_max_ctas)
    rank, world = h.rank, h.world
    global P2P_CTAS, BARRIER, SYNC_CTAS
    if args.p2p_ctas:   # override the scheduler's policy-dependent cap, both arms
        P2P_CTAS = args.p2p_ctas
    if args.p2p_registers or args.reg_shape is not None:
        from paper_2103_07974_b200 import _lib as _cs

        if args.p2p_registers:
            _cs.tune("p2p_bulk", 0)
        if args.reg_shape is not None:
            _cs.tune("reg_shape", args.reg_shape)
    BARRIER = args.barrier
    SYNC_CTAS = args.sync_ctas
    if args.bn_no_pdl:
        _lib.tune("bn_no_pdl", 1)
    if args.side_grads:
        from paper_2103_07974_b200 import bn as _bn
        _bn._SIDE_GRADS = True
    K, W = args.steps, args.warmup
    base, host_data, h2d_bytes, graph_launches = build_apps(args, h)
    samples_per_rot = sum(a.samples_per_batch * a.local_workers for a in base) * world
    unit = unit_of(args)

    prio = -1 if args.comm_priority == "high" else 0
    graph = args.rotation_graph == "on" or (args.rotation_graph == "auto" and args.config == "mlp")
    if graph:
        # whole-rotation CUDA graphs (graphs.RotationGraph), one graph launch per rotation for both
        # arms; every transport is capturable -- `auto` = the NCCL bucket all-reduce (W simulated
        # workers at W = 1)
        sm = sm_seq_best = "bucket" if args.sync_mode == "auto" or world == 1 else args.sync_mode
        tuner = None
        W = max(W, 2)
    else:
        sm, sm_seq_best, tuner = calibrate_transport(h, base, args.sync_mode, prio)
    args.sync_mode = sm
    cross = timed_run(h, base, Policy.CROSSOVER, W, K, clocks=True, sync_mode=sm, comm_priority=prio,
                      graph=graph)
    # the same transport with the same launch caps for the sequential arm: the speedup measures
    # the schedule alone (crossover vs back-to-back, same kernels)
    s0 = cross["sched"].states[0].sync
    p2p_cap = (s0._p2p.max_ctas if hasattr(s0, "_p2p") else
               s0._nvls.max_ctas if hasattr(s0, "_nvls") else None)
    seq = timed_run(h, base, Policy.SEQUENTIAL, W, K, sync_mode=sm, comm_priority=prio,
                    p2p_ctas=p2p_cap, graph=graph)
    # and the fastest back-to-back configuration (full-grid P2P kernel at W > 1)
    seq_best = seq if (sm_seq_best == sm and p2p_cap is None) else timed_run(
        h, base, Policy.SEQUENTIAL, W, K, sync_mode=sm_seq_best, comm_priority=prio, graph=graph)
    e2e = None if args.no_e2e else timed_run(h, base, Policy.CROSSOVER, W, K, host_data=host_data,
                                             time_kernels=False, sync_mode=sm, comm_priority=prio,
                                             graph=graph)

    # the models must still be numerically healthy: a diverged model (NaN weights) changes the
    # kernels' speed and invalidates the measurement
    import torch as _torch
    weights_finite = all(bool(_torch.isfinite(p).all()) for a in base for p in a.params)

    # legality + bit-exact schedule of the measured runs (graph mode: the eager prefix; the replays
    # record no per-phase spans -- their schedule is the captured one, graphs.py)
    order = [a.job_id for a in base]
    for r in (cross, seq, seq_best):
        assert validate_trace(r["trace"]) == [], validate_trace(r["trace"])[:3]
        assert schedule_key(r["trace"]) == rotation_schedule(order, [W if graph else W + K] * len(order))

    hbm_peak, peak_kind = peaks()
    sync0 = cross["sched"].states[0].sync
    sync_seq = seq_best["sched"].states[0].sync
    if graph:
        comp, comm_t = cross["phases"]
        kernels = kernels_isolated = {"sync_graph": {"ms": round(comm_t[0], 4), "bytes": sync0.k2_bytes(),
                                                     "GB/s": round(sync0.k2_bytes() / (comm_t[0] / 1e3) / 1e9, 1)}}
        if world == 1:   # the sync graph is K2 alone (two simulated workers' rows)
            kernels["k2_update"] = kernels["sync_graph"]
        else:            # C1 + K2: report the exchange against NVLink (latency-bound for small buckets)
            nv = sync0.c1_bus_bytes()
            kernels["c1_allreduce"] = {"ms": round(comm_t[0], 4), "bus_bytes": nv,
                                       "busbw_GB/s": round(nv / (comm_t[0] / 1e3) / 1e9, 1),
                                       "peak_GB/s": 900.0, "note": "whole sync graph (C1 + K2)"}
    else:
        comp, comm_t = phase_medians(seq["timed_spans"], order)
        kernels = kernel_summary(cross["kernels"], sync0)
        kernels_isolated = kernel_summary(seq_best["kernels"], sync_seq)
    split = None
    if cross.get("timed_spans"):
        # where the crossover rotation goes (tools/band.py): compute phases measured while the syncs
        # overlap them vs alone, and the GPU lane's busy fraction
        cc, cm = phase_medians(cross["timed_spans"], order)
        split = {"crossover_comp_ms": [round(c, 4) for c in cc], "crossover_comm_ms": [round(c, 4) for c in cm],
                 "comp_inflation": round(sum(cc) / sum(comp), 4) if sum(comp) else None,
                 "gpu_lane_busy_frac": round(sum(cc) / (cross["ms"] / K), 4)}
    roof = overlap_roofline(comp, comm_t)
    rot_cross, rot_seq, rot_best = cross["ms"] / K, seq["ms"] / K, seq_best["ms"] / K
    value = samples_per_rot * K / (cross["ms"] / 1e3)

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            host = host_threads()
            if args.config == "mlp":
                cv, wall = cpu_mlp(2, 200, 5)
                sample = (f"2 MLP jobs x 2 workers (simulated serially) x batch 64, 200 rotations, "
                          f"oracle fp64 numpy ({wall:.2f} s)")
            else:
                rot = 20   # ~10-20 s of host work on the pool's boxes
                cv, _, wall = cpu_crossover(args.model, args.jobs, args.cpu_batch, rot, 1)
                sample = (f"{args.jobs} x {args.model}, batch {args.cpu_batch}/job per rotation (bounded "
                          f"sample of batch {args.batch}), {rot} rotations after 1 warm-up, torch-CPU "
                          f"fwd/bwd + oracle rotation / fusion / average / SGD-momentum ({wall:.1f} s)")
            cpu = {"value": round(cv, 3), "unit": unit, "cores": host["cores"], "kind": "port",
                   "sample": sample, "threads": host, "reference_paths": reference_paths()}
        e2e_line = None
        if e2e is not None:
            ev = samples_per_rot * K / (e2e["ms"] / 1e3)
            e2e_line = {"value": round(ev, 2), "unit": unit, "h2d_bytes_per_step": h2d_bytes * world,
                        "d2h_bytes_per_step": len(base) * 4 * world,
                        "per_rank": {"h2d_bytes": h2d_bytes, "d2h_bytes": len(base) * 4}}
        impl = {"rotation_graph": graph,
                "precision": ("fp32" if args.config == "mlp" else "bf16 autocast, fp32 params / grads / update"),
                "sync_mode": (sync0.mode if sync0.mode == sync_seq.mode else
                              {"crossover": sync0.mode, "sequential_best": sync_seq.mode}),
                "rank_barrier": sync0.barrier_kind, "k1_k2_grid_cap": sync0.sync_ctas or "one CTA per chunk"}
        if args.config != "mlp":
            impl["model_compute"] = (("fwd/bwd as CUDA graphs" if not args.no_graphs else "eager fwd/bwd")
                                     + ("" if args.aten_bn else ", NHWC BN(+ReLU/+residual) and max-pool kernels")
                                     + ("" if args.cudnn_stem else ", RGB stem as im2col + GEMMs"))
        if args.mix:
            impl["mix"] = args.mix
        impl["p2p_capped_variant"] = "registers" if args.p2p_registers else "cp.async.bulk (TMA) tiles"
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": unit, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": round(rot_cross, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.config == "mlp" else "bf16",
            "data": ("synthetic (seeded N(0,1) dataset, reference batch-index seeding)" if args.config == "mlp"
                     else "synthetic (random-init weights, N(0,1) images / random labels)"),
            "config": workload_config(args, world),
            "impl_config": impl,
            "transport_tuner": tuner,
            "weights_finite": weights_finite,
            "replicas_identical": cross["replicas_identical"],
            "speedup_vs_sequential": round(rot_seq / rot_cross, 4),
            "sequential": {"value": round(samples_per_rot * K / (seq["ms"] / 1e3), 2),
                           "ms_per_step": round(rot_seq, 3), "sync_mode": seq["sched"].states[0].sync.mode,
                           "note": "same transport and launch caps as the crossover arm"},
            "speedup_vs_best_sequential": round(rot_best / rot_cross, 4),
            "sequential_best": {"value": round(samples_per_rot * K / (seq_best["ms"] / 1e3), 2),
                                "ms_per_step": round(rot_best, 3), "sync_mode": sync_seq.mode},
            "rho": round(sum(comm_t) / sum(comp), 5) if sum(comp) else None,
            "predicted_speedup": (round((sum(comp) + sum(comm_t)) / max(sum(comp), sum(comm_t)), 4)
                                  if sum(comp) else None),
            "overlap_roofline": {"per_rotation_ms": {k: round(v, 4) for k, v in roof.items()},
                                 "measured_ms": round(rot_cross, 4),
                                 "frac": round(roof["north_star"] / rot_cross, 4),
                                 "frac_tight": round(roof["tight"] / rot_cross, 4),
                                 "comp_ms": [round(c, 4) for c in comp],
                                 "comm_ms": [round(c, 4) for c in comm_t],
                                 "crossover_split": split},
            "roofline": roofline_line(kernels, sync0, hbm_peak, peak_kind,
                                      "mlp" if args.config == "mlp" else args.model,
                                      kernels_isolated, sync_seq),
            "kernels": kernels,
            "kernels_isolated": kernels_isolated,
            "gpu_launches": (2 * len(base) * K if graph else cross["launches"]) + graph_launches * K,
            "gpu_launches_breakdown": {"k1_k2_p2p": cross["launches"],
                                       "bn_and_pool_kernels": graph_launches * K},
            "clocks": cross["clocks"],
            "e2e": e2e_line,
            "cpu_baseline": cpu,
        }
        if args.trace_out:
            Path(args.trace_out).write_text(trace_to_chrome_json(cross["trace"]))
            Path(args.trace_out).with_suffix(".spans.json").write_text(json.dumps(
                [[s.lane_id, s.job_id, s.phase.value, s.iteration, s.start, s.end]
                 for s in cross["trace"].spans]))
        if args.metrics_out:
            # the reference's own measure / compare / report (metrics.py:62-200) on measured traces
            from paper_2103_07974_b200.metrics import compare, measure, report
            from paper_2103_07974_b200.scheduler import SchedulePlan

            mx = measure(cross["trace"], SchedulePlan(Policy.CROSSOVER, base), "bench")
            ms_ = measure(seq["trace"], SchedulePlan(Policy.SEQUENTIAL, base), "bench")
            c = compare(mx, ms_)
            Path(args.metrics_out).write_text(report(c, "json"))
            Path(args.metrics_out).with_suffix(".csv").write_text(report(c, "csv") + report(ms_, "csv"))
    h.close()
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
