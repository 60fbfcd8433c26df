"""Config 4: comm/comp ratio sweep -- synthetic bucket S (1 MB .. 1 GB) vs a fixed GEMM compute.

    torchrun --nproc-per-node N tools/sweep.py [--sizes-mb 1,4,16,64,256,1024] [--out f.json]

For every S: two co-located synthetic jobs, crossover and sequential with the same kernels,
measured rho = sync / compute (sequential medians), speedup = T_seq / T_cross, the reference's
closed form (1 + rho) / max(1, rho) (scheduler.py:251-258) and the overlap-roofline fraction.
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import Harness, calibrate_transport, kernel_summary, phase_medians, timed_run  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--gemm-reps", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--sync-mode", default="auto", choices=["auto", "bucket", "sharded", "p2p", "ce", "unfused"])
    ap.add_argument("--p2p-ctas", type=int, default=0)
    ap.add_argument("--nccl-max-ctas", type=int, default=0)
    ap.add_argument("--barrier", default="auto", choices=["auto", "flags", "nccl"])
    args = ap.parse_args()
    from paper_2103_07974_b200.apps import synthetic_app
    from paper_2103_07974_b200.scheduler import Policy, overlap_roofline

    h = Harness(args.nccl_max_ctas)
    import bench
    bench.BARRIER = args.barrier
    if args.p2p_ctas:
        import bench
        bench.P2P_CTAS = args.p2p_ctas
    rows = []
    for mb in [int(x) for x in args.sizes_mb.split(",")]:
        flat = ({"sharded": True, "p2p": "ipc", "ce": "ipc", "auto": "ipc"}.get(args.sync_mode, False)
                if h.world > 1 else False)
        base = [synthetic_app(f"syn{j}", mb * 2**20, 1, h.dev, gemm_reps=args.gemm_reps, seed=j,
                              flat=flat) for j in range(2)]
        sm, sm_seq, tuner = calibrate_transport(h, base, args.sync_mode)
        cross = timed_run(h, base, Policy.CROSSOVER, args.warmup, args.steps, sync_mode=sm)
        seq = timed_run(h, base, Policy.SEQUENTIAL, args.warmup, args.steps, sync_mode=sm_seq)
        comp, comm = phase_medians(seq["timed_spans"], [a.job_id for a in base])
        rho = sum(comm) / sum(comp)
        roof = overlap_roofline(comp, comm)
        rot_x, rot_s = cross["ms"] / args.steps, seq["ms"] / args.steps
        row = {"bucket_MB": mb, "world": h.world, "sync_mode": cross["sched"].states[0].sync.mode,
               "sync_mode_sequential": seq["sched"].states[0].sync.mode,
               "rank_barrier": cross["sched"].states[0].sync.barrier_kind,
               "transport_tuner": tuner,
               "p2p_ctas": args.p2p_ctas, "nccl_max_ctas": args.nccl_max_ctas,
               "rho": round(rho, 4),
               "speedup": round(rot_s / rot_x, 4),
               "predicted": round((1 + rho) / max(1.0, rho), 4),
               "rotation_ms": {"crossover": round(rot_x, 4), "sequential": round(rot_s, 4)},
               "overlap_roofline_frac": round(roof["north_star"] / rot_x, 4),
               "overlap_roofline_frac_tight": round(roof["tight"] / rot_x, 4),
               "comp_ms": round(comp[0], 4), "comm_ms": round(comm[0], 4),
               "kernels_isolated": kernel_summary(seq["kernels"], seq["sched"].states[0].sync),
               "kernels_overlapped": kernel_summary(cross["kernels"], cross["sched"].states[0].sync)}
        rows.append(row)
        if h.rank == 0:
            print(json.dumps(row), flush=True)
        del base, cross, seq
        import torch
        torch.cuda.empty_cache()
    if h.rank == 0 and args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))
    h.close()


if __name__ == "__main__":
    main()
