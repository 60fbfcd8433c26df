"""Multi-rank parity check of the NCCL path (launched by tests/test_gpu_multirank.py).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/mp_crossover_check.py OUT.json

Each rank is one data-parallel worker (worker index = rank, ≙ equivalence.py:131):
K1 packs its gradients, NCCL sums the bucket over NVLink, K2 divides by W and
updates.  Rank 0 checks (a) per-iteration weights vs the reference golden /
oracle within the fp32 tolerance, (b) at W = 2 bitwise equality with the
single-GPU run that reduces W simulated workers left to right (two-operand
IEEE addition is commutative), (c) the bit-exact schedule and trace legality.
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import sgd as osgd  # noqa: E402
from paper_2103_07974_b200.apps import (LossKind, MlpConfig, SgdConfig, linear_app,  # noqa: E402
                                        mlp_app)
from paper_2103_07974_b200.comm import NcclCommunicator  # noqa: E402
from paper_2103_07974_b200.engine import schedule_key, validate_trace  # noqa: E402
from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy, rotation_schedule  # noqa: E402


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = NcclCommunicator(rank, world)
    res = {"world": world, "ok": True, "checks": []}

    # (1) MLP config 1 over real ranks
    T = 8
    specs = [(11, 0), (12, 1)]
    s = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True)
    for k, (ds, rs) in enumerate(specs):
        s.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world), f"mlp{k}", rs, T, dev,
                           local_workers=1, worker_count=world))
    tr = s.run()
    w_ranks = [s.weights(f"mlp{k}").cpu() for k in range(2)]
    legal = validate_trace(tr) == [] and schedule_key(tr) == rotation_schedule(["mlp0", "mlp1"], [T, T])
    res["checks"].append({"name": "mlp_trace_legal_and_schedule_exact", "ok": legal})

    # (2) linear reference problem (W = world workers) -> compared with the oracle on rank 0
    lcfg = [SgdConfig(0.05, world, LossKind.LEAST_SQUARES, 123), SgdConfig(0.05, world, LossKind.LOGISTIC, 124)]
    s2 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True)
    for k, c in enumerate(lcfg):
        s2.register(linear_app(c, f"lin{k}", 40 + k, 20, dev, local_workers=1))
    s2.run()
    lin = [s2.weights(f"lin{k}")[:, :8].cpu().numpy().astype(np.float64) for k in range(2)]

    # (3) sharded sync (reduce-scatter -> shard K2 -> all-gather into flat params) vs the
    #     all-reduce bucket path, both with momentum: bitwise at W = 2, tolerance otherwise
    mom_w = {}
    for mode, flat in (("bucket", False), ("sharded", True)):
        s4 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode=mode)
        for k, (ds, rs) in enumerate(specs):
            s4.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T,
                                dev, local_workers=1, worker_count=world, flat=flat))
        s4.run()
        mom_w[mode] = [s4.weights(f"m{k}").cpu() for k in range(2)]
        if mode == "sharded":
            res["checks"].append({"name": "sharded_mode_used",
                                  "ok": all(st.sync.mode == "sharded" for st in s4.states)})
    n = mom_w["bucket"][0].shape[1]
    if world == 2:
        same = all(torch.equal(mom_w["bucket"][k], mom_w["sharded"][k][:, :n]) for k in range(2))
        res["checks"].append({"name": "sharded_bitwise_eq_allreduce_w2", "ok": bool(same)})
    # (3a) per-tensor (unfused) all-reduces == fused bucket at W = 2 (same two-operand sums)
    s8 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode="unfused")
    for k, (ds, rs) in enumerate(specs):
        s8.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T,
                            dev, local_workers=1, worker_count=world))
    s8.run()
    unf_w = [s8.weights(f"m{k}").cpu() for k in range(2)]
    res["checks"].append({"name": "unfused_mode_used", "ok": all(st.sync.mode == "unfused" for st in s8.states)})
    if world == 2:
        same = all(torch.equal(mom_w["bucket"][k], unf_w[k]) for k in range(2))
        res["checks"].append({"name": "unfused_bitwise_eq_fused_w2", "ok": bool(same)})

    # (MLP trajectories are compared bitwise only: a ReLU whose pre-activation sits within an
    #  ulp of zero flips with the reduction order, so ReLU nets are chaotic at the ulp level.
    #  Tolerance checks of every mode use the smooth linear problems below.)

    # (3b) momentum on the reference's linear problems, every sync mode vs the fp64 oracle
    Tl = 20
    lin_m = {}
    for mode, flat in (("bucket", False), ("sharded", True), ("p2p", "ipc"), ("ce", "ipc"),
                       ("unfused", False)):
        s7 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode=mode)
        for k, c in enumerate(lcfg):
            s7.register(linear_app(c, f"lm{k}", 40 + k, Tl, dev, local_workers=1, momentum=0.9, flat=flat))
        s7.run()
        lin_m[mode] = [s7.weights(f"lm{k}")[:, :8].cpu().numpy().astype(np.float64) for k in range(2)]
        s7.close()

    # (4) collective-fused P2P sync (one kernel: NVLink reads of every rank's bucket shard in
    #     rank order, / W, SGD-momentum, NVLink writes of the new shard to every rank)
    s5 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode="p2p")
    for k, (ds, rs) in enumerate(specs):
        s5.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T,
                            dev, local_workers=1, worker_count=world, flat="ipc"))
    s5.run()
    p2p_w = [s5.weights(f"m{k}").cpu() for k in range(2)]
    s5.close()
    res["checks"].append({"name": "p2p_mode_used", "ok": all(st.sync.mode == "p2p" for st in s5.states)})
    if world == 2:
        same = all(torch.equal(mom_w["bucket"][k], p2p_w[k][:, :n]) for k in range(2))
        res["checks"].append({"name": "p2p_bitwise_eq_allreduce_w2", "ok": bool(same)})

    # (4b) copy-engine sync: CE pulls + K2 over the W shard copies in rank order -- the same
    #      arithmetic as the P2P kernel, so bitwise equal to it at any W
    s8 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode="ce")
    for k, (ds, rs) in enumerate(specs):
        s8.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T,
                            dev, local_workers=1, worker_count=world, flat="ipc"))
    s8.run()
    ce_w = [s8.weights(f"m{k}").cpu() for k in range(2)]
    s8.close()
    res["checks"].append({"name": "ce_mode_used", "ok": all(st.sync.mode == "ce" for st in s8.states)})
    res["checks"].append({"name": "sm_free_flag_barrier_used",
                          "ok": all(st.sync.barrier_kind == "flags" for st in s8.states)})
    res["checks"].append({"name": f"ce_bitwise_eq_p2p_w{world}",
                          "ok": all(torch.equal(ce_w[k], p2p_w[k]) for k in range(2))})

    # (4b') the same ce run with the NCCL 1-element all-reduce barriers instead of the flags
    s10 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode="ce",
                             barrier="nccl")
    for k, (ds, rs) in enumerate(specs):
        s10.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T,
                             dev, local_workers=1, worker_count=world, flat="ipc"))
    s10.run()
    ce_nccl_w = [s10.weights(f"m{k}").cpu() for k in range(2)]
    kinds = {st.sync.barrier_kind for st in s10.states}
    s10.close()
    res["checks"].append({"name": "ce_nccl_barrier_bitwise_eq_flags",
                          "ok": kinds == {"nccl"} and all(torch.equal(ce_nccl_w[k], ce_w[k]) for k in range(2))})

    # (4c) auto under crossover with IPC flat parameters = adaptive transport: copy engines for
    #      two rotations, the P2P kernel for two, then the measured faster one; the choice is the
    #      same on every rank and the weights stay bitwise equal to either transport
    s9 = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True)
    for k, (ds, rs) in enumerate(specs):
        s9.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs,
                            max(T, 14), dev, local_workers=1, worker_count=world, flat="ipc"))
    s9.run()
    ad_w = [s9.weights(f"m{k}").cpu() for k in range(2)]
    summ = s9.tuner.summary() if s9.tuner is not None else None
    s9.close()
    choices = [None] * world
    dist.all_gather_object(choices, summ["choice"] if summ else None)
    res["checks"].append({"name": "adaptive_tuner_decided", "ok": bool(summ and summ["active"]
                          and summ["calibration_period_ms"] is not None), "summary": summ})
    res["checks"].append({"name": "adaptive_choice_same_on_every_rank",
                          "ok": len(set(choices)) == 1 and choices[0] in ("ce", "p2p")})
    res["checks"].append({"name": f"adaptive_bitwise_eq_p2p_w{world}",
                          "ok": all(torch.equal(ad_w[k][:T], p2p_w[k]) for k in range(2))})

    # every rank must hold identical weights after every iteration
    for k in range(2):
        gathered = [torch.empty_like(w_ranks[k]) for _ in range(world)] if rank == 0 else None
        dist.gather(w_ranks[k], gathered, dst=0)
        if rank == 0:
            same = all(torch.equal(gathered[0], x) for x in gathered)
            res["checks"].append({"name": f"ranks_identical_mlp{k}", "ok": bool(same)})

    if rank == 0:
        ref = osgd.run_mlp_crossover(specs, T, workers=world)
        from paper_2103_07974_b200.workload import BucketLayout

        lay = BucketLayout.build([256 * 784, 256, 10 * 256, 10], 32)
        worst = 0.0
        for k in range(2):
            w = w_ranks[k].numpy().astype(np.float64)
            for t in range(T):
                for i, o in enumerate(lay.offsets):
                    r = ref[k][t][i].reshape(-1)
                    worst = max(worst, float(np.max(np.abs(w[t, o:o + r.size] - r) / (1e-5 + 1e-4 * np.abs(r)))))
        res["checks"].append({"name": "mlp_vs_oracle", "ok": worst <= 1.0, "worst_ratio": worst})

        jobs = [osgd.LinearJob(0.05, world, c.loss.value, c.dataset_seed, 40 + k) for k, c in enumerate(lcfg)]
        lref = osgd.run_crossover(jobs, 20)
        lw = 0.0
        for k in range(2):
            r = np.stack(lref[k])
            lw = max(lw, float(np.max(np.abs(lin[k] - r) / (1e-5 + 1e-4 * np.abs(r)))))
        res["checks"].append({"name": "linear_vs_oracle", "ok": lw <= 1.0, "worst_ratio": lw})

        # the P2P path sums in rank order 0..W-1 exactly like K2 over W simulated workers
        # on one GPU (and like the reference's average_gradients): bitwise for ANY W
        s6 = CrossoverScheduler(Policy.CROSSOVER, record_weights=True)
        for k, (ds, rs) in enumerate(specs):
            s6.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev))
        s6.run()
        same = all(torch.equal(s6.weights(f"m{k}").cpu(), p2p_w[k][:, :n]) for k in range(2))
        res["checks"].append({"name": f"p2p_w{world}_bitwise_eq_simulated_w{world}", "ok": bool(same)})

        ljobs = [osgd.LinearJob(0.05, world, c.loss.value, c.dataset_seed, 40 + k) for k, c in enumerate(lcfg)]
        lref_m = [np.stack(osgd.run_isolated_momentum(j, Tl, 0.9)) for j in ljobs]
        for mode, ws in lin_m.items():
            wr = max(float(np.max(np.abs(ws[k] - lref_m[k]) / (1e-5 + 1e-4 * np.abs(lref_m[k]))))
                     for k in range(2))
            res["checks"].append({"name": f"momentum_{mode}_vs_oracle", "ok": wr <= 1.0, "worst_ratio": wr})

        if world == 2:
            # single-GPU run with 2 simulated workers, reduced left to right by K2
            s3 = CrossoverScheduler(Policy.CROSSOVER, record_weights=True)
            for k, (ds, rs) in enumerate(specs):
                s3.register(mlp_app(MlpConfig(dataset_seed=ds, workers=2), f"mlp{k}", rs, T, dev))
            s3.run()
            same = all(torch.equal(s3.weights(f"mlp{k}").cpu(), w_ranks[k]) for k in range(2))
            res["checks"].append({"name": "nccl_w2_bitwise_eq_simulated_w2", "ok": bool(same)})
        res["ok"] = all(c["ok"] for c in res["checks"])
        Path(out_path).write_text(json.dumps(res, indent=1))
        print("MPCHECK " + json.dumps(res), flush=True)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not res["ok"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
