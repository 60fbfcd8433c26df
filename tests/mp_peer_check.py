"""W > 1 data plane of the peer-memory transports, W processes on ONE GPU (no NCCL).

    python -m torch.distributed.run --nproc-per-node W --master-addr 127.0.0.1 \
        --master-port P tests/mp_peer_check.py OUT.json CASE

Launched by tests/test_gpu_peer_transports.py.  Every rank is one data-parallel worker (worker
index = rank, as equivalence.py:131) with its own CUDA context on cuda:0; the ranks see each other
through CUDA IPC (buckets, flat parameters) and the shared host flag segment of the SM-free barrier
-- exactly the code path of W GPUs over NVLink, only the bytes stay in one HBM.  torch.distributed
(gloo) carries the one-off handle exchange and the result gather; the data plane has no collective
library in it.

CASE parity   golden linear jobs (reference fp64 trajectories, equivalence.py:150-232) through
              p2p / ce: within 1e-5 + 1e-4|w| of the reference and bitwise equal to the
              single-process run that reduces W simulated workers left to right; momentum
              trajectories (MLP 784-256-10 and linear) bitwise across p2p / ce / adaptive and
              vs the simulated workers, linear momentum vs the fp64 oracle; ranks identical.
CASE fail     rank 1 stops issuing work after two slots; rank 0's watchdog must raise
              DeadlockError(job, iteration) and its device must drain (no stream stays blocked
              in a flag-barrier wait), all within seconds.
CASE graph    whole-rotation CUDA graphs over ce and p2p (captured flag barriers, CE memcpy nodes,
              the P2P kernel): final weights bitwise equal to the eager run.
CASE resnet   two ResNet-50 apps (bf16 autocast, CUDA graphs, momentum 0.9, weight decay 1e-4)
              through ce for 3 iterations: every rank's update equals torch.optim.SGD
              (foreach=False) on the CPU applied to the rank-order average of the W ranks'
              captured gradients, bit for bit.
CASE gather_mlp  p2p_gather at W = 2 / 4 / 8 on two CUDA-graphed MLPs: bitwise equal to p2p.
CASE gather   the same with the K1-free p2p_gather transport (the kernel reads every rank's
              graph-static gradient tensors in place): bitwise vs torch.optim.SGD, one kernel
              launch per sync.
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import sgd as osgd  # noqa: E402
from paper_2103_07974_b200.apps import (LossKind, MlpConfig, SgdConfig, linear_app,  # noqa: E402
                                        mlp_app)
from paper_2103_07974_b200.comm import PeerGroup  # noqa: E402
from paper_2103_07974_b200.engine import schedule_key, validate_trace  # noqa: E402
from paper_2103_07974_b200.errors import DeadlockError  # noqa: E402
from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy, rotation_schedule  # noqa: E402

ATOL, RTOL = 1e-5, 1e-4


def _gather_equal(t: torch.Tensor, rank: int, world: int) -> bool:
    """True on every rank iff every rank holds bitwise the same tensor."""
    objs = [None] * world
    dist.all_gather_object(objs, t.cpu().numpy().tobytes())
    return all(o == objs[0] for o in objs)


def _run(apps, comm, mode, policy=Policy.CROSSOVER):
    s = CrossoverScheduler(policy, comm=comm, record_weights=True, sync_mode=mode)
    for a in apps:
        s.register(a)
    tr = s.run()
    w = [s.weights(a.job_id).cpu().clone() for a in apps]
    modes = {st.sync.mode for st in s.states}
    barriers = {st.sync.barrier_kind for st in s.states}
    summ = s.tuner.summary() if s.tuner is not None else None
    s.close()
    return w, tr, modes, barriers, summ


def case_parity(rank, world, dev, comm, res):
    golden_meta = json.loads((ROOT / "tests" / "golden" / "equivalence_meta.json").read_text())
    golden = dict(np.load(ROOT / "tests" / "golden" / "equivalence.npz"))
    worst = 0.0
    for m in golden_meta:
        if "perturb" in m or any(c["workers"] != world for c in m["configs"]):
            continue
        cfgs = [SgdConfig(c["learning_rate"], c["workers"], LossKind(c["loss"]), c["dataset_seed"])
                for c in m["configs"]]
        T, seeds = m["iterations"], m["rng_seeds"]
        ids = [f"job{j}" for j in range(len(cfgs))]
        per_mode = {}
        for mode in ("p2p", "ce"):
            apps = [linear_app(c, ids[j], seeds[j], T, dev, local_workers=1, flat="ipc")
                    for j, c in enumerate(cfgs)]
            w, tr, modes, barriers, _ = _run(apps, comm, mode)
            per_mode[mode] = [x[:, :8].numpy() for x in w]
            res["checks"].append({"name": f"{m['key']}_{mode}_mode_and_flags",
                                  "ok": modes == {mode} and barriers == {"flags"}})
            res["checks"].append({"name": f"{m['key']}_{mode}_schedule_exact_trace_legal",
                                  "ok": validate_trace(tr) == [] and
                                  schedule_key(tr) == rotation_schedule(ids, [T] * len(ids))})
            got = np.stack(per_mode[mode]).astype(np.float64)
            ratio = float((np.abs(got - golden[m["key"]]) / (ATOL + RTOL * np.abs(golden[m["key"]]))).max())
            worst = max(worst, ratio)
            res["checks"].append({"name": f"{m['key']}_{mode}_vs_reference_golden", "ok": ratio <= 1.0,
                                  "worst_ratio": ratio})
            res["checks"].append({"name": f"{m['key']}_{mode}_ranks_identical",
                                  "ok": _gather_equal(torch.as_tensor(got), rank, world)})
        res["checks"].append({"name": f"{m['key']}_ce_bitwise_eq_p2p",
                              "ok": all(np.array_equal(a.view(np.int32), b.view(np.int32))
                                        for a, b in zip(per_mode["ce"], per_mode["p2p"]))})
        if rank == 0:
            # the same jobs in ONE process, K2 reducing W simulated workers' bucket rows left to
            # right (the reference's average_gradients order): bitwise equal to the W real ranks
            from paper_2103_07974_b200 import equivalence as deq

            sim = deq.run_crossover(cfgs, T, seeds)
            same = all(np.array_equal(np.stack([st.parameters for st in sim[j]]).view(np.int32),
                                      per_mode["p2p"][j].view(np.int32)) for j in range(len(cfgs)))
            res["checks"].append({"name": f"{m['key']}_p2p_bitwise_eq_simulated_w{world}", "ok": same})
        dist.barrier()
    res["golden_worst_ratio"] = worst

    # momentum: MLP 784-256-10 (config 1) and the linear problems, every peer transport
    T = 8
    specs = [(11, 0), (12, 1)]
    mlp_w = {}
    for mode in ("p2p", "ce"):
        apps = [mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev,
                        local_workers=1, worker_count=world, flat="ipc") for k, (ds, rs) in enumerate(specs)]
        mlp_w[mode], _, modes, _, _ = _run(apps, comm, mode)
        res["checks"].append({"name": f"mlp_momentum_{mode}_mode", "ok": modes == {mode}})
    res["checks"].append({"name": "mlp_momentum_ce_bitwise_eq_p2p",
                          "ok": all(torch.equal(a, b) for a, b in zip(mlp_w["ce"], mlp_w["p2p"]))})
    # L4 at W ranks: the schedule adds no staleness -- sequential == crossover, bit for bit
    apps = [mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev,
                    local_workers=1, worker_count=world, flat="ipc") for k, (ds, rs) in enumerate(specs)]
    seq_w, _, _, _, _ = _run(apps, comm, "ce", policy=Policy.SEQUENTIAL)
    res["checks"].append({"name": "mlp_momentum_ce_sequential_bitwise_eq_crossover",
                          "ok": all(torch.equal(a, b) for a, b in zip(seq_w, mlp_w["ce"]))})
    res["checks"].append({"name": "mlp_momentum_ranks_identical",
                          "ok": _gather_equal(torch.cat([x.reshape(-1) for x in mlp_w["ce"]]), rank, world)})
    # adaptive: calibrate() measures both transports on real iterations, every rank keeps the same one
    Ta = 14
    apps = [mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, Ta, dev,
                    local_workers=1, worker_count=world, flat="ipc") for k, (ds, rs) in enumerate(specs)]
    ad_w, _, modes, _, summ = _run(apps, comm, "auto")
    choices = [None] * world
    dist.all_gather_object(choices, summ["choice"] if summ else None)
    res["checks"].append({"name": "adaptive_calibrated_same_choice_every_rank",
                          "ok": modes == {"adaptive"} and bool(summ and summ["active"]) and
                          len(set(choices)) == 1, "summary": summ})
    res["checks"].append({"name": "adaptive_bitwise_eq_p2p",
                          "ok": all(torch.equal(a[:T], b) for a, b in zip(ad_w, mlp_w["p2p"]))})
    if rank == 0:
        s = CrossoverScheduler(Policy.CROSSOVER, record_weights=True)
        for k, (ds, rs) in enumerate(specs):
            s.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev))
        s.run()
        n = s.weights("m0").shape[1]
        same = all(torch.equal(s.weights(f"m{k}").cpu(), mlp_w["p2p"][k][:, :n]) for k in range(2))
        res["checks"].append({"name": f"mlp_momentum_p2p_bitwise_eq_simulated_w{world}", "ok": same})
    dist.barrier()

    lcfg = [SgdConfig(0.05, world, LossKind.LEAST_SQUARES, 123), SgdConfig(0.05, world, LossKind.LOGISTIC, 124)]
    Tl = 20
    for mode in ("p2p", "ce"):
        apps = [linear_app(c, f"lm{k}", 40 + k, Tl, dev, local_workers=1, momentum=0.9, flat="ipc")
                for k, c in enumerate(lcfg)]
        w, _, _, _, _ = _run(apps, comm, mode)
        jobs = [osgd.LinearJob(0.05, world, c.loss.value, c.dataset_seed, 40 + k) for k, c in enumerate(lcfg)]
        ref = [np.stack(osgd.run_isolated_momentum(j, Tl, 0.9)) for j in jobs]
        wr = max(float(np.max(np.abs(w[k][:, :8].numpy().astype(np.float64) - ref[k]) /
                              (ATOL + RTOL * np.abs(ref[k])))) for k in range(2))
        res["checks"].append({"name": f"linear_momentum_{mode}_vs_fp64_oracle", "ok": wr <= 1.0,
                              "worst_ratio": wr})


def case_fail(rank, world, dev, comm, res):
    T = 10
    specs = [(11, 0), (12, 1)]
    s = CrossoverScheduler(Policy.CROSSOVER, comm=comm, sync_mode="ce", watchdog_s=5.0)
    for k, (ds, rs) in enumerate(specs):
        s.register(mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev,
                           local_workers=1, worker_count=world, flat="ipc"))
    if rank == 1:
        for _ in range(2):
            s.step()                     # then this rank stops issuing work (stays alive)
        torch.cuda.synchronize()         # its queued syncs complete: rank 0 is ahead of it
        dist.barrier()                   # until rank 0 has finished its checks
        return
    t0 = time.monotonic()
    while s.step():
        pass
    raised = None
    try:
        s.drain()
    except DeadlockError as exc:
        raised = exc
    t_raise = time.monotonic() - t0
    t1 = time.monotonic()
    torch.cuda.synchronize()             # would hang forever if a flag wait were still pending
    t_sync = time.monotonic() - t1
    res["checks"].append({"name": "deadlock_error_raised", "ok": raised is not None,
                          "error": str(raised) if raised else None})
    res["checks"].append({"name": "deadlock_names_oldest_pending_sync",
                          "ok": raised is not None and raised.job_id == "m0" and raised.iteration == 2,
                          "job": getattr(raised, "job_id", None), "iteration": getattr(raised, "iteration", None)})
    res["checks"].append({"name": "device_drained_after_release", "ok": t_sync < 10.0,
                          "raise_s": round(t_raise, 2), "sync_s": round(t_sync, 3)})
    res["checks"].append({"name": "scheduler_marked_failed",
                          "ok": s.failed and all(st.sync.failed for st in s.states)})
    dist.barrier()


def case_graph(rank, world, dev, comm, res):
    """Whole-rotation CUDA graphs over the peer transports: the flag barriers (constant-valued,
    self-resetting stream memory operations), the copy-engine pulls and the P2P kernel captured
    once and replayed; final weights bitwise equal to the eager run of the same transport."""
    from paper_2103_07974_b200.graphs import RotationGraph

    T = 12
    specs = [(11, 0), (12, 1)]
    for mode in ("ce", "p2p"):
        finals = {}
        for graph in (False, True):
            apps = [mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"g{k}", rs, T, dev,
                            local_workers=1, worker_count=world, flat="ipc") for k, (ds, rs) in enumerate(specs)]
            s = CrossoverScheduler(Policy.CROSSOVER, comm=comm, sync_mode=mode)
            for a in apps:
                s.register(a)
            if graph:
                for _ in range(2 * len(apps)):
                    s.step()
                rg = RotationGraph(s)
                rg.begin()
                while rg.t < T:
                    rg.replay()
                rg.end()
                s.drain()
                rg.release()
            else:
                s.run()
            finals[graph] = [torch.cat([p.detach().reshape(-1) for p in a.params]).cpu() for a in apps]
            s.close()
        same = all(torch.equal(a.view(torch.int32), b.view(torch.int32))
                   for a, b in zip(finals[False], finals[True]))
        res["checks"].append({"name": f"graph_{mode}_bitwise_eq_eager_w{world}", "ok": same})
        res["checks"].append({"name": f"graph_{mode}_ranks_identical",
                              "ok": _gather_equal(torch.cat(finals[True]), rank, world)})


def case_resnet(rank, world, dev, comm, res):
    """Config-2 update path at W ranks: 161 tensors, channels_last conv weights, CUDA-graph static
    gradients, IPC flat parameters, copy-engine transport; bitwise vs torch.optim.SGD."""
    _resnet_update_check(rank, world, dev, comm, res, "ce")


def case_gather(rank, world, dev, comm, res):
    """The K1-free p2p_gather transport (every rank's graph-static gradient tensors read in place
    over NVLink / IPC) on the same check: bitwise vs torch.optim.SGD, one kernel per sync."""
    _resnet_update_check(rank, world, dev, comm, res, "p2p_gather")


def case_gather_mlp(rank, world, dev, comm, res):
    """p2p_gather at any W on a cheap model: two CUDA-graphed MLP 784-256-10 apps (momentum),
    per-iteration weights bitwise equal to the p2p transport on the same graphed apps and to p2p on
    the eager apps, ranks identical, one kernel per sync."""
    T = 6
    specs = [(11, 0), (12, 1)]
    out = {}
    for mode, graphed in (("p2p_gather", True), ("p2p", True), ("p2p", False)):
        apps = [mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev,
                        local_workers=1, worker_count=world, flat="ipc", graphed=graphed)
                for k, (ds, rs) in enumerate(specs)]
        s = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode=mode)
        for a in apps:
            s.register(a)
        s.run()
        out[(mode, graphed)] = [s.weights(a.job_id).cpu().clone() for a in apps]
        if mode == "p2p_gather":
            launches = [st.sync.kernel_launches for st in s.states]
            res["checks"].append({"name": "gather_mlp_one_kernel_per_sync", "ok": launches == [T, T],
                                  "launches": launches})
        s.close()
    g, p, e = out[("p2p_gather", True)], out[("p2p", True)], out[("p2p", False)]
    res["checks"].append({"name": f"gather_mlp_w{world}_bitwise_eq_p2p_graphed",
                          "ok": all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for a, b in zip(g, p))})
    res["checks"].append({"name": f"gather_mlp_w{world}_bitwise_eq_p2p_eager",
                          "ok": all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for a, b in zip(g, e))})
    res["checks"].append({"name": "gather_mlp_ranks_identical",
                          "ok": _gather_equal(torch.cat([x.reshape(-1) for x in g]), rank, world)})


def _resnet_update_check(rank, world, dev, comm, res, mode):
    from paper_2103_07974_b200.apps import DEFAULT_IMAGE_SGD, resnet50_app

    steps, batch = 3, 32
    apps = [resnet50_app(f"r{j}", batch, steps, dev, seed=1000 * j, data_seed=1000 * j + rank,
                         graphed=True, flat="ipc",
                         fast_bn=True) for j in range(2)]
    s = CrossoverScheduler(Policy.CROSSOVER, comm=comm, sync_mode=mode)
    for a in apps:
        s.register(a)
    before = {a.job_id: [p.detach().cpu().clone() for p in a.params] for a in apps}
    bufs = {a.job_id: None for a in apps}
    worst = {}
    ok = True
    while True:
        st = s._next_with_work()
        if st is None:
            break
        s.step()
        torch.cuda.synchronize()        # the graph's static gradients are rewritten by the next replay
        grads = [g.detach().cpu().clone() for g in st.held[0]]
        after = [p.detach().cpu().clone() for p in st.app.params]
        # every rank's gradients, summed in rank order 0..W-1 as K2 does, then / W
        allg = [None] * world
        dist.all_gather_object(allg, [g.numpy() for g in grads])
        sgd = DEFAULT_IMAGE_SGD
        params = [torch.nn.Parameter(p.clone()) for p in before[st.job_id]]
        opt = torch.optim.SGD(params, lr=sgd.lr, momentum=sgd.momentum, weight_decay=sgd.weight_decay,
                              foreach=False)
        if bufs[st.job_id] is not None:
            for p, b in zip(params, bufs[st.job_id]):
                opt.state[p]["momentum_buffer"] = b
        for i, p in enumerate(params):
            acc = torch.zeros_like(p)
            for r in range(world):
                acc = acc + torch.from_numpy(allg[r][i])
            p.grad = acc / world
        opt.step()
        bufs[st.job_id] = [opt.state[p]["momentum_buffer"] for p in params]
        mism = sum(int((a.view(torch.int32) != p.detach().view(torch.int32)).sum())
                   for a, p in zip(after, params))
        worst[f"{st.job_id}_t{st.next_iteration - 1}"] = mism
        ok = ok and mism == 0
        before[st.job_id] = after
    s.drain()
    launches = [st.sync.kernel_launches for st in s.states]
    modes = {st.sync.mode for st in s.states}
    s.close()
    res["checks"].append({"name": f"resnet50_{mode}_w{world}_bitwise_eq_torch_sgd", "ok": ok and modes == {mode},
                          "mismatched_elements": worst, "tensors": len(apps[0].params)})
    if mode == "p2p_gather":   # one kernel per sync: no K1 pack
        res["checks"].append({"name": "p2p_gather_one_kernel_per_sync", "ok": launches == [steps, steps],
                              "launches": launches})


def main():
    out_path, case = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev_index = 0 if os.environ.get("CS_PEER_SPREAD", "0") != "1" else rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = PeerGroup(rank, world)
    res = {"world": world, "case": case, "ok": True, "checks": []}
    {"parity": case_parity, "fail": case_fail, "resnet": case_resnet,
     "graph": case_graph, "gather": case_gather, "gather_mlp": case_gather_mlp}[case](rank, world, dev, comm, res)
    res["ok"] = all(c["ok"] for c in res["checks"])
    oks = [None] * world
    dist.all_gather_object(oks, res["ok"])
    if rank == 0:
        res["ranks_ok"] = oks
        res["ok"] = all(oks)
        Path(out_path).write_text(json.dumps(res, indent=1))
        print("PEERCHECK " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not res["ok"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
