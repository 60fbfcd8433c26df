"""The NVSwitch-multicast transport (``nvls``) on W GPUs (launched by tests/test_gpu_multirank.py).

The switch sums the W bucket shards in an unspecified order, so the check is tolerance-based:
linear momentum jobs vs the fp64 oracle within 1e-5 + 1e-4|w| (equivalence.py:150-232 structure),
the MLP trajectories within a few fp32 ulps of the rank-order p2p transport, and every rank holds
bitwise the same weights (the switch broadcasts one value to all of them).
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
from paper_2103_07974_b200.apps import LossKind, MlpConfig, SgdConfig, linear_app, mlp_app  # noqa: E402
from paper_2103_07974_b200.comm import PeerGroup  # noqa: E402
from paper_2103_07974_b200.nvls import nvls_available  # noqa: E402
from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy  # noqa: E402


def run(apps, comm, mode):
    s = CrossoverScheduler(Policy.CROSSOVER, comm=comm, record_weights=True, sync_mode=mode)
    for a in apps:
        s.register(a)
    s.run()
    w = [s.weights(a.job_id).cpu().clone() for a in apps]
    modes = {st.sync.mode for st in s.states}
    s.close()
    return w, modes


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dev = torch.device("cuda", torch.cuda.current_device())
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = PeerGroup(rank, world)
    res = {"world": world, "checks": []}
    avail = [None] * world
    dist.all_gather_object(avail, nvls_available(dev))
    if not all(avail):
        res["skipped"] = "no NVSwitch multicast"
        res["ok"] = True
    else:
        T = 8
        specs = [(11, 0), (12, 1)]
        w = {}
        for mode, flat in (("p2p", "ipc"), ("nvls", "nvls")):
            apps = [mlp_app(MlpConfig(dataset_seed=ds, workers=world, momentum=0.9), f"m{k}", rs, T, dev,
                            local_workers=1, worker_count=world, flat=flat) for k, (ds, rs) in enumerate(specs)]
            w[mode], modes = run(apps, comm, mode)
            res["checks"].append({"name": f"{mode}_mode_used", "ok": modes == {mode}})
        n = min(w["p2p"][0].shape[1], w["nvls"][0].shape[1])
        rel = max(float(((a[:, :n] - b[:, :n]).abs() / (1e-6 + b[:, :n].abs())).max())
                  for a, b in zip(w["nvls"], w["p2p"]))
        res["checks"].append({"name": "mlp_nvls_close_to_p2p", "ok": rel <= 1e-3, "max_rel": rel})
        allw = [None] * world
        dist.all_gather_object(allw, torch.cat([x.reshape(-1) for x in w["nvls"]]).numpy().tobytes())
        res["checks"].append({"name": "nvls_ranks_identical", "ok": len(set(allw)) == 1})
        lcfg = [SgdConfig(0.05, world, LossKind.LEAST_SQUARES, 123), SgdConfig(0.05, world, LossKind.LOGISTIC, 124)]
        apps = [linear_app(c, f"lm{k}", 40 + k, 20, dev, local_workers=1, momentum=0.9, flat="nvls")
                for k, c in enumerate(lcfg)]
        lw, _ = run(apps, comm, "nvls")
        jobs = [osgd.LinearJob(0.05, world, c.loss.value, c.dataset_seed, 40 + k) for k, c in enumerate(lcfg)]
        ref = [np.stack(osgd.run_isolated_momentum(j, 20, 0.9)) for j in jobs]
        wr = max(float(np.max(np.abs(lw[k][:, :8].numpy().astype(np.float64) - ref[k]) /
                              (1e-5 + 1e-4 * np.abs(ref[k])))) for k in range(2))
        res["checks"].append({"name": "linear_momentum_nvls_vs_fp64_oracle", "ok": wr <= 1.0, "worst_ratio": wr})
        # sync_mode="auto" with multicast-bound flat parameters selects nvls (both policies)
        apps = [linear_app(lcfg[0], "auto0", 40, 4, dev, local_workers=1, momentum=0.9, flat="nvls")]
        for pol in (Policy.CROSSOVER, Policy.SEQUENTIAL):
            s = CrossoverScheduler(pol, comm=comm, sync_mode="auto")
            s.register(apps[0])
            res["checks"].append({"name": f"auto_selects_nvls_{pol.value}", "ok": s.states[0].sync.mode == "nvls"})
            s.run()
            s.close()
        res["ok"] = all(c["ok"] for c in res["checks"])
    oks = [None] * world
    dist.all_gather_object(oks, res["ok"])
    if rank == 0:
        res["ok"] = all(oks)
        Path(out_path).write_text(json.dumps(res, indent=1))
        print("NVLSCHECK " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not res["ok"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
