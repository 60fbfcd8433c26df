"""World-size-2 host logic on CPU (gloo): the sharded data-parallel step.

Each rank is one worker (worker index = rank, equivalence.py:131), computes its
local gradient, the bucket is summed across ranks (gloo stands in for NCCL),
divided by W and applied.  The result must equal the single-process oracle
with W workers BITWISE (two-operand sums are commutative), every rank must end
with identical weights, and every rank must emit the identical collective order
(the rotation schedule), which NCCL requires.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sgd as osgd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_07974_b200.scheduler import rotation_schedule

    jobs = [osgd.LinearJob(0.05, world, osgd.LEAST_SQUARES, 5, 0),
            osgd.LinearJob(0.05, world, osgd.LOGISTIC, 6, 1)]
    params = [j.p0.copy() for j in jobs]
    order = rotation_schedule(["a", "b"], [6, 6])
    traj = [[], []]
    for lane, job, phase, t in order:
        if phase != "sync":
            continue
        k = 0 if job == "a" else 1
        j = jobs[k]
        idx = osgd.batch_indices(j.rng_seed, t, rank, j.size, j.batch)   # worker = rank
        g = torch.from_numpy(osgd.loss_gradient(j.loss, params[k], j.x[idx], j.y[idx]))
        dist.all_reduce(g)                                               # C1 (sum)
        params[k] = osgd.sgd_step(params[k], g.numpy() / world, j.lr)     # K2 (/W, SGD)
        traj[k].append(params[k].copy())
    gathered = [None] * world
    dist.all_gather_object(gathered, (order, [np.stack(t) for t in traj]))
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_step_equals_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    orders = [g[0] for g in gathered]
    assert all(o == orders[0] for o in orders)
    trajs = [g[1] for g in gathered]
    for k in range(2):
        assert all(np.array_equal(trajs[0][k], t[k]) for t in trajs)
    jobs = [osgd.LinearJob(0.05, world, osgd.LEAST_SQUARES, 5, 0),
            osgd.LinearJob(0.05, world, osgd.LOGISTIC, 6, 1)]
    ref = osgd.run_crossover(jobs, 6)
    for k in range(2):
        assert np.array_equal(np.stack(ref[k]), trajs[0][k])
