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


def _ce_worker(rank, world, port, q):
    """The copy-engine transport's data movement on CPU: each rank 'pulls' its shard of every
    peer's bucket (an all-gather stands in for the copy engines), reduces the W shard copies in
    rank order, divides by W, applies SGD to its parameter shard, then 'pulls' every peer's
    updated shard.  Must equal the single-process W-worker oracle bitwise for any W.  Also the
    collective agreement used before enabling the flag barrier (p2p.all_ranks_agree)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_07974_b200.p2p import all_ranks_agree

    agree_all = all_ranks_agree(True)
    agree_one_no = all_ranks_agree(rank != world - 1)
    job = osgd.LinearJob(0.05, world, osgd.LEAST_SQUARES, 7, 0)
    p = job.p0.astype(np.float32).copy()
    n = p.size
    shard = -(-n // world)
    pad = shard * world - n
    traj = []
    for t in range(1, 6):
        idx = osgd.batch_indices(job.rng_seed, t, rank, job.size, job.batch)
        g = osgd.loss_gradient(job.loss, p.astype(np.float64), job.x[idx], job.y[idx]).astype(np.float32)
        bucket = torch.from_numpy(np.concatenate([g, np.zeros(pad, np.float32)]))
        copies = [torch.empty_like(bucket) for _ in range(world)]
        dist.all_gather(copies, bucket)                               # "pull" every peer's bucket
        acc = np.zeros(shard, np.float32)
        for r in range(world):                                        # rank order, one rounding per add
            acc = acc + copies[r].numpy()[rank * shard:(rank + 1) * shard]
        avg = acc / np.float32(world)
        pp = np.concatenate([p, np.zeros(pad, np.float32)])
        mine = pp[rank * shard:(rank + 1) * shard] - np.float32(job.lr) * avg
        parts = [torch.empty(shard) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine.astype(np.float32)))   # "pull" updated shards
        p = torch.cat(parts).numpy()[:n].copy()
        traj.append(p.copy())
    gathered = [None] * world
    dist.all_gather_object(gathered, (agree_all, agree_one_no, np.stack(traj)))
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ce_transport_data_movement_equals_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ce_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert all(g[0] is True for g in gathered)
    assert all(g[1] is False for g in gathered)          # one rank said no -> every rank hears no
    trajs = [g[2] for g in gathered]
    assert all(np.array_equal(trajs[0], t) for t in trajs)
    # fp32 restatement of the oracle's W-worker step: same rank-order sum, / W, p - lr * avg
    job = osgd.LinearJob(0.05, world, osgd.LEAST_SQUARES, 7, 0)
    p = job.p0.astype(np.float32).copy()
    for t in range(1, 6):
        acc = np.zeros_like(p)
        for w in range(world):
            idx = osgd.batch_indices(job.rng_seed, t, w, job.size, job.batch)
            acc = acc + osgd.loss_gradient(job.loss, p.astype(np.float64), job.x[idx], job.y[idx]).astype(np.float32)
        p = p - np.float32(job.lr) * (acc / np.float32(world))
        assert np.array_equal(p, trajs[0][t - 1])
