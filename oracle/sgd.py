"""Numeric oracle of the crossover step (CPU, numpy) -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/colosim/equivalence.py:
  make_dataset        equivalence.py:84-95
  initial_state       equivalence.py:98-100
  loss_gradient       equivalence.py:103-126   (sigmoid via tanh)
  batch indices       equivalence.py:129-132
  local_gradient      equivalence.py:135-147
  average_gradients   equivalence.py:150-160   (fixed left-to-right sum, then / W)
  sgd_step            equivalence.py:163-168   (p - lr * avg)
  run_isolated        equivalence.py:177-187
  run_crossover       equivalence.py:190-232   (update j before its next compute; drain)
Everything is float64 like the reference; `dtype=np.float32` runs the same
sequence in fp32 (the device's arithmetic type) to bound the expected drift.

Extensions with no reference counterpart (parity UNPINNED by reference vectors):
  mlp_*               784-256-10 MLP, cross-entropy (config 1); cross-checked against torch
                      autograd + torch.optim.SGD in fp64 (tests/test_oracle_golden.py)
  torch_sgd_step      torch.optim.SGD momentum/weight-decay/nesterov semantics
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np

LEAST_SQUARES = "least_squares"
LOGISTIC = "logistic_regression"


def make_dataset(seed: int, dim: int, size: int, loss: str):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((size, dim))
    w_true = rng.standard_normal(dim)
    z = x @ w_true
    y = z if loss == LEAST_SQUARES else (z > 0).astype(np.float64)
    return x, y


def initial_parameters(dim: int, rng_seed: int) -> np.ndarray:
    return np.random.default_rng([rng_seed, 0]).standard_normal(dim)


def batch_indices(rng_seed: int, iteration: int, worker: int, size: int, batch: int) -> np.ndarray:
    return np.random.default_rng([rng_seed, 1, iteration, worker]).integers(0, size, size=batch)


def sigmoid(z):
    return 0.5 * (1.0 + np.tanh(0.5 * z))


def loss_gradient(loss: str, p: np.ndarray, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    z = x @ p
    r = z - y if loss == LEAST_SQUARES else sigmoid(z) - y
    return x.T @ r / len(y)


def average_gradients(grads: Sequence[np.ndarray]) -> np.ndarray:
    acc = np.zeros_like(grads[0])
    for g in grads:
        acc = acc + g
    return acc / acc.dtype.type(len(grads))


def sgd_step(p: np.ndarray, avg: np.ndarray, lr: float) -> np.ndarray:
    return p - p.dtype.type(lr) * avg


class LinearJob:
    """One reference SGD job: config fields of equivalence.SgdConfig + rng seed."""

    def __init__(self, lr: float, workers: int, loss: str, dataset_seed: int, rng_seed: int,
                 dim: int = 8, size: int = 128, batch: int = 16, dtype=np.float64):
        self.lr, self.workers, self.loss = lr, workers, loss
        self.size, self.batch, self.rng_seed, self.dtype = size, batch, rng_seed, dtype
        x, y = make_dataset(dataset_seed, dim, size, loss)
        self.x, self.y = x.astype(dtype), y.astype(dtype)
        self.p0 = initial_parameters(dim, rng_seed).astype(dtype)

    def averaged_gradient(self, p: np.ndarray, iteration: int) -> np.ndarray:
        grads = []
        for w in range(self.workers):
            idx = batch_indices(self.rng_seed, iteration, w, self.size, self.batch)
            grads.append(loss_gradient(self.loss, p, self.x[idx], self.y[idx]))
        return average_gradients(grads)


def run_isolated(job: LinearJob, iterations: int) -> list[np.ndarray]:
    p = job.p0
    out = []
    for t in range(1, iterations + 1):
        p = sgd_step(p, job.averaged_gradient(p, t), job.lr)
        out.append(p)
    return out


def run_isolated_momentum(job: LinearJob, iterations: int, momentum: float) -> list[np.ndarray]:
    """run_isolated with torch.optim.SGD momentum (no reference counterpart; fp64)."""
    p, buf, out = job.p0, None, []
    for t in range(1, iterations + 1):
        p, buf = torch_sgd_step(p, job.averaged_gradient(p, t), buf, job.lr, momentum=momentum,
                                first=t == 1)
        out.append(p)
    return out


def run_crossover(jobs: Sequence[LinearJob], iterations: int, perturb=None) -> list[list[np.ndarray]]:
    """Interleaved order of equivalence.py:224-231 (+ 1-ulp perturb hook, :214-219)."""
    params = [j.p0 for j in jobs]
    done = [0] * len(jobs)
    pending: list = [None] * len(jobs)
    traj: list[list[np.ndarray]] = [[] for _ in jobs]

    def apply(k):
        p = sgd_step(params[k], pending[k], jobs[k].lr)
        done[k] += 1
        if perturb is not None and perturb == (k, done[k]):
            p = p.copy()
            p[0] = np.nextafter(p[0], np.inf)
        params[k] = p
        traj[k].append(p)
        pending[k] = None

    for _ in range(iterations):
        for k, job in enumerate(jobs):
            if pending[k] is not None:
                apply(k)
            pending[k] = job.averaged_gradient(params[k], done[k] + 1)
    for k in range(len(jobs)):
        if pending[k] is not None:
            apply(k)
    return traj


# ---------------------------------------------------------------------------
# MLP 784-256-10 (config 1) -- no reference counterpart
# ---------------------------------------------------------------------------
def mlp_dataset(seed: int, size: int = 4096, in_dim: int = 784, classes: int = 10):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((size, in_dim)), rng.integers(0, classes, size=size)


def mlp_init(rng_seed: int, in_dim: int = 784, hidden: int = 256, classes: int = 10):
    rng = np.random.default_rng([rng_seed, 0])
    s1, s2 = 1.0 / math.sqrt(in_dim), 1.0 / math.sqrt(hidden)
    return [rng.standard_normal((hidden, in_dim)) * s1, rng.standard_normal(hidden) * s1,
            rng.standard_normal((classes, hidden)) * s2, rng.standard_normal(classes) * s2]


def mlp_gradient(params, x, y):
    """Mean cross-entropy gradient of Linear-ReLU-Linear (torch.nn.Linear layout)."""
    w1, b1, w2, b2 = params
    h_pre = x @ w1.T + b1
    h = np.maximum(h_pre, 0.0)
    logits = h @ w2.T + b2
    logits = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(logits)
    prob = e / e.sum(axis=1, keepdims=True)
    n = x.shape[0]
    d = prob
    d[np.arange(n), y] -= 1.0
    d /= n
    gw2 = d.T @ h
    gb2 = d.sum(axis=0)
    dh = (d @ w2) * (h_pre > 0)
    gw1 = dh.T @ x
    gb1 = dh.sum(axis=0)
    return [gw1, gb1, gw2, gb2]


def run_mlp_crossover(job_specs, iterations: int, workers: int, batch: int = 64, lr: float = 0.05,
                      dataset_size: int = 4096, momentum: float = 0.0):
    """job_specs: [(dataset_seed, rng_seed)]; returns per-job lists of per-iteration params.

    momentum > 0 applies torch.optim.SGD's momentum rule (torch_sgd_step) in fp64."""
    jobs = []
    for ds, rs in job_specs:
        x, y = mlp_dataset(ds, dataset_size)
        jobs.append((x, y, rs, mlp_init(rs)))
    params = [j[3] for j in jobs]
    bufs = [[None] * 4 for _ in jobs]
    traj = [[] for _ in jobs]
    for t in range(1, iterations + 1):       # isolated == crossover order (neutrality)
        for k, (x, y, rs, _) in enumerate(jobs):
            grads = []
            for w in range(workers):
                idx = batch_indices(rs, t, w, dataset_size, batch)
                grads.append(mlp_gradient(params[k], x[idx], y[idx]))
            avg = [average_gradients([g[i] for g in grads]) for i in range(4)]
            if momentum:
                new = []
                for i, (p, a) in enumerate(zip(params[k], avg)):
                    q, bufs[k][i] = torch_sgd_step(p, a, bufs[k][i], lr, momentum=momentum,
                                                   first=t == 1)
                    new.append(q)
                params[k] = new
            else:
                params[k] = [sgd_step(p, a, lr) for p, a in zip(params[k], avg)]
            traj[k].append(params[k])
    return traj


# ---------------------------------------------------------------------------
# torch.optim.SGD update semantics (momentum / dampening / nesterov / wd)
# ---------------------------------------------------------------------------
def torch_sgd_step(p, d, buf, lr, momentum=0.0, dampening=0.0, weight_decay=0.0,
                   nesterov=False, first=False):
    """float64 restatement of torch.optim.SGD's single-tensor update; returns (p, buf)."""
    if weight_decay:
        d = d + weight_decay * p
    if momentum:
        buf = d.copy() if first else momentum * buf + (1.0 - dampening) * d
        d = d + momentum * buf if nesterov else buf
    return p - lr * d, buf
