"""The reference's numeric API, executed by the device crossover pipeline.

Reference: colosim.equivalence (equivalence.py:177-266).  Same function names,
arguments and return shapes; the difference is where the arithmetic runs:
every gradient, the fixed-order worker reduction, the 1/W average and the SGD
update happen on the GPU (K2 reduces the W simulated workers' bucket rows left
to right exactly like ``average_gradients``), in fp32.  Trajectories are
captured by K2 itself (snapshot rows) and copied to the host once at the end.

Parity statement: per-iteration weights match the fp64 reference
within ``atol + rtol*|w|`` (see tests); GPU crossover vs GPU isolated is bitwise.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .apps import LossKind, SgdConfig, linear_app
from .scheduler import CrossoverScheduler, Policy

__all__ = ["LossKind", "SgdConfig", "TrainingState", "run_isolated", "run_crossover",
           "NeutralityReport", "check_neutrality"]


@dataclass
class TrainingState:
    """Parameters after ``iteration`` completed updates (equivalence.py:68-74)."""

    parameters: np.ndarray
    iteration: int
    rng_seed: int


def _run(configs: Sequence[SgdConfig], iterations: int, rng_seeds: Sequence[int],
         perturb, policy: Policy, device) -> list[list[TrainingState]]:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    sched = CrossoverScheduler(policy, device=dev, record_weights=True, perturb=perturb)
    for j, (cfg, seed) in enumerate(zip(configs, rng_seeds)):
        sched.register(linear_app(cfg, f"job{j}", seed, iterations, dev))
    sched.run()
    out = []
    for j, (cfg, seed) in enumerate(zip(configs, rng_seeds)):
        w = sched.weights(f"job{j}")[:, :cfg.dim].cpu().numpy()
        out.append([TrainingState(w[t].copy(), t + 1, seed) for t in range(iterations)])
    return out


def run_isolated(config: SgdConfig, iterations: int, rng_seed: int = 0,
                 device=None) -> list[TrainingState]:
    """Plain synchronous SGD of one job on the device (equivalence.py:177-187)."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    return _run([config], iterations, [rng_seed], None, Policy.CROSSOVER, device)[0]


def run_crossover(configs: Sequence[SgdConfig], iterations: int,
                  rng_seeds: Sequence[int] | None = None,
                  perturb: tuple[int, int] | None = None, device=None,
                  policy: Policy = Policy.CROSSOVER) -> list[list[TrainingState]]:
    """All jobs co-located under crossover sync on the device (equivalence.py:190-232)."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if not configs:
        raise ValueError("at least one job config required")
    if rng_seeds is None:
        rng_seeds = list(range(len(configs)))
    if len(rng_seeds) != len(configs):
        raise ValueError("rng_seeds must match configs")
    return _run(list(configs), iterations, list(rng_seeds), perturb, policy, device)


@dataclass(frozen=True)
class NeutralityReport:
    max_abs_deviation: float
    first_divergence: tuple[int, int, int] | None

    @property
    def equal(self) -> bool:
        return self.first_divergence is None and self.max_abs_deviation == 0.0


def check_neutrality(configs: Sequence[SgdConfig], iterations: int,
                     rng_seeds: Sequence[int] | None = None,
                     perturb: tuple[int, int] | None = None, device=None) -> NeutralityReport:
    """Device crossover vs device isolated, bit for bit (equivalence.py:247-266)."""
    if rng_seeds is None:
        rng_seeds = list(range(len(configs)))
    crossed = run_crossover(configs, iterations, rng_seeds, perturb=perturb, device=device)
    max_dev, first = 0.0, None
    for j, (cfg, seed) in enumerate(zip(configs, rng_seeds)):
        iso = run_isolated(cfg, iterations, seed, device=device)
        for t, (a, b) in enumerate(zip(iso, crossed[j]), start=1):
            diff = np.abs(a.parameters.astype(np.float64) - b.parameters.astype(np.float64))
            dev = float(diff.max()) if diff.size else 0.0
            max_dev = max(max_dev, dev)
            if first is None and dev != 0.0:
                first = (j, t, int(np.argmax(diff != 0.0)))
    return NeutralityReport(max_dev, first)
