"""Scenario files: the reference's JSON config surface, as schedule plans and as real device runs.

Parsing restates ``colosim/scenario.py`` (units, exact-or-reject conversion, error texts):

* ``*_ms``  -> ns (x 1e6), ``grad_mb`` -> bytes (x 1e6), ``latency_us`` -> ns (x 1e3),
  ``bandwidth_gbps`` -> bytes/s (x 1e9 / 8), each through exact rational arithmetic on the
  decimal literal: a value that does not land on a whole internal unit is rejected
  (scenario.py:49-67);
* a job is either ``{"job_id", "profile": "resnet50"|"vgg16", ["iterations"]}`` (the bundled
  profile, workload.py:128-142) or inline ``{"job_id", "forward_ms", "backward_ms", "grad_mb",
  ["tensor_count"], "iterations"}`` whose payload is split into ``tensor_count`` tensors with the
  remainder spread over the first ones (scenario.py:114-158);
* ``iterations_override`` replaces every budget (scenario.py:40-47).

``Scenario.plan()`` is the reference's schedule plan (JobProfiles + the priced cluster).
``Scenario.device_plan()`` is what this package adds: the same jobs as
:class:`~.scheduler.App` objects that really train on the GPU -- profile jobs become the
torchvision model they name, inline jobs a synthetic app with exactly the job's tensor split and
a bf16 GEMM chain calibrated on the device to the job's forward + backward time -- so a reference
scenario file runs through the crossover pipeline and its measured trace feeds ``measure``.
"""

from __future__ import annotations

import dataclasses
import json
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path
from typing import Any, Mapping

from .comm import Architecture, ClusterSpec
from .errors import ConfigError
from .scheduler import Policy, SchedulePlan
from .workload import JobProfile, TensorSpec, fixture_names, fixture_profile

__all__ = ["Scenario", "load_config", "parse_scenario", "scaled_int", "calibrate_gemm_ms"]

_LIMIT = 1 << 63          # internal integers stay inside signed 64-bit (scenario.py:25-27)
_MAX_TENSORS = 10_000


@dataclass(frozen=True)
class Scenario:
    """A validated scenario in internal units (scenario.py:30-47)."""

    name: str
    jobs: tuple[JobProfile, ...]
    cluster: ClusterSpec
    policy: Policy
    iterations_override: int | None = None
    profiles: tuple[str | None, ...] = ()      # per job: the bundled profile it names, if any

    def _budgeted(self, iterations: int | None) -> tuple[JobProfile, ...]:
        n = self.iterations_override if iterations is None else iterations
        if n is None:
            return self.jobs
        if n < 1:
            raise ConfigError("iterations override must be >= 1")
        return tuple(dataclasses.replace(j, iterations=n) for j in self.jobs)

    def plan(self, iterations: int | None = None) -> SchedulePlan:
        """The reference's schedule plan: JobProfiles under the scenario's policy and cluster."""
        return SchedulePlan(self.policy, self._budgeted(iterations), self.cluster)

    def device_plan(self, device, iterations: int | None = None, *,
                    batch: Mapping[str, int] | None = None, time_scale: float = 1.0,
                    workers: int | None = None, policy: Policy | None = None,
                    flat: Any = False, graphed: bool = True, fast_bn: bool = True,
                    gemm_n: int = 4096, seed: int = 0,
                    data_seed: int | None = None) -> SchedulePlan:
        """The scenario's jobs as device Apps (see module docstring).

        ``workers`` (default ``cluster.workers``) is either the process group's world size (one
        worker per GPU) or, on a single GPU, up to 8 workers simulated back to back per job (the
        reference's own emulation, equivalence.py:171-174).  ``time_scale`` multiplies inline
        jobs' compute times before calibration (P100-era milliseconds are long); ``batch``
        sets the per-worker batch of profile jobs (default resnet50 256, vgg16 64).  ``seed``
        initialises the weights (identical on every rank), ``data_seed`` (default ``seed``) the
        per-rank batches.
        """
        from . import apps as _apps

        world = _apps._world()
        w = self.cluster.workers if workers is None else int(workers)
        if w < 1 or (world > 1 and w != world) or (world == 1 and w > 8):
            raise ConfigError(f"{self.name}: {w} workers cannot be spread over {world} rank(s): "
                              "use one worker per rank, or up to 8 simulated workers on one GPU "
                              "(device_plan(workers=...))")
        local = w // world
        sizes = {"resnet50": 256, "vgg16": 64, **(dict(batch) if batch else {})}
        jobs, gemm_ms = [], None
        for k, (job, prof) in enumerate(zip(self._budgeted(iterations), self.profiles)):
            if prof is not None:
                make = {"resnet50": _apps.resnet50_app, "vgg16": _apps.vgg16_app}[prof]
                app = make(job.job_id, sizes[prof], job.iterations, device, seed=seed + k,
                           data_seed=(seed if data_seed is None else data_seed) + k,
                           graphed=graphed and local == 1, flat=flat, fast_bn=fast_bn)
            else:
                if gemm_ms is None:
                    gemm_ms = calibrate_gemm_ms(device, gemm_n)
                target_ms = (job.forward_time + job.backward_time) * time_scale / 1e6
                reps = max(0, round(target_ms / gemm_ms))
                app = _apps.synthetic_app(job.job_id, job.grad_bytes, job.iterations, device,
                                          gemm_n=gemm_n, gemm_reps=reps, seed=seed + k,
                                          flat=flat, tensor_bytes=[t.size_bytes for t in job.tensors])
            jobs.append(dataclasses.replace(app, local_workers=local) if local > 1 else app)
        return SchedulePlan(policy or self.policy, tuple(jobs), self.cluster)


def calibrate_gemm_ms(device, n: int = 4096, reps: int = 20) -> float:
    """Device time of one bf16 [n,n] @ [n,n] (CUDA events, after warm-up)."""
    import torch

    a = torch.randn(n, n, device=device, dtype=torch.bfloat16)
    b = torch.randn(n, n, device=device, dtype=torch.bfloat16) / n ** 0.5
    for _ in range(3):
        a @ b
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(reps):
        a @ b
    stop.record()
    stop.synchronize()
    return start.elapsed_time(stop) / reps


# -- parsing ------------------------------------------------------------------

def scaled_int(value, num: int, den: int, field: str) -> int:
    """value * num / den as an exact integer, or ConfigError (scenario.py:49-67)."""
    if isinstance(value, bool) or not isinstance(value, (int, float)):
        raise ConfigError(f"{field}: expected a number, got {value!r}")
    try:
        q = Fraction(str(value)) * num / den
    except (ValueError, ZeroDivisionError):
        raise ConfigError(f"{field}: {value!r} is not a finite number") from None
    if q.denominator != 1:
        raise ConfigError(f"{field}: {value!r} does not land on a whole internal unit "
                          f"(scale {num}/{den})")
    if not -_LIMIT < q.numerator < _LIMIT:
        raise ConfigError(f"{field}: {value!r} overflows the internal integer range")
    return q.numerator


_MISSING = object()


def _get(obj: dict, key: str, where: str, default=_MISSING):
    if key in obj:
        return obj[key]
    if default is _MISSING:
        raise ConfigError(f"{where}: missing required field {key!r}")
    return default


def _count(obj: dict, key: str, where: str, default=_MISSING, minimum: int | None = None) -> int:
    v = _get(obj, key, where, default)
    if key not in obj:
        return v
    if isinstance(v, bool) or not isinstance(v, int):
        raise ConfigError(f"{where}.{key}: expected an integer, got {v!r}")
    if minimum is not None and v < minimum:
        raise ConfigError(f"{where}.{key}: must be >= {minimum}")
    return v


def _enum(cls, raw, field: str):
    try:
        return cls(raw)
    except ValueError:
        allowed = ", ".join(m.value for m in cls)
        raise ConfigError(f"{field}: unknown value {raw!r} (allowed: {allowed})") from None


def _cluster(obj) -> ClusterSpec:
    where = "cluster"
    if not isinstance(obj, dict):
        raise ConfigError(f"{where}: expected an object")
    arch = _enum(Architecture, _get(obj, "architecture", where), f"{where}.architecture")
    bw = scaled_int(_get(obj, "bandwidth_gbps", where), 10**9, 8, f"{where}.bandwidth_gbps")
    if bw <= 0:
        raise ConfigError(f"{where}.bandwidth_gbps: must be > 0")
    workers = _count(obj, "workers", where, minimum=1)
    gpus = _count(obj, "gpus_per_worker", where, 1, minimum=1)
    latency = scaled_int(obj.get("latency_us", 0), 10**3, 1, f"{where}.latency_us")
    servers = _count(obj, "ps_servers", where, 1, minimum=1)
    return ClusterSpec(workers=workers, bandwidth_bytes_per_sec=bw, latency_per_message=latency,
                       architecture=arch, gpus_per_worker=gpus, ps_servers=servers)


def _split(total: int, parts: int) -> tuple[TensorSpec, ...]:
    q, r = divmod(total, parts)
    return tuple(TensorSpec(f"grad_{i:03d}", q + (i < r)) for i in range(parts))


def _job(obj, index: int) -> tuple[JobProfile, str | None]:
    where = f"jobs[{index}]"
    if not isinstance(obj, dict):
        raise ConfigError(f"{where}: expected an object")
    job_id = _get(obj, "job_id", where)
    if not isinstance(job_id, str) or not job_id:
        raise ConfigError(f"{where}.job_id: expected a non-empty string")
    if "profile" in obj:
        name = obj["profile"]
        if name not in fixture_names():
            raise ConfigError(f"{where}.profile: unknown profile {name!r} "
                              f"(available: {', '.join(fixture_names())})")
        iters = _count(obj, "iterations", where, None, minimum=1)
        return fixture_profile(name, job_id=job_id, iterations=iters), name
    iters = _count(obj, "iterations", where, minimum=1)
    n_tensors = _count(obj, "tensor_count", where, 1, minimum=1)
    if n_tensors > _MAX_TENSORS:
        raise ConfigError(f"{where}.tensor_count: must be <= {_MAX_TENSORS}")
    payload = scaled_int(_get(obj, "grad_mb", where), 10**6, 1, f"{where}.grad_mb")
    if payload < 0:
        raise ConfigError(f"{where}.grad_mb: must be >= 0")
    fwd = scaled_int(_get(obj, "forward_ms", where), 10**6, 1, f"{where}.forward_ms")
    bwd = scaled_int(_get(obj, "backward_ms", where), 10**6, 1, f"{where}.backward_ms")
    if fwd < 0 or bwd < 0:
        raise ConfigError(f"{where}: compute times must be >= 0")
    if fwd + bwd <= 0:
        raise ConfigError(f"{where}: forward_ms + backward_ms must be > 0")
    return JobProfile(job_id, fwd, bwd, _split(payload, n_tensors), iters), None


def parse_scenario(doc, origin: str = "<config>") -> Scenario:
    """Validate a decoded JSON document (scenario.py:161-194)."""
    if not isinstance(doc, dict):
        raise ConfigError(f"{origin}: top level must be a JSON object")
    name = _get(doc, "name", origin)
    if not isinstance(name, str) or not name:
        raise ConfigError(f"{origin}: name must be a non-empty string")
    policy = _enum(Policy, _get(doc, "policy", origin), "policy")
    raw_jobs = _get(doc, "jobs", origin)
    if not isinstance(raw_jobs, list) or not raw_jobs:
        raise ConfigError("jobs: expected a non-empty array")
    parsed = [_job(j, i) for i, j in enumerate(raw_jobs)]
    ids = [j.job_id for j, _ in parsed]
    if len(set(ids)) != len(ids):
        raise ConfigError("jobs: job_id values must be unique")
    override = None
    if doc.get("iterations_override") is not None:
        override = _count(doc, "iterations_override", origin, minimum=1)
    return Scenario(name, tuple(j for j, _ in parsed), _cluster(_get(doc, "cluster", origin)),
                    policy, override, tuple(p for _, p in parsed))


def load_config(path: str | Path) -> Scenario:
    """Read and validate a scenario file; errors name the file and the field (scenario.py:197-212)."""
    path = Path(path)
    try:
        text = path.read_text()
    except OSError as exc:
        raise ConfigError(f"{path}: cannot read config: {exc}") from exc
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ConfigError(f"{path}: parse error at line {exc.lineno} column {exc.colno}: "
                          f"{exc.msg}") from exc
    return parse_scenario(doc, origin=str(path))
