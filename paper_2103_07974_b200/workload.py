"""App registration records and the fused-gradient bucket layout.

Reference: colosim.workload (workload.py:31-115).  ``TensorSpec``/``JobProfile``
keep the reference's fields and invariants; ``fuse_gradients`` keeps its
meaning (one message whose payload is the byte sum of all gradient tensors).
What is new is :class:`BucketLayout`: the fused payload is no longer only a
number, it is a real contiguous fp32 buffer in HBM, and the layout decides
where every gradient lands in it (tensor order = ``named_parameters()`` order,
offsets = exclusive prefix sum, optionally padded so each tensor starts on a
16-byte / 128-byte boundary for the 128-bit vector path of K1/K2).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

__all__ = [
    "TensorSpec",
    "JobProfile",
    "FusedGradient",
    "fuse_gradients",
    "unfused_messages",
    "comp_time",
    "BucketLayout",
    "tensor_specs_from_module",
    "profile_from_module",
    "fixture_names",
    "fixture_profile",
]

FP32_BYTES = 4


@dataclass(frozen=True)
class TensorSpec:
    """One gradient tensor: name and payload bytes (workload.py:31-40)."""

    name: str
    size_bytes: int

    def __post_init__(self):
        if self.size_bytes < 0:
            raise ValueError(f"tensor {self.name!r}: size_bytes must be >= 0")


@dataclass(frozen=True)
class JobProfile:
    """Per-iteration cost profile of one app (workload.py:43-74).

    On the device path the durations are *measured* (CUDA events) rather than
    given; the tensor list is the model's parameter list in registration order.
    """

    job_id: str
    forward_time: int
    backward_time: int
    tensors: tuple[TensorSpec, ...]
    iterations: int

    def __post_init__(self):
        object.__setattr__(self, "tensors", tuple(self.tensors))
        if self.forward_time < 0 or self.backward_time < 0:
            raise ValueError(f"job {self.job_id!r}: compute times must be >= 0")
        if self.forward_time + self.backward_time <= 0:
            raise ValueError(f"job {self.job_id!r}: forward + backward must be > 0")
        if self.iterations < 1:
            raise ValueError(f"job {self.job_id!r}: iterations must be >= 1")
        if not self.tensors:
            raise ValueError(f"job {self.job_id!r}: tensor list must be non-empty")
        if len({t.name for t in self.tensors}) != len(self.tensors):
            raise ValueError(f"job {self.job_id!r}: tensor names must be unique")

    @property
    def grad_bytes(self) -> int:
        return sum(t.size_bytes for t in self.tensors)


@dataclass(frozen=True)
class FusedGradient:
    """A gradient payload ready for synchronization (workload.py:77-84)."""

    job_id: str
    iteration: int
    size_bytes: int
    message_count: int = 1


def _check_iteration(job: JobProfile, iteration: int) -> None:
    if not 1 <= iteration <= job.iterations:
        raise ValueError(
            f"job {job.job_id!r}: iteration {iteration} out of range [1, {job.iterations}]")


def fuse_gradients(job: JobProfile, iteration: int) -> FusedGradient:
    """All gradients as one message (workload.py:94-101); the device gather is K1."""
    _check_iteration(job, iteration)
    return FusedGradient(job.job_id, iteration, job.grad_bytes, 1)


def unfused_messages(job: JobProfile, iteration: int) -> list[FusedGradient]:
    """One message per tensor (workload.py:104-110): the per-tensor counterfactual."""
    _check_iteration(job, iteration)
    return [FusedGradient(job.job_id, iteration, t.size_bytes, 1) for t in job.tensors]


def comp_time(job: JobProfile) -> int:
    """Forward + backward nanoseconds of one iteration (workload.py:113-115)."""
    return job.forward_time + job.backward_time


@dataclass(frozen=True)
class BucketLayout:
    """Placement of every gradient tensor inside one contiguous fp32 bucket.

    ``offsets[i]`` is the element offset of tensor i; tensor order is the
    registration order.  ``align`` (elements) pads each offset up to a multiple
    of ``align``: 1 reproduces the reference's exact prefix sum (the payload is
    exactly ``grad_bytes``), 4 gives 16-byte alignment for 128-bit vector
    access, 32 gives 128-byte (cache-line) alignment.  Padding elements are
    zero in the bucket and never read back into parameters.
    """

    numels: tuple[int, ...]
    offsets: tuple[int, ...]
    total: int          # padded bucket length in elements (multiple of `align`)
    align: int

    @staticmethod
    def build(numels: Sequence[int], align: int = 32, multiple: int | None = None) -> "BucketLayout":
        """``multiple`` pads the total length (default ``align``), e.g. to align * W so the
        bucket splits into W equal, aligned shards for reduce-scatter / sharded updates."""
        if align < 1:
            raise ValueError("align must be >= 1")
        if not numels:
            raise ValueError("bucket needs at least one tensor")
        offs = []
        cur = 0
        for n in numels:
            if n < 0:
                raise ValueError("numel must be >= 0")
            cur = -(-cur // align) * align
            offs.append(cur)
            cur += int(n)
        mult = align if multiple is None else int(multiple)
        if mult < 1 or mult % align:
            raise ValueError("multiple must be a positive multiple of align")
        total = -(-cur // mult) * mult
        return BucketLayout(tuple(int(n) for n in numels), tuple(offs), total, align)

    @property
    def payload_elems(self) -> int:
        """Σ numel: the reference's fused payload (workload.py:72-74) in elements."""
        return sum(self.numels)

    @property
    def payload_bytes(self) -> int:
        return FP32_BYTES * self.payload_elems

    @property
    def bucket_bytes(self) -> int:
        return FP32_BYTES * self.total

    def offsets_array(self) -> np.ndarray:
        return np.asarray(self.offsets, dtype=np.int64)


def tensor_specs_from_module(module, dtype_bytes: int = FP32_BYTES) -> tuple[TensorSpec, ...]:
    """TensorSpec list of a torch module's trainable parameters, in registration order."""
    return tuple(TensorSpec(name, p.numel() * dtype_bytes)
                 for name, p in module.named_parameters() if p.requires_grad)


def profile_from_module(module, job_id: str, forward_time: int, backward_time: int,
                        iterations: int) -> JobProfile:
    """A reference JobProfile for a real model (e.g. after measuring its fwd/bwd)."""
    return JobProfile(job_id, int(forward_time), int(backward_time),
                      tensor_specs_from_module(module), iterations)


def total_bytes(specs: Iterable[TensorSpec]) -> int:
    return sum(s.size_bytes for s in specs)


# Bundled calibration profiles (colosim/data/profiles.json, read by workload.py:118-142): the
# reference pins order-of-magnitude P100 step times at batch 32 and the models' fp32 parameter
# tensors.  The times are restated here; the tensor tables are taken from the torchvision model
# itself (built on the meta device, no allocation) -- tests/test_scenario.py checks both against
# the reference's fixture, tensor by tensor.
_FIXTURE_TIMES = {"resnet50": (75_000_000, 155_000_000, 100),
                  "vgg16": (190_000_000, 390_000_000, 100)}


def fixture_names() -> list[str]:
    return sorted(_FIXTURE_TIMES)


def fixture_profile(name: str, job_id: str | None = None,
                    iterations: int | None = None) -> JobProfile:
    """The reference's named profile (workload.py:128-142) as a JobProfile."""
    if name not in _FIXTURE_TIMES:
        raise KeyError(f"unknown fixture profile {name!r}; available: {fixture_names()}")
    import torch
    import torchvision

    with torch.device("meta"):
        module = getattr(torchvision.models, name)()
    specs = tensor_specs_from_module(module)
    if name == "vgg16":
        specs = _vgg_layer_names(module, specs)
    fwd, bwd, iters = _FIXTURE_TIMES[name]
    return JobProfile(job_id if job_id is not None else name, fwd, bwd, specs,
                      iterations if iterations is not None else iters)


def _vgg_layer_names(module, specs: tuple[TensorSpec, ...]) -> tuple[TensorSpec, ...]:
    """torchvision's ``features.<i>`` / ``classifier.<i>`` -> the paper's convB_L / fcK names
    (the fixture's naming); block B advances at each max-pool."""
    import torch

    rename, block, layer = {}, 1, 0
    for i, m in enumerate(module.features):
        if isinstance(m, torch.nn.MaxPool2d):
            block, layer = block + 1, 0
        elif isinstance(m, torch.nn.Conv2d):
            layer += 1
            rename[f"features.{i}"] = f"conv{block}_{layer}"
    fc = 0
    for i, m in enumerate(module.classifier):
        if isinstance(m, torch.nn.Linear):
            fc += 1
            rename[f"classifier.{i}"] = f"fc{fc}"
    out = []
    for t in specs:
        prefix, _, leaf = t.name.rpartition(".")
        out.append(TensorSpec(f"{rename.get(prefix, prefix)}.{leaf}", t.size_bytes))
    return tuple(out)
