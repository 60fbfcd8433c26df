"""Fused-gradient synchronization of one app: K1 pack -> C1 all-reduce -> K2 update.

Reference: the fused payload of workload.fuse_gradients (workload.py:94-101),
the averaging of equivalence.average_gradients (equivalence.py:150-160) and
the update of equivalence.sgd_step (equivalence.py:163-168).  On the device
these are one ordered sequence on the comm stream:

  K1  pack      every gradient tensor of every local worker -> bucket row(s)
  C1  NCCL      in-place sum of the bucket across ranks (skipped at world 1)
  K2  update    sum the source rows left to right, / W, SGD(-momentum), in place

Modes
  ``bucket``  K1 -> (C1) -> K2: the general path (required whenever W > 1).
  ``direct``  W == 1 (one rank, one worker): nothing to communicate, so K2 reads
              the gradient tensors directly -- the bucket copy is skipped and
              the update costs 3S (5S with momentum) instead of 2S + 3S.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .comm import NcclCommunicator
from .errors import ConfigError
from .workload import BucketLayout

__all__ = ["SgdSettings", "FusedGradientSync"]


@dataclass(frozen=True)
class SgdSettings:
    """Per-app update rule.

    With no momentum and no weight decay the default rounding is the
    reference's ``p - lr * avg`` (equivalence.py:167, two roundings).  Otherwise
    the update follows torch.optim.SGD (dampening, nesterov, weight decay) with
    ATen's FMA rounding of ``add(x, alpha=a)``.
    """

    lr: float
    momentum: float = 0.0
    dampening: float = 0.0
    weight_decay: float = 0.0
    nesterov: bool = False
    rounding: str | None = None   # "reference" | "torch" | None (auto)

    def __post_init__(self):
        if self.lr <= 0:
            raise ValueError("learning_rate must be > 0")
        if self.momentum < 0 or self.weight_decay < 0:
            raise ValueError("momentum and weight_decay must be >= 0")
        if self.nesterov and (self.momentum <= 0 or self.dampening != 0):
            raise ValueError("nesterov needs momentum > 0 and dampening 0")
        if self.rounding not in (None, "reference", "torch"):
            raise ValueError("rounding must be 'reference' or 'torch'")
        if self.resolved_rounding == "reference" and (self.momentum or self.weight_decay):
            raise ValueError("reference rounding has no momentum / weight decay")

    @property
    def resolved_rounding(self) -> str:
        if self.rounding is not None:
            return self.rounding
        return "torch" if (self.momentum or self.weight_decay) else "reference"


class FusedGradientSync:
    """Owns one app's bucket, momentum buffers and K1/K2 descriptor tables."""

    def __init__(self, params: Sequence[torch.Tensor], settings: SgdSettings,
                 comm: NcclCommunicator | None = None, local_workers: int = 1,
                 align: int = 32, mode: str = "auto", snapshot_rows: int = 0):
        if not params:
            raise ConfigError("an app needs at least one trainable parameter")
        dev = params[0].device
        if dev.type != "cuda":
            raise ConfigError("parameters must live on a CUDA device (no CPU fallback)")
        for p in params:
            if p.dtype != torch.float32 or not _dense(p) or p.device != dev:
                raise ConfigError("parameters must be dense fp32 tensors on one device")
        self.params = list(params)
        self.settings = settings
        self.comm = comm
        self.ranks = comm.world if comm is not None else 1
        self.local_workers = int(local_workers)
        if self.local_workers < 1 or self.local_workers > _lib.CS_MAX_SOURCES:
            raise ConfigError(f"local_workers must be in [1, {_lib.CS_MAX_SOURCES}]")
        if self.ranks > 1 and self.local_workers > 1:
            raise ConfigError("simulated local workers are only supported at world size 1")
        self.workers = self.ranks * self.local_workers
        if mode == "auto":
            mode = "direct" if self.workers == 1 else "bucket"
        if mode not in ("bucket", "direct"):
            raise ConfigError(f"unknown sync mode {mode!r}")
        if mode == "direct" and self.workers != 1:
            raise ConfigError("direct mode has no bucket and needs exactly one worker")
        self.mode = mode
        self.layout = BucketLayout.build([p.numel() for p in self.params], align)
        n = len(self.params)
        lay = self.layout
        row_bytes = lay.bucket_bytes

        self.bucket = None
        if mode == "bucket":
            self.bucket = torch.zeros(self.local_workers * lay.total, dtype=torch.float32, device=dev)
        self.momentum_bufs = None
        if settings.momentum != 0:
            self.momentum_bufs = [torch.zeros_like(p) for p in self.params]
        self.first_step = True
        self.snapshot = None
        if snapshot_rows:
            self.snapshot = torch.zeros(snapshot_rows, lay.total, dtype=torch.float32, device=dev)

        offs_bytes = lay.offsets_array() * 4
        numels = np.asarray(lay.numels, dtype=np.int64)
        # K1 descriptors: one per (worker, tensor); src filled per iteration
        self._pack = np.zeros(self.local_workers * n, dtype=_lib.PACK_DESC)
        if self.bucket is not None:
            base = self.bucket.data_ptr()
            for w in range(self.local_workers):
                sl = self._pack[w * n:(w + 1) * n]
                sl["dst"] = base + w * row_bytes + offs_bytes
                sl["numel"] = numels
        # K2 descriptors: fixed except grad_offset in direct mode
        self._upd = np.zeros(n, dtype=_lib.UPDATE_DESC)
        self._upd["param"] = [p.data_ptr() for p in self.params]
        if self.momentum_bufs is not None:
            self._upd["momentum_buf"] = [b.data_ptr() for b in self.momentum_bufs]
        self._upd["snap_offset"] = offs_bytes
        self._upd["numel"] = numels
        if mode == "bucket":
            self._upd["grad_offset"] = offs_bytes
            self._sources = np.asarray([self.bucket.data_ptr() + w * row_bytes
                                        for w in range(self.local_workers)], dtype=np.uint64)
        else:
            self._sources = np.zeros(1, dtype=np.uint64)
        self._hyper = _lib.SgdHyper(
            lr=settings.lr, momentum=settings.momentum,
            dampening_complement=float(1.0 - settings.dampening),
            weight_decay=settings.weight_decay, nesterov=int(settings.nesterov), first_step=1,
            divisor=self.workers,
            rounding=_lib.CS_ROUND_TORCH if settings.resolved_rounding == "torch" else _lib.CS_ROUND_REFERENCE)
        self.kernel_launches = 0

    # -- per-iteration pieces (all asynchronous on `stream`) -----------------
    def pack(self, grads_per_worker: Sequence[Sequence[torch.Tensor]], stream: int) -> None:
        """K1: gather each worker's gradients into its bucket row."""
        if self.mode != "bucket":
            raise ConfigError("pack() needs bucket mode")
        n = len(self.params)
        if len(grads_per_worker) != self.local_workers:
            raise ValueError(f"expected gradients of {self.local_workers} worker(s)")
        for w, grads in enumerate(grads_per_worker):
            self._pack["src"][w * n:(w + 1) * n] = _grad_ptrs(grads, self.params)
        _lib.pack(self._pack, stream)
        self.kernel_launches += 1

    def all_reduce(self, stream: int) -> None:
        """C1: in-place NCCL sum of the bucket across ranks (no-op at world 1)."""
        if self.comm is not None and self.comm.active:
            self.comm.all_reduce_(self.bucket.data_ptr(), self.layout.total, stream)

    def update(self, stream: int, grads: Sequence[torch.Tensor] | None = None,
               snapshot_row: int | None = None) -> None:
        """K2: reduce the source rows left to right, / W, SGD step in place."""
        if self.mode == "direct":
            if grads is None:
                raise ValueError("direct mode needs the gradient tensors")
            self._upd["grad_offset"] = _grad_ptrs(grads, self.params)
        snap = 0
        if snapshot_row is not None:
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            snap = self.snapshot[snapshot_row].data_ptr()
        self._hyper.first_step = int(self.first_step)
        _lib.unpack_sgd(self._upd, self._sources, snap, self._hyper, stream)
        self.first_step = False
        self.kernel_launches += 1

    def sync(self, grads_per_worker: Sequence[Sequence[torch.Tensor]], stream: int,
             snapshot_row: int | None = None, timer=None) -> None:
        """The whole sync phase of one iteration: K1 -> C1 -> K2 (or K2 alone in direct mode)."""
        if self.mode == "direct":
            if timer is not None:
                timer.begin("k2_update")
            self.update(stream, grads_per_worker[0], snapshot_row)
            if timer is not None:
                timer.end("k2_update")
            return
        if timer is not None:
            timer.begin("k1_pack")
        self.pack(grads_per_worker, stream)
        if timer is not None:
            timer.end("k1_pack")
        if self.comm is not None and self.comm.active:
            if timer is not None:
                timer.begin("c1_allreduce")
            self.all_reduce(stream)
            if timer is not None:
                timer.end("c1_allreduce")
        if timer is not None:
            timer.begin("k2_update")
        self.update(stream, None, snapshot_row)
        if timer is not None:
            timer.end("k2_update")

    # -- algorithmic bytes per launch ---------------------------
    def k1_bytes(self) -> int:
        return 2 * self.local_workers * self.layout.payload_bytes

    def k2_bytes(self) -> int:
        s = self.layout.payload_bytes
        streams = self.local_workers if self.mode == "bucket" else 1
        per = (streams + 2) * s            # read sources + read p + write p
        if self.settings.momentum:
            per += 2 * s                   # read + write the momentum buffer
        return per

    def c1_bus_bytes(self) -> float:
        w = self.ranks
        return 0.0 if w <= 1 else 2.0 * (w - 1) / w * self.layout.bucket_bytes


_zero_cache: dict[tuple, torch.Tensor] = {}


def _dense(t: torch.Tensor) -> bool:
    """Non-overlapping and dense in one of the layouts the models use.

    K1/K2 walk a tensor's storage linearly, so a channels_last conv weight is
    fine as long as its gradient (and momentum buffer) share its strides.
    """
    if t.is_contiguous():
        return True
    return t.dim() == 4 and t.is_contiguous(memory_format=torch.channels_last)


def _grad_ptrs(grads: Sequence[torch.Tensor | None], params: Sequence[torch.Tensor]) -> list[int]:
    """Device addresses of the gradients, in parameter order.

    A gradient whose strides differ from its parameter's (rare: autograd
    usually mirrors the parameter layout) is re-laid-out to the parameter's
    strides so storage order matches element for element.
    """
    if len(grads) != len(params):
        raise ValueError("one gradient per parameter expected")
    out = []
    for i, (g, p) in enumerate(zip(grads, params)):
        if g is None:   # parameter unused in this iteration's graph: zero gradient
            key = (p.device, p.numel())
            z = _zero_cache.get(key)
            if z is None:
                z = _zero_cache[key] = torch.zeros(p.numel(), dtype=torch.float32, device=p.device)
            g = z
        else:
            if g.dtype != torch.float32:
                raise ConfigError("gradients must be fp32 (parameters are fp32 masters)")
            if g.stride() != p.stride() or not _dense(g):
                fixed = torch.empty_like(p)
                fixed.copy_(g)
                g = fixed
                if isinstance(grads, list):
                    grads[i] = fixed  # keep it alive as long as the caller holds the list
        out.append(g.data_ptr())
    return out
