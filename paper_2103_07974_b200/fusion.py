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

import ctypes

import numpy as np
import torch

from . import _lib
from .comm import NcclCommunicator
from .errors import ConfigError
from .workload import BucketLayout

__all__ = ["SgdSettings", "FusedGradientSync", "flatten_parameters"]


def flatten_parameters(params: Sequence[torch.Tensor], align: int = 32, shards: int = 1,
                       ipc: bool = False):
    """Move every parameter into one contiguous fp32 buffer laid out like the bucket.

    Each parameter keeps its shape and strides (channels_last stays channels_last) but
    its storage becomes a view of ``flat`` at ``layout.offsets[i]``; the total is padded
    to ``align * shards`` so the buffer splits into equal aligned shards.  This is what
    lets the sharded sync all-gather updated shards straight into the model's weights.
    Call it before anything captures parameter addresses (CUDA graphs).  ``ipc=True``
    allocates the buffer with cs_device_alloc so peers can map it (p2p / ce sync modes);
    ``ipc="nvls"`` binds it to an NVSwitch multicast object (nvls sync mode, collective).
    """
    lay = BucketLayout.build([p.numel() for p in params], align, multiple=align * shards)
    dev = params[0].device
    if ipc == "nvls":
        import torch.distributed as dist

        from .nvls import NvlsBuffer

        flat = NvlsBuffer(lay.total, dev, dist.get_rank(), dist.get_world_size()).tensor
    elif ipc:
        from .p2p import DeviceBuffer

        flat = DeviceBuffer(lay.total, dev).tensor
    else:
        flat = torch.zeros(lay.total, dtype=torch.float32, device=dev)
    with torch.no_grad():
        for p, off in zip(params, lay.offsets):
            if p.dtype != torch.float32 or not _dense(p):
                raise ConfigError("flat parameters need dense fp32 tensors")
            view = torch.as_strided(flat, p.shape, p.stride(), off)
            view.copy_(p.data)
            p.data = view
    return flat, lay


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
    """Owns one app's bucket, momentum buffers and K1/K2 descriptor tables.

    Sync modes (one per app):
      direct    W = 1: K2 reads the gradient tensors in place (no bucket)
      bucket    K1 -> NCCL all-reduce of the bucket -> K2 (also W simulated workers on one GPU)
      sharded   K1 -> reduce-scatter -> K2 on this rank's shard -> all-gather into flat params
      p2p       K1 -> barrier -> one NVLink kernel (rank-order reduce, /W, SGD, broadcast writes)
      p2p_gather  no K1: barrier -> the same kernel reading every rank's gradient tensors in place
                (static gradient addresses: CUDA-graphed backward passes) -> barrier
      ce        K1 -> barrier -> copy-engine pulls -> shard K2 -> barrier -> copy-engine pulls
      adaptive  p2p and ce over the same buffers; the scheduler picks one per sync
      unfused   one all-reduce per gradient tensor (the per-message counterfactual), then K2
    """

    def __init__(self, params: Sequence[torch.Tensor], settings: SgdSettings,
                 comm: NcclCommunicator | None = None, local_workers: int = 1,
                 align: int = 32, mode: str = "auto", snapshot_rows: int = 0,
                 flat_params: torch.Tensor | None = None, p2p_ctas: int = 0,
                 barrier: str = "auto", sync_ctas: int = 0, pack_engine: str = "sm"):
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
        self.sync_ctas = int(sync_ctas)     # K1 / K2 persistent grid cap (0: one CTA per chunk)
        if pack_engine not in ("sm", "ce"):
            raise ConfigError(f"unknown pack engine {pack_engine!r}")
        self.pack_engine = pack_engine      # K1 by the SMs (kernel) or by the copy engines
        self.comm = comm
        self.ranks = comm.world if comm is not None else 1
        self.local_workers = int(local_workers)
        if self.local_workers < 1 or self.local_workers > _lib.CS_MAX_SOURCES:
            raise ConfigError(f"local_workers must be in [1, {_lib.CS_MAX_SOURCES}]")
        if self.ranks > 1 and self.local_workers > 1:
            raise ConfigError("simulated local workers are only supported at world size 1")
        self.workers = self.ranks * self.local_workers
        if mode == "auto":
            if self.workers == 1:
                mode = "direct"
            elif not getattr(comm, "has_collectives", True):
                mode = "ce"
            else:
                mode = "sharded" if (flat_params is not None and self.local_workers == 1) else "bucket"
        if mode not in ("bucket", "direct", "sharded", "p2p", "p2p_gather", "ce", "adaptive", "unfused", "nvls"):
            raise ConfigError(f"unknown sync mode {mode!r}")
        if mode == "direct" and self.workers != 1:
            raise ConfigError("direct mode has no bucket and needs exactly one worker")
        if mode == "unfused" and self.local_workers != 1:
            raise ConfigError("unfused mode all-reduces each gradient tensor in place: one worker per rank")
        if mode in ("sharded", "p2p", "p2p_gather", "ce", "adaptive", "nvls") and (
                flat_params is None or self.local_workers != 1 or self.ranks < 2):
            raise ConfigError("sharded mode needs flat parameters (flatten_parameters), world > 1 "
                              "and one worker per rank")
        if (self.ranks > 1 and mode in ("bucket", "sharded", "unfused")
                and not getattr(comm, "has_collectives", True)):
            raise ConfigError(f"{mode} sync needs an NCCL communicator at world > 1")
        self.mode = mode
        self.flat = flat_params
        sharded = mode in ("sharded", "p2p", "p2p_gather", "ce", "adaptive", "nvls")
        multiple = align * self.ranks if sharded else None
        self.layout = BucketLayout.build([p.numel() for p in self.params], align, multiple=multiple)
        if sharded:
            if flat_params.numel() != self.layout.total or flat_params.dtype != torch.float32:
                raise ConfigError("flat parameter buffer does not match the sharded layout")
            base = flat_params.data_ptr()
            for p, off in zip(self.params, self.layout.offsets):
                if p.data_ptr() != base + 4 * off:
                    raise ConfigError("parameters are not views of the flat buffer at the layout offsets")
        n = len(self.params)
        lay = self.layout
        row_bytes = lay.bucket_bytes

        self.bucket = None
        self._peer_maps = []
        self._flags = None
        self.failed = False
        self.transport = None
        if mode == "nvls":
            from .nvls import NvlsBuffer, nvls_buffer_of

            self._flat_nvls = nvls_buffer_of(flat_params)
            if self._flat_nvls is None:
                raise ConfigError("nvls sync needs multicast-bound flat parameters "
                                  "(flatten_parameters(ipc='nvls'))")
            self._bucket_nvls = NvlsBuffer(lay.total, dev, comm.rank, self.ranks)
            self.bucket = self._bucket_nvls.tensor
        elif mode in ("p2p", "p2p_gather", "ce", "adaptive"):
            from .p2p import DeviceBuffer, buffer_of

            if self.ranks > _lib.CS_MAX_SOURCES:
                raise ConfigError(f"{mode} sync supports up to {_lib.CS_MAX_SOURCES} ranks")
            if buffer_of(flat_params) is None:
                raise ConfigError(f"{mode} sync needs IPC-capable flat parameters (flatten_parameters(ipc=True))")
            if mode != "p2p_gather":           # p2p_gather reads the gradients: no bucket
                self._bucket_buf = DeviceBuffer(lay.total, dev)
                self.bucket = self._bucket_buf.tensor
        elif mode in ("bucket", "sharded"):
            self.bucket = torch.zeros(self.local_workers * lay.total, dtype=torch.float32, device=dev)
        self.momentum_bufs = None
        self.shard = lay.total // self.ranks
        self.rank = comm.rank if comm is not None else 0
        if settings.momentum != 0:
            if sharded:   # momentum only for this rank's shard: S / W per GPU
                self.momentum_bufs = [torch.zeros(self.shard, dtype=torch.float32, device=dev)]
            else:
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
        if mode == "nvls":
            off = self.rank * self.shard * 4
            self._barrier = torch.zeros(32, dtype=torch.float32, device=dev)
            self._init_barrier(barrier)
            self._nvls = _lib.NvlsDesc()
            self._nvls.mc_bucket = self._bucket_nvls.mc_ptr + off
            self._nvls.mc_param = self._flat_nvls.mc_ptr + off
            self._nvls.param = flat_params.data_ptr() + off
            self._nvls.momentum_buf = self.momentum_bufs[0].data_ptr() if self.momentum_bufs else None
            self._nvls.numel = self.shard
            self._nvls.nranks = self.ranks
            self._nvls.max_ctas = int(p2p_ctas)
            self.transport = "nvls"
            self._finish_init(settings)
            return
        if mode == "p2p_gather":
            from .p2p import buffer_of, exchange_peer_addresses

            self._flat_map = exchange_peer_addresses(buffer_of(flat_params), self.rank, self.ranks)
            self._peer_maps = [self._flat_map]
            self._barrier = torch.zeros(32, dtype=torch.float32, device=dev)
            self._init_barrier(barrier)
            self._gather_ctas = int(p2p_ctas)
            self._gather = None               # built at the first sync, from its gradient tensors
            self._gather_keys = []
            self.transport = "p2p_gather"
            self._finish_init(settings)
            return
        if mode in ("p2p", "ce", "adaptive"):
            from .p2p import buffer_of, exchange_peer_addresses

            off = self.rank * self.shard * 4
            bmap = exchange_peer_addresses(self._bucket_buf, self.rank, self.ranks)
            fmap = exchange_peer_addresses(buffer_of(flat_params), self.rank, self.ranks)
            self._peer_maps = [bmap, fmap]
            self._barrier = torch.zeros(32, dtype=torch.float32, device=dev)
            self._init_barrier(barrier)
            if mode in ("p2p", "adaptive"):
                self._init_p2p(bmap, fmap, off, p2p_ctas)
            if mode in ("ce", "adaptive"):
                self._init_ce(bmap, fmap, off)
            # adaptive: both transports are built over the same bucket, flat parameters and
            # momentum shard (bitwise-identical arithmetic); the scheduler picks one per sync
            self.transport = "p2p" if mode == "p2p" else "ce"
            self._finish_init(settings)
            return
        if mode == "sharded":
            # one flat range: this rank's shard of the parameters, bucket and momentum
            off = self.rank * self.shard * 4
            self._upd = np.zeros(1, dtype=_lib.UPDATE_DESC)
            self._upd["param"] = flat_params.data_ptr() + off
            if self.momentum_bufs is not None:
                self._upd["momentum_buf"] = self.momentum_bufs[0].data_ptr()
            self._upd["grad_offset"] = off
            self._upd["snap_offset"] = off
            self._upd["numel"] = self.shard
            self._sources = np.asarray([self.bucket.data_ptr()], dtype=np.uint64)
            self._finish_init(settings)
            return
        self._upd = np.zeros(n, dtype=_lib.UPDATE_DESC)
        self._upd["param"] = [p.data_ptr() for p in self.params]
        if self.momentum_bufs is not None:
            self._upd["momentum_buf"] = [b.data_ptr() for b in self.momentum_bufs]
        self._upd["snap_offset"] = offs_bytes
        self._upd["numel"] = numels
        if mode == "unfused":
            self._sources = np.zeros(1, dtype=np.uint64)   # grad_offset = gradient pointer, per step
        elif mode == "bucket":
            self._upd["grad_offset"] = offs_bytes
            self._sources = np.asarray([self.bucket.data_ptr() + w * row_bytes
                                        for w in range(self.local_workers)], dtype=np.uint64)
        elif mode == "direct":
            self._sources = np.zeros(1, dtype=np.uint64)
        self._finish_init(settings)

    def _init_barrier(self, barrier: str) -> None:
        """Cross-rank barriers of the p2p / ce transports: SM-free stream-memory-op flags
        (cs_flag_barrier) when every rank supports them ("auto" / "flags"), else a 1-element
        NCCL all-reduce ("nccl").  The NCCL barrier's kernel needs a free SM, which it may wait
        for while the other app's GEMMs hold every SM; the flag barrier runs in the GPU front end."""
        from .p2p import FlagArray, all_ranks_agree

        if barrier not in ("auto", "flags", "nccl"):
            raise ConfigError(f"unknown barrier {barrier!r}")
        self._flag_peers = None
        self._flags = None
        self._barrier_kind = "nccl"
        nccl = getattr(self.comm, "has_collectives", True)
        if barrier == "nccl":
            if not nccl:
                raise ConfigError("the NCCL barrier needs an NcclCommunicator")
            return
        supported = bool(_lib.lib.cs_stream_memops_supported())
        if not all_ranks_agree(supported):
            if barrier == "flags" or not nccl:
                raise ConfigError("stream memory operations are not supported on every rank")
            return
        try:
            self._flags = FlagArray(self.rank, self.ranks)  # host shared memory, zeroed
        except ConfigError:
            # the segment failed on some rank (every rank raises together): the NCCL barrier
            # still works where there is a communicator
            if barrier == "flags" or not nccl:
                raise
            return
        self._flag_peers = self._flags.peer_rows               # per phase
        self._flag_local = self._flags.local_rows
        self._barrier_kind = "flags"

    def _rank_barrier(self, stream: int, phase: int) -> None:
        """Barrier `phase` (0: every rank's K1 landed; 1: every shard updated and every bucket
        read) of one sync.  The flag protocol is constant-valued and self-resetting (graph-safe)."""
        if self._flag_peers is None:
            self.comm.all_reduce_(self._barrier.data_ptr(), 1, stream)
            return
        peers = self._flag_peers[phase]
        _lib.check("cs_flag_barrier", _lib.lib.cs_flag_barrier(
            peers.ctypes.data, self._flag_local[phase], self.rank, self.ranks, stream))

    @property
    def barrier_kind(self) -> str | None:
        if self.mode not in ("p2p", "p2p_gather", "ce", "adaptive", "nvls"):
            return None
        return self._barrier_kind

    def set_transport(self, transport: str) -> None:
        """Pick the NVLink transport of the next syncs (adaptive mode switches freely: both
        transports sum the W shards in rank order with the same update rule)."""
        allowed = {"p2p": ("p2p",), "ce": ("ce",), "adaptive": ("p2p", "ce")}.get(self.mode, ())
        if transport not in allowed:
            raise ConfigError(f"transport {transport!r} is not available in {self.mode!r} mode")
        self.transport = transport

    def _init_p2p(self, bmap, fmap, off: int, p2p_ctas: int) -> None:
        self._p2p = _lib.P2PDesc()
        for r in range(self.ranks):
            # sources in rank order: the sum order is the reference's (rotating the destination
            # order measured no difference, tools/c1bench.py: thousands of threads interleave)
            self._p2p.src[r] = bmap.addresses[r] + off
            self._p2p.dst[r] = fmap.addresses[r] + off
        self._p2p.param = self.flat.data_ptr() + off
        self._p2p.momentum_buf = self.momentum_bufs[0].data_ptr() if self.momentum_bufs else None
        self._p2p.numel = self.shard
        self._p2p.nranks = self.ranks
        self._p2p.max_ctas = int(p2p_ctas)

    def _init_ce(self, bmap, fmap, off: int) -> None:
        """Copy-engine transport: pull every peer's copy of my bucket shard (reduce-scatter half),
        K2 over the W shard copies in rank order, pull every peer's updated parameter shard
        (all-gather half).  No SM moves a byte across NVLink."""
        sb = self.shard * 4
        self._recv = torch.empty(self.layout.total, dtype=torch.float32, device=self.flat.device)
        # rank r pulls from r+1, r+2, ... (mod W): at every moment each GPU serves exactly one
        # reader; pulling in rank order would make every rank read rank 0 first (one hot source)
        peers = [(self.rank + k) % self.ranks for k in range(1, self.ranks)]
        self._ce_rs = [(self._recv.data_ptr() + s * sb, bmap.addresses[s] + off) for s in peers]
        f = self.flat.data_ptr()
        self._ce_ag = [(f + s * sb, fmap.addresses[s] + s * sb) for s in peers]
        self._upd = np.zeros(1, dtype=_lib.UPDATE_DESC)
        self._upd["param"] = f + off
        if self.momentum_bufs is not None:
            self._upd["momentum_buf"] = self.momentum_bufs[0].data_ptr()
        self._upd["numel"] = self.shard
        self._sources = np.asarray([self.bucket.data_ptr() + off if s == self.rank
                                    else self._recv.data_ptr() + s * sb
                                    for s in range(self.ranks)], dtype=np.uint64)

    def _finish_init(self, settings: SgdSettings) -> None:
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
        if self.mode not in ("bucket", "sharded", "p2p", "ce", "adaptive", "nvls"):
            raise ConfigError("pack() needs bucket mode")
        n = len(self.params)
        if len(grads_per_worker) != self.local_workers:
            raise ValueError(f"expected gradients of {self.local_workers} worker(s)")
        for w, grads in enumerate(grads_per_worker):
            self._pack["src"][w * n:(w + 1) * n] = _grad_ptrs(grads, self.params)
        if self.pack_engine == "ce":
            # the copy engines gather the gradients (one DMA per tensor, no SM): for apps with few
            # large tensors whose sync overlaps tensor-core compute that would lose the SMs
            for d in self._pack:
                if d["numel"]:
                    _lib.check("cs_copy_async", _lib.lib.cs_copy_async(
                        int(d["dst"]), int(d["src"]), int(d["numel"]) * 4, stream))
            return
        _lib.pack(self._pack, stream, self.sync_ctas)
        self.kernel_launches += 1

    def all_reduce(self, stream: int) -> None:
        """C1: in-place NCCL sum of the bucket across ranks (no-op at world 1)."""
        if self.comm is not None and self.comm.active:
            self.comm.all_reduce_(self.bucket.data_ptr(), self.layout.total, stream)

    def update(self, stream: int, grads: Sequence[torch.Tensor] | None = None,
               snapshot_row: int | None = None) -> None:
        """K2: reduce the source rows left to right, / W, SGD step in place."""
        if self.mode in ("direct", "unfused"):
            if grads is None:
                raise ValueError("direct mode needs the gradient tensors")
            self._upd["grad_offset"] = _grad_ptrs(grads, self.params)
        snap = 0
        if snapshot_row is not None and self.mode not in ("sharded", "ce", "adaptive"):
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            snap = self.snapshot[snapshot_row].data_ptr()
        self._hyper.first_step = int(self.first_step)
        _lib.unpack_sgd(self._upd, self._sources, snap, self._hyper, stream, self.sync_ctas)
        self.first_step = False
        self.kernel_launches += 1

    def sync(self, grads_per_worker: Sequence[Sequence[torch.Tensor]], stream: int,
             snapshot_row: int | None = None, timer=None) -> None:
        """The whole sync phase of one iteration: K1 -> C1 -> K2 (or K2 alone in direct mode)."""
        if self.mode == "unfused":
            # per-tensor counterfactual (workload.unfused_messages, workload.py:104-110): one
            # collective per gradient tensor, each paying the per-message latency
            grads = grads_per_worker[0]
            ptrs = _grad_ptrs(grads, self.params)
            if timer is not None:
                timer.begin("c1_unfused")
            if self.comm is not None and self.comm.active:
                for ptr, n in zip(ptrs, self.layout.numels):
                    if n:
                        self.comm.all_reduce_(ptr, n, stream)
            if timer is not None:
                timer.end("c1_unfused")
                timer.begin("k2_update")
            self.update(stream, grads, snapshot_row)
            if timer is not None:
                timer.end("k2_update")
            return
        if self.mode == "direct":
            if timer is not None:
                timer.begin("k2_update")
            self.update(stream, grads_per_worker[0], snapshot_row)
            if timer is not None:
                timer.end("k2_update")
            return
        if self.transport == "p2p_gather":
            self._gather_tail(grads_per_worker[0], stream, snapshot_row, timer)
            return
        if timer is not None:
            timer.begin("k1_pack")
        self.pack(grads_per_worker, stream)
        if timer is not None:
            timer.end("k1_pack")
        if self.mode == "sharded":
            self._sharded_tail(stream, snapshot_row, timer)
            return
        if self.transport == "nvls":
            self._nvls_tail(stream, snapshot_row, timer)
            return
        if self.transport == "p2p":
            self._p2p_tail(stream, snapshot_row, timer)
            return
        if self.transport == "ce":
            self._ce_tail(stream, snapshot_row, timer)
            return
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

    def sync_packed(self, stream: int) -> None:
        """The sync phase after K1 already ran (graph mode packs on the compute stream right after
        the backward): C1 -> K2 from the bucket (bucket), RS -> K2 -> AG (sharded), or the peer
        transports' barrier / exchange / update / barrier (p2p, ce)."""
        if self.mode == "sharded":
            self._sharded_tail(stream, None, None)
        elif self.transport == "p2p":
            self._p2p_tail(stream, None, None)
        elif self.transport == "nvls":
            self._nvls_tail(stream, None, None)
        elif self.transport == "ce":
            self._ce_tail(stream, None, None)
        elif self.mode == "bucket":
            self.all_reduce(stream)
            self.update(stream, None, None)
        else:
            raise ConfigError(f"sync_packed has no {self.mode!r} path (direct / unfused read the gradients)")

    def _sharded_tail(self, stream: int, snapshot_row: int | None, timer) -> None:
        """reduce-scatter -> K2 on this rank's shard -> all-gather into the flat parameters."""
        shard_bytes = self.shard * 4
        b = self.bucket.data_ptr()
        if timer is not None:
            timer.begin("c1_reduce_scatter")
        self.comm.reduce_scatter(b, b + self.rank * shard_bytes, self.shard, stream)
        if timer is not None:
            timer.end("c1_reduce_scatter")
            timer.begin("k2_update")
        self.update(stream, None, None)
        if timer is not None:
            timer.end("k2_update")
            timer.begin("c1_all_gather")
        f = self.flat.data_ptr()
        self.comm.all_gather(f + self.rank * shard_bytes, f, self.shard, stream)
        if timer is not None:
            timer.end("c1_all_gather")
        if snapshot_row is not None:
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self.snapshot[snapshot_row].copy_(self.flat)

    def _p2p_tail(self, stream: int, snapshot_row: int | None, timer) -> None:
        """barrier -> fused reduce + update + all-gather over NVLink -> barrier."""
        self._rank_barrier(stream, 0)                  # every rank's K1 has landed
        if timer is not None:
            timer.begin("k2_p2p_fused")
        self._hyper.first_step = int(self.first_step)
        _lib.check("cs_p2p_reduce_sgd_bcast", _lib.lib.cs_p2p_reduce_sgd_bcast(
            ctypes.byref(self._p2p), ctypes.byref(self._hyper), stream))
        self.first_step = False
        self.kernel_launches += 1
        if timer is not None:
            timer.end("k2_p2p_fused")
        self._rank_barrier(stream, 1)                  # every rank's parameter writes landed
        if snapshot_row is not None:
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self.snapshot[snapshot_row].copy_(self.flat)

    def _gather_plan(self, grads: Sequence[torch.Tensor]) -> None:
        """Chunks of this rank's shard -- none crossing a gradient tensor -- with every rank's
        gradient addresses (collective: map_peer_tensors), uploaded once; the gradients must keep
        these addresses for every later sync.  Runs inside the app's first sync (the addresses
        exist only after the first backward), so that one step pays a host round trip for the
        handle exchange and the table upload; every later step is asynchronous."""
        from .p2p import map_peer_tensors

        if len(grads) != len(self.params):
            raise ValueError(f"expected {len(self.params)} gradients")
        for i, (g, p) in enumerate(zip(grads, self.params)):
            if (g is None or g.dtype != torch.float32 or g.shape != p.shape or g.stride() != p.stride()
                    or not _dense(g) or g.data_ptr() % 16):
                raise ConfigError(f"p2p_gather: gradient {i} must be a dense fp32 tensor laid out like its "
                                  "parameter, 16-byte aligned")
        addrs, self._gather_keys = map_peer_tensors(grads, self.rank, self.ranks, self.flat.device)
        lay = self.layout
        s0, s1 = self.rank * self.shard, (self.rank + 1) * self.shard
        ch = int(_lib.lib.cs_p2p_gather_chunk_elems(self.ranks))
        flat = self._flat_map.addresses
        mom = self.momentum_bufs[0].data_ptr() if self.momentum_bufs else 0
        rows = []
        for i, o, a, b in gather_chunks(lay.offsets, lay.numels, s0, s1, ch):
            row = np.zeros((), dtype=_lib.P2P_DESC)
            row["src"][:self.ranks] = [addrs[r][i] + 4 * (a - o) for r in range(self.ranks)]
            row["dst"][:self.ranks] = [flat[r] + 4 * a for r in range(self.ranks)]
            row["param"] = self.flat.data_ptr() + 4 * a
            row["momentum_buf"] = mom + 4 * (a - s0) if mom else 0
            row["numel"] = b - a
            row["nranks"] = self.ranks
            rows.append(row)
        table = np.array(rows, dtype=_lib.P2P_DESC)
        _lib.check("cs_p2p_gather_check", _lib.lib.cs_p2p_gather_check(
            table.ctypes.data, len(table), self.ranks, int(bool(mom))))
        self._gather = (torch.from_numpy(table.view(np.uint8).copy()).to(self.flat.device), len(table))
        self._gather_ptrs = [g.data_ptr() for g in grads]

    def _gather_tail(self, grads: Sequence[torch.Tensor], stream: int, snapshot_row: int | None, timer) -> None:
        """barrier -> one NVLink kernel over every rank's gradient tensors (rank-order reduce, /W,
        SGD, broadcast writes of the new shard) -> barrier.  No K1, no bucket."""
        if self._gather is None:
            self._gather_plan(grads)
        elif [g.data_ptr() for g in grads] != self._gather_ptrs:
            raise ConfigError("p2p_gather: the gradients moved since the first sync (the transport "
                              "needs a CUDA-graphed backward with static gradient buffers)")
        self._rank_barrier(stream, 0)                  # every rank's gradients are complete
        if timer is not None:
            timer.begin("k2_p2p_gather")
        self._hyper.first_step = int(self.first_step)
        table, n = self._gather
        _lib.check("cs_p2p_gather_reduce_sgd_bcast", _lib.lib.cs_p2p_gather_reduce_sgd_bcast(
            table.data_ptr(), n, self.ranks, self._gather_ctas, ctypes.byref(self._hyper), stream))
        self.first_step = False
        self.kernel_launches += 1
        if timer is not None:
            timer.end("k2_p2p_gather")
        self._rank_barrier(stream, 1)                  # every peer read my gradients, wrote my shard
        if snapshot_row is not None:
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self.snapshot[snapshot_row].copy_(self.flat)

    def _nvls_tail(self, stream: int, snapshot_row: int | None, timer) -> None:
        """barrier -> one kernel: switch-reduced shard (multimem.ld_reduce), /W, SGD, switch-broadcast
        new shard (multimem.st) -> barrier."""
        self._rank_barrier(stream, 0)                  # every rank's K1 has landed
        if timer is not None:
            timer.begin("k2_nvls_fused")
        self._hyper.first_step = int(self.first_step)
        _lib.check("cs_nvls_reduce_sgd_bcast", _lib.lib.cs_nvls_reduce_sgd_bcast(
            ctypes.byref(self._nvls), ctypes.byref(self._hyper), stream))
        self.first_step = False
        self.kernel_launches += 1
        if timer is not None:
            timer.end("k2_nvls_fused")
        self._rank_barrier(stream, 1)                  # every rank's multicast stores landed
        if snapshot_row is not None:
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self.snapshot[snapshot_row].copy_(self.flat)

    def _ce_copies(self, pairs, stream: int) -> None:
        nbytes = self.shard * 4
        for dst, src in pairs:
            _lib.check("cs_copy_async", _lib.lib.cs_copy_async(dst, src, nbytes, stream))

    def _ce_tail(self, stream: int, snapshot_row: int | None, timer) -> None:
        """barrier -> CE pulls of my shard from every peer -> K2 (rank-order sum, /W, SGD) on the
        shard -> barrier -> CE pulls of every peer's updated shard into the flat parameters.

        The second barrier orders three things: every rank's shard is updated before anyone
        pulls it, every peer has finished reading my bucket before my next K1 rewrites it, and
        (by stream order on each peer) a peer's all-gather pulls of iteration t complete before
        it enters iteration t+1's first barrier, so my K2 at t+1 never races them."""
        self._rank_barrier(stream, 0)                  # every rank's K1 has landed
        if timer is not None:
            timer.begin("c1_ce_reduce_scatter")
        self._ce_copies(self._ce_rs, stream)
        if timer is not None:
            timer.end("c1_ce_reduce_scatter")
            timer.begin("k2_update")
        self.update(stream, None, None)
        if timer is not None:
            timer.end("k2_update")
        self._rank_barrier(stream, 1)                  # every shard updated, every bucket read
        if timer is not None:
            timer.begin("c1_ce_all_gather")
        self._ce_copies(self._ce_ag, stream)
        if timer is not None:
            timer.end("c1_ce_all_gather")
        if snapshot_row is not None:
            if self.snapshot is None:
                raise ConfigError("no snapshot buffer (snapshot_rows=0)")
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self.snapshot[snapshot_row].copy_(self.flat)

    def release_waits(self) -> None:
        """Failure path: satisfy every pending flag-barrier wait of every rank (host writes into
        the shared flag segment, no GPU work), so no comm stream stays blocked behind a peer that
        stopped.  Each released wait resets its row, so the caller repeats this until the device
        drained.  The transport is unusable afterwards."""
        if self._flags is not None:
            self._flags.release()
            self.failed = True

    def close(self) -> None:
        """Unmap the peers' buffers, then free this app's IPC bucket and flag segment.  At W > 1
        this is collective (every rank unmaps before any rank frees) unless the sync failed."""
        for m in self._peer_maps:
            m.close()
        self._peer_maps = []
        if getattr(self, "_gather_keys", None):
            from .p2p import unmap_peer_tensors

            unmap_peer_tensors(self._gather_keys)
            self._gather_keys = []
        bucket = getattr(self, "_bucket_buf", None) or getattr(self, "_bucket_nvls", None)
        if bucket is None and self._flags is None:
            return
        if self.ranks > 1 and not self.failed:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.barrier()
        if bucket is not None:
            self.bucket = None
            bucket.close()
            self._bucket_buf = self._bucket_nvls = None
        if self._flags is not None:
            self._flags.close()
            self._flags = None
            self._flag_peers = None

    # -- algorithmic bytes per launch ---------------------------
    def k1_bytes(self) -> int:
        if self.mode == "p2p_gather":
            return 0                       # no pack: the kernel reads the gradients in place
        return 2 * self.local_workers * self.layout.payload_bytes

    def k2_bytes(self, transport: str | None = None) -> int:
        transport = transport or self.transport
        if transport == "nvls":
            # local HBM: read p (+ momentum r/w); the reduced shard arrives from and the new shard
            # leaves through the switch
            return (1 + (2 if self.settings.momentum else 0)) * self.shard * 4
        if transport in ("p2p", "p2p_gather"):
            # W source shards + p read + W destination shards (+ momentum read/write)
            return (2 * self.ranks + 1 + (2 if self.settings.momentum else 0)) * self.shard * 4
        if self.mode == "sharded":
            return (5 if self.settings.momentum else 3) * self.shard * 4
        if transport == "ce":
            # W source shards + p read/write (+ momentum read/write)
            return (self.ranks + 2 + (2 if self.settings.momentum else 0)) * self.shard * 4
        s = self.layout.payload_bytes
        streams = self.local_workers if self.mode == "bucket" else 1
        per = (streams + 2) * s            # read sources + read p + write p
        if self.settings.momentum:
            per += 2 * s                   # read + write the momentum buffer
        return per

    def nvls_link_bytes(self) -> int:
        """Bytes through each GPU's NVLink ports per direction for one nvls sync: the switch reads
        every member's copy of every rank's shard (W shards out, the local copy included) and fans
        each rank's new shard out to every member (W shards in), plus the reduced shard back to
        the issuer and the issuer's own stores: (W + 1) shards each way."""
        return (self.ranks + 1) * self.shard * 4

    def c1_bus_bytes(self) -> float:
        """All-reduce bus bytes 2(W-1)/W * S (== reduce-scatter + all-gather in sharded mode)."""
        w = self.ranks
        return 0.0 if w <= 1 else 2.0 * (w - 1) / w * self.layout.bucket_bytes


def gather_chunks(offsets: Sequence[int], numels: Sequence[int], s0: int, s1: int, ch: int):
    """The p2p_gather work list of the shard [s0, s1) of a bucket layout: (tensor index, tensor
    offset, a, b) for every chunk [a, b) -- inside one tensor and the shard, at most `ch` elements,
    in bucket order; the padding between tensors is not covered (it holds no gradient)."""
    for i, (o, n) in enumerate(zip(offsets, numels)):
        for a in range(max(o, s0), min(o + n, s1), ch):
            yield i, o, a, min(a + ch, o + n, s1)


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
                # the copy runs on the current (comm) stream while `g` was allocated on the
                # compute stream: record the use, or the caching allocator could hand g's
                # memory to the next app's forward before the queued copy has read it
                g.record_stream(torch.cuda.current_stream(g.device))
                fixed = torch.empty_like(p)
                fixed.copy_(g)
                g = fixed
                if isinstance(grads, list):
                    grads[i] = fixed  # keep it alive as long as the caller holds the list
        out.append(g.data_ptr())
    return out
