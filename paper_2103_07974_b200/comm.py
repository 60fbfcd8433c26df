"""Bucket synchronization: the measured NCCL collective plus the reference's predictor.

Reference: colosim.comm (comm.py:39-135).  There the synchronization is only
*priced*: ring all-reduce ``2(W-1)a + ceil(2(W-1) S 1e9 / (W B))`` ns.  Here it
is executed: :class:`NcclCommunicator` runs ``ncclAllReduce`` (sum, fp32) of a
job's fused bucket on the caller's comm stream through libcrossover.so, and
the alpha-beta formula is kept as the *predictor* of the comm/comp ratio and
as the NVLink roofline (bus bytes = 2(W-1)/W * S, nccl-tests convention).

The parameter-server architecture (comm.py:102-110) is out of scope: one
NVSwitch box has no parameter server and the north star names all-reduce only.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum
from fractions import Fraction
from typing import Iterable

from .errors import ConfigError
from .workload import FusedGradient, JobProfile, comp_time, fuse_gradients

__all__ = [
    "Architecture",
    "comm_time_ps",
    "ClusterSpec",
    "SyncRequest",
    "comm_time_allreduce",
    "comm_time",
    "comm_time_unfused",
    "comm_comp_ratio",
    "allreduce_bus_bytes",
    "NcclCommunicator",
    "PeerGroup",
    "NVLINK5_GBPS",
]

NS_PER_S = 10**9
NVLINK5_GBPS = 900.0  # per direction per GPU, nominal


class Architecture(Enum):
    """Predictor topologies (comm.py:39-41).  The device always syncs over NVLink collectives;
    ``parameter_server`` exists so the reference's scenario files price the same way."""

    PARAMETER_SERVER = "parameter_server"
    RING_ALLREDUCE = "ring_allreduce"


@dataclass(frozen=True)
class ClusterSpec:
    """Cluster description for the predictor (comm.py:44-71)."""

    workers: int
    bandwidth_bytes_per_sec: int
    latency_per_message: int = 0
    architecture: Architecture = Architecture.RING_ALLREDUCE
    gpus_per_worker: int = 1
    ps_servers: int = 1

    def __post_init__(self):
        if not isinstance(self.architecture, Architecture):
            raise ConfigError(f"cluster.architecture: {self.architecture!r} is not an Architecture")
        if self.workers < 1:
            raise ConfigError("cluster.workers must be >= 1")
        if self.gpus_per_worker < 1:
            raise ConfigError("cluster.gpus_per_worker must be >= 1")
        if self.bandwidth_bytes_per_sec <= 0:
            raise ConfigError("cluster.bandwidth must be > 0")
        if self.latency_per_message < 0:
            raise ConfigError("cluster.latency must be >= 0")
        if self.architecture is Architecture.PARAMETER_SERVER and self.ps_servers < 1:
            raise ConfigError("cluster.ps_servers must be >= 1 for parameter_server")

    @staticmethod
    def nvswitch(workers: int, busbw_gbps: float = 725.0, latency_ns: int = 10_000) -> "ClusterSpec":
        """Calibrated B200 NVSwitch box: 725 GB/s is the measured 8-rank all-reduce busbw."""
        return ClusterSpec(workers, int(busbw_gbps * 1e9), latency_ns)


@dataclass(frozen=True)
class SyncRequest:
    """One outstanding synchronization (comm.py:74-80)."""

    job_id: str
    iteration: int
    payload: FusedGradient


def comm_time_allreduce(size_bytes: int, cluster: ClusterSpec) -> int:
    """Ring all-reduce duration, integer ns with ceiling rounding; 0 at W=1 (comm.py:87-99)."""
    if cluster.architecture is not Architecture.RING_ALLREDUCE:
        raise ConfigError("comm_time_allreduce requires architecture=ring_allreduce")
    if size_bytes < 0:
        raise ValueError("size_bytes must be >= 0")
    w = cluster.workers
    if w == 1:
        return 0
    num = 2 * (w - 1) * size_bytes * NS_PER_S
    den = w * cluster.bandwidth_bytes_per_sec
    return 2 * (w - 1) * cluster.latency_per_message + (num + den - 1) // den


def comm_time_ps(size_bytes: int, cluster: ClusterSpec) -> int:
    """Parameter-server push + pull through the worker NIC, integer ns, ceiling (comm.py:102-110)."""
    if cluster.architecture is not Architecture.PARAMETER_SERVER:
        raise ConfigError("comm_time_ps requires architecture=parameter_server")
    if size_bytes < 0:
        raise ValueError("size_bytes must be >= 0")
    den = cluster.bandwidth_bytes_per_sec
    return 2 * cluster.latency_per_message + (2 * size_bytes * NS_PER_S + den - 1) // den


def _priced(size_bytes: int, cluster: ClusterSpec) -> int:
    if cluster.architecture is Architecture.PARAMETER_SERVER:
        return comm_time_ps(size_bytes, cluster)
    return comm_time_allreduce(size_bytes, cluster)


def comm_time(request: SyncRequest, cluster: ClusterSpec) -> int:
    """One sync under the cluster's architecture (comm.py:119-121)."""
    return _priced(request.payload.size_bytes, cluster)


def comm_time_unfused(messages: Iterable[FusedGradient], cluster: ClusterSpec) -> int:
    """Per-tensor messages each pay the latency term (comm.py:124-126)."""
    return sum(_priced(m.size_bytes, cluster) for m in messages)


def comm_comp_ratio(job: JobProfile, cluster: ClusterSpec) -> Fraction:
    """rho = sync / compute for one iteration (comm.py:129-135)."""
    comp = comp_time(job)
    if comp <= 0:
        raise ValueError(f"job {job.job_id!r}: compute time must be > 0")
    return Fraction(comm_time(SyncRequest(job.job_id, 1, fuse_gradients(job, 1)), cluster), comp)


def allreduce_bus_bytes(size_bytes: int, world: int) -> float:
    """Bytes each GPU moves over NVLink for a ring all-reduce: 2(W-1)/W * S."""
    return 0.0 if world <= 1 else 2.0 * (world - 1) / world * size_bytes


class NcclCommunicator:
    """One NCCL communicator per process over NVLink/NVSwitch (libcrossover.so C1).

    The unique id is created on rank 0 and broadcast with torch.distributed
    (any backend; only the rendezvous uses it).  All collectives are enqueued
    on the stream passed in; nothing here blocks the host.
    """

    def __init__(self, rank: int, world: int, min_ctas: int = 0, max_ctas: int = 0):
        from . import _lib

        self._lib = _lib
        self.rank = rank
        self.world = world
        self.handle = ctypes.c_void_p(None)
        if world == 1:
            return
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ConfigError("world > 1 needs torch.distributed initialised for the NCCL rendezvous")
        uid = (ctypes.c_uint8 * _lib.CS_NCCL_UNIQUE_ID_BYTES)()
        if rank == 0:
            _lib.check("cs_nccl_get_unique_id", _lib.lib.cs_nccl_get_unique_id(uid))
        payload = [bytes(uid) if rank == 0 else None]
        dist.broadcast_object_list(payload, src=0)
        uid = (ctypes.c_uint8 * _lib.CS_NCCL_UNIQUE_ID_BYTES).from_buffer_copy(payload[0])
        _lib.check("cs_nccl_init", _lib.lib.cs_nccl_init(
            ctypes.byref(self.handle), world, rank, uid, min_ctas, max_ctas))

    has_collectives = True

    @property
    def active(self) -> bool:
        return self.world > 1

    def all_reduce_(self, ptr: int, count: int, stream: int) -> None:
        """In-place sum of `count` fp32 elements at device address `ptr`."""
        if self.world == 1:
            return
        self._lib.check("cs_nccl_allreduce_sum_f32", self._lib.lib.cs_nccl_allreduce_sum_f32(
            self.handle, ptr, ptr, count, stream))

    def reduce_scatter(self, send: int, recv: int, recv_count: int, stream: int) -> None:
        self._lib.check("cs_nccl_reduce_scatter_sum_f32", self._lib.lib.cs_nccl_reduce_scatter_sum_f32(
            self.handle, send, recv, recv_count, stream))

    def all_gather(self, send: int, recv: int, send_count: int, stream: int) -> None:
        self._lib.check("cs_nccl_all_gather_f32", self._lib.lib.cs_nccl_all_gather_f32(
            self.handle, send, recv, send_count, stream))

    def check_async_error(self) -> None:
        if self.world > 1:
            self._lib.check("cs_nccl_async_error", self._lib.lib.cs_nccl_async_error(self.handle))

    def abort(self) -> None:
        """Abort the communicator (unblocks kernels stuck waiting for a dead peer)."""
        if self.world > 1 and self.handle:
            self._lib.lib.cs_nccl_abort(self.handle)
            self.handle = ctypes.c_void_p(None)

    def close(self) -> None:
        if self.world > 1 and self.handle:
            self._lib.check("cs_nccl_destroy", self._lib.lib.cs_nccl_destroy(self.handle))
            self.handle = ctypes.c_void_p(None)


class PeerGroup:
    """The ranks of the peer-memory transports without an NCCL communicator.

    The ``p2p`` and ``ce`` syncs move every byte themselves (NVLink loads / stores or copy-engine
    pulls from IPC-mapped peer buffers) and order the ranks with SM-free flag barriers, so they need
    only the process group's rank and size -- torch.distributed (any backend) for the one-off
    exchange of IPC handles.  This is also what lets W ranks share ONE GPU (NCCL refuses two ranks
    on a device): CUDA IPC and stream memory operations work between processes on the same device,
    which is how the W > 1 data plane is parity-tested on a single B200.
    """

    has_collectives = False

    def __init__(self, rank: int, world: int):
        if world < 1 or not 0 <= rank < world:
            raise ConfigError(f"invalid rank {rank} of world {world}")
        if world > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                raise ConfigError("world > 1 needs torch.distributed initialised for the handle exchange")
        self.rank = rank
        self.world = world
        self.handle = None

    @property
    def active(self) -> bool:
        return False      # no collectives: the bucket all-reduce path is unavailable

    def _no_collectives(self, *_args) -> None:
        raise ConfigError("this sync mode needs an NCCL communicator (PeerGroup serves p2p / ce only)")

    all_reduce_ = reduce_scatter = all_gather = _no_collectives

    def check_async_error(self) -> None:
        pass

    def abort(self) -> None:
        pass

    def close(self) -> None:
        pass
