"""IPC-capable device buffers and their peer mapping over NVLink (for the fused P2P sync).

The collective-fused update (``cs_p2p_reduce_sgd_bcast``) reads every rank's bucket
shard and writes every rank's parameter shard directly through NVLink, so those two
buffers must be mappable into every process: they are allocated with
``cs_device_alloc`` (plain cudaMalloc) instead of the torch caching allocator, exposed
to torch zero-copy through ``__cuda_array_interface__``, and opened in the peers with
``cudaIpcOpenMemHandle`` (handles travel over torch.distributed's object collectives).
"""

from __future__ import annotations

import ctypes
import weakref

import torch

from . import _lib

__all__ = ["DeviceBuffer", "exchange_peer_addresses", "PeerMapping", "all_ranks_agree", "FlagArray",
           "map_peer_tensors", "unmap_peer_tensors"]

# ptr -> DeviceBuffer, weakly: a buffer lives exactly as long as a tensor viewing it (torch keeps
# the __cuda_array_interface__ provider alive as the storage's owner), then cudaFree runs
_live: "weakref.WeakValueDictionary[int, DeviceBuffer]" = weakref.WeakValueDictionary()


class DeviceBuffer:
    """A zero-filled fp32 cudaMalloc allocation shown to torch as a 1-D tensor.

    Ownership: the tensor owns the buffer (the buffer only keeps a weak reference back), so
    dropping every view frees the memory; :meth:`close` frees it explicitly (after which the
    tensor must not be used)."""

    def __init__(self, numel: int, device: torch.device):
        if numel <= 0:
            raise ValueError("numel must be > 0")
        ptr = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check("cs_device_alloc", _lib.lib.cs_device_alloc(numel * 4, ctypes.byref(ptr)))
        self.ptr = int(ptr.value)
        self.numel = int(numel)
        self.device = torch.device(device)
        self.__cuda_array_interface__ = {"shape": (self.numel,), "typestr": "<f4",
                                         "data": (self.ptr, False), "version": 3, "strides": None}
        t = torch.as_tensor(self, device=self.device)
        assert t.data_ptr() == self.ptr
        self._tensor = weakref.ref(t)
        self._first = t          # handed to the creator by the first .tensor access
        _live[self.ptr] = self

    @property
    def tensor(self) -> torch.Tensor:
        first, self._first = self._first, None
        t = first if first is not None else self._tensor()
        if t is None:
            raise RuntimeError("DeviceBuffer: every tensor view was dropped")
        return t

    def ipc_handle(self) -> bytes:
        out = (ctypes.c_uint8 * _lib.CS_IPC_HANDLE_BYTES)()
        _lib.check("cs_ipc_get_handle", _lib.lib.cs_ipc_get_handle(self.ptr, out))
        return bytes(out)

    def close(self) -> None:
        if self.ptr:
            _live.pop(self.ptr, None)
            self._first = None
            _lib.check("cs_device_free", _lib.lib.cs_device_free(self.ptr))
            self.ptr = 0

    def __del__(self):
        if getattr(self, "ptr", 0):
            try:
                _lib.lib.cs_device_free(self.ptr)
            except Exception:   # interpreter shutdown: the context may already be gone
                pass
            self.ptr = 0


def buffer_of(t: torch.Tensor) -> DeviceBuffer | None:
    """The DeviceBuffer whose base is exactly t's storage start, if any."""
    return _live.get(t.data_ptr())


class PeerMapping:
    """Addresses of one buffer in every rank, as seen from this process."""

    def __init__(self, addresses: list[int], opened: list[int]):
        self.addresses = addresses
        self._opened = opened

    def close(self) -> None:
        for p in self._opened:
            _lib.check("cs_ipc_close_handle", _lib.lib.cs_ipc_close_handle(p))
        self._opened = []


def exchange_peer_addresses(buf: DeviceBuffer, rank: int, world: int) -> PeerMapping:
    """All-gather IPC handles and open every peer's buffer (collective over torch.distributed).

    Failure is agreed on collectively: if any rank cannot map any peer, every rank closes what
    it opened and raises ConfigError -- no rank is left waiting in a later collective.
    """
    import torch.distributed as dist

    from .errors import ConfigError

    handles: list = [None] * world
    dist.all_gather_object(handles, buf.ipc_handle())
    addrs, opened, error = [], [], ""
    with torch.cuda.device(buf.device):
        for r in range(world):
            if r == rank:
                addrs.append(buf.ptr)
                continue
            h = (ctypes.c_uint8 * _lib.CS_IPC_HANDLE_BYTES).from_buffer_copy(handles[r])
            p = ctypes.c_void_p()
            rc = _lib.lib.cs_ipc_open_handle(h, ctypes.byref(p))
            if rc:
                error = f"rank {rank}: cannot map rank {r}: {_lib.lib.cs_last_error().decode()}"
                break
            addrs.append(int(p.value))
            opened.append(int(p.value))
    mapping = PeerMapping(addrs, opened)
    if not all_ranks_agree(not error):
        mapping.close()
        raise ConfigError("p2p peer mapping failed on some rank" + (f" ({error})" if error else ""))
    return mapping


# (peer rank, peer allocation base) -> [address here, users]: one mapping per peer allocation and
# process however many syncs read tensors inside it (CUDA maps an allocation once per context)
_peer_allocs: dict[tuple[int, int], list] = {}


def map_peer_tensors(tensors, rank: int, world: int, device) -> tuple[list[list[int]], list[tuple[int, int]]]:
    """Addresses of every rank's `tensors` (same count and order on every rank) as seen from this
    process -- the p2p_gather transport reads the gradient tensors of the peers in place.

    Each tensor's IPC handle is its allocation's (cs_ipc_base_of: a caching-allocator segment) plus
    its offset in it.  Collective over torch.distributed; a failure anywhere is agreed on, every rank
    releases what it mapped and raises ConfigError.  Returns (addresses[rank][i], keys to release
    with unmap_peer_tensors)."""
    import torch.distributed as dist

    from .errors import ConfigError

    bases: dict[int, int] = {}
    mine, error = [], ""
    for t in tensors:
        base, size = ctypes.c_void_p(), ctypes.c_size_t()
        if _lib.lib.cs_ipc_base_of(t.data_ptr(), ctypes.byref(base), ctypes.byref(size)):
            error = f"rank {rank}: {_lib.lib.cs_last_error().decode()}"
            break
        b = int(base.value)
        if b not in bases:
            bases[b] = len(bases)
        mine.append((bases[b], t.data_ptr() - b))
    handles = []
    for b in bases:
        out = (ctypes.c_uint8 * _lib.CS_IPC_HANDLE_BYTES)()
        if not error and _lib.lib.cs_ipc_get_handle(b, out):
            error = f"rank {rank}: {_lib.lib.cs_last_error().decode()}"
        handles.append((b, bytes(out)))
    if not all_ranks_agree(not error):
        raise ConfigError("gradient IPC export failed on some rank" + (f" ({error})" if error else ""))
    everyone: list = [None] * world
    dist.all_gather_object(everyone, (handles, mine))
    keys, addrs = [], []
    with torch.cuda.device(device):
        for r, (hs, items) in enumerate(everyone):
            if r == rank:
                addrs.append([int(t.data_ptr()) for t in tensors])
                continue
            mapped = []
            for b, h in hs:
                key = (r, b)
                ent = _peer_allocs.get(key)
                if ent is None and not error:
                    hb = (ctypes.c_uint8 * _lib.CS_IPC_HANDLE_BYTES).from_buffer_copy(h)
                    p = ctypes.c_void_p()
                    if _lib.lib.cs_ipc_open_handle(hb, ctypes.byref(p)):
                        error = f"rank {rank}: cannot map rank {r}: {_lib.lib.cs_last_error().decode()}"
                        mapped.append(0)
                        continue
                    ent = _peer_allocs[key] = [int(p.value), 0]
                if ent is None:
                    mapped.append(0)
                    continue
                ent[1] += 1
                keys.append(key)
                mapped.append(ent[0])
            addrs.append([mapped[i] + off for i, off in items])
    if not all_ranks_agree(not error):
        unmap_peer_tensors(keys)
        raise ConfigError("gradient peer mapping failed on some rank" + (f" ({error})" if error else ""))
    return addrs, keys


def unmap_peer_tensors(keys) -> None:
    for key in keys:
        ent = _peer_allocs.get(key)
        if ent is None:
            continue
        ent[1] -= 1
        if ent[1] == 0:
            del _peer_allocs[key]
            _lib.check("cs_ipc_close_handle", _lib.lib.cs_ipc_close_handle(ent[0]))


def all_ranks_agree(ok: bool) -> bool:
    """True iff every rank passes True (collective over the default torch.distributed group; a
    CUDA tensor when that group is NCCL-backed, which takes no CPU tensors)."""
    import torch.distributed as dist

    t = torch.tensor([1 if ok else 0], dtype=torch.int32)
    if dist.get_backend() == "nccl":
        t = t.to(torch.cuda.current_device())
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(int(t.item()))


class FlagArray:
    """The barrier flags of one app's p2p / ce transport, shared by every rank of the node.

    Two phases (a sync passes two barriers: every rank's K1 landed; every shard updated / every
    bucket read), each a W x W uint32 matrix, in one POSIX shared-memory segment (rank 0 creates
    it, the others attach by name, every rank page-locks and device-maps it with
    cs_host_register).  Row r of a phase holds the flags rank r waits on; rank p writes column p
    of every row (cs_flag_barrier).  The GPU front ends write, poll and reset it with constant-value
    stream memory operations, so a barrier occupies no SM and can be captured into a CUDA graph.
    Because the host can write the segment directly, a watchdog can release every rank's pending
    waits without issuing GPU work (:meth:`release`), which a wait on device memory behind a
    blocked stream could not guarantee.
    """

    PHASES = 2

    def __init__(self, rank: int, world: int):
        import torch.distributed as dist
        from multiprocessing import shared_memory

        import numpy as np

        from .errors import ConfigError

        self.rank, self.world = rank, world
        nbytes = 4 * self.PHASES * world * world
        self._size = max(4096, nbytes)
        self._shm = None
        name = [None]
        error = ""
        if rank == 0:
            try:
                self._shm = shared_memory.SharedMemory(create=True, size=self._size)
                name[0] = self._shm.name
            except OSError as exc:
                error = f"rank 0: cannot create the flag segment: {exc}"
        dist.broadcast_object_list(name, src=0)
        if name[0] is not None and rank != 0:
            try:
                self._shm = shared_memory.SharedMemory(name=name[0], create=False)
                # rank 0 owns (and unlinks) the segment; keep this process's resource tracker
                # from unlinking it a second time at exit
                from multiprocessing import resource_tracker

                resource_tracker.unregister(self._shm._name, "shared_memory")
            except OSError as exc:
                error = f"rank {rank}: cannot attach the flag segment: {exc}"
        self._dev = 0
        if self._shm is not None and not error:
            self._host = np.ndarray((self.PHASES, world, world), dtype=np.uint32, buffer=self._shm.buf)
            if rank == 0:
                self._host[:] = 0
            addr = ctypes.addressof(ctypes.c_char.from_buffer(self._shm.buf))
            dev = ctypes.c_void_p()
            rc = _lib.lib.cs_host_register(addr, self._size, ctypes.byref(dev))
            if rc:
                error = f"rank {rank}: cs_host_register failed: {_lib.lib.cs_last_error().decode()}"
            else:
                self._addr = addr
                self._dev = int(dev.value)
        ok = all_ranks_agree(not error)
        if rank == 0 and self._shm is not None:
            self._shm.unlink()            # every rank has attached (or failed): no /dev/shm leak
        if not ok:
            self.close()
            raise ConfigError("flag segment setup failed on some rank" + (f" ({error})" if error else ""))
        w2 = world * world
        self.peer_rows = [np.asarray([self._dev + 4 * (ph * w2 + p * world) for p in range(world)],
                                     dtype=np.uint64) for ph in range(self.PHASES)]
        self.local_rows = [self._dev + 4 * (ph * w2 + rank * world) for ph in range(self.PHASES)]

    def release(self) -> None:
        """Satisfy every pending wait of every rank: write 1 into every slot.  A released wait is
        followed by its own reset, so the caller repeats this until the streams drained.  Only for
        failure handling -- afterwards the flags order nothing, so the transport is retired."""
        if self._dev:
            self._host[:] = 1

    def close(self) -> None:
        if getattr(self, "_dev", 0):
            _lib.check("cs_host_unregister", _lib.lib.cs_host_unregister(self._addr))
            self._dev = 0
        if self._shm is not None:
            self._host = None
            try:
                self._shm.close()
            except BufferError:
                pass
            self._shm = None
