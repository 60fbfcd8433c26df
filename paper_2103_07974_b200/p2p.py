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

import torch

from . import _lib

__all__ = ["DeviceBuffer", "exchange_peer_addresses", "PeerMapping", "all_ranks_agree"]

_live: dict[int, "DeviceBuffer"] = {}


class DeviceBuffer:
    """A zero-filled fp32 cudaMalloc allocation shown to torch as a 1-D tensor."""

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
        self.tensor = torch.as_tensor(self, device=self.device)
        assert self.tensor.data_ptr() == self.ptr
        _live[self.ptr] = self

    def ipc_handle(self) -> bytes:
        out = (ctypes.c_uint8 * _lib.CS_IPC_HANDLE_BYTES)()
        _lib.check("cs_ipc_get_handle", _lib.lib.cs_ipc_get_handle(self.ptr, out))
        return bytes(out)

    def close(self) -> None:
        if self.ptr:
            _live.pop(self.ptr, None)
            self.tensor = None
            _lib.check("cs_device_free", _lib.lib.cs_device_free(self.ptr))
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
    ok = torch.tensor([0 if error else 1], dtype=torch.int32)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    mapping = PeerMapping(addrs, opened)
    if int(ok.item()) == 0:
        mapping.close()
        raise ConfigError("p2p peer mapping failed on some rank" + (f" ({error})" if error else ""))
    return mapping


def all_ranks_agree(ok: bool) -> bool:
    """True iff every rank passes True (collective over torch.distributed's CPU group)."""
    import torch.distributed as dist

    t = torch.tensor([1 if ok else 0], dtype=torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(int(t.item()))
