"""Buffers bound to an NVSwitch multicast object (NVLS), for the ``nvls`` sync transport.

A :class:`NvlsBuffer` is one fp32 buffer per rank, all bound to one multicast object: each rank
sees its own copy through a unicast mapping (a plain device pointer, shown to torch as a tensor)
and all copies at once through a multicast mapping, on which ``multimem.ld_reduce`` returns the
sum over the ranks (computed in the switch) and ``multimem.st`` writes every rank's copy.  The
multicast object travels from rank 0 to the others as a POSIX file descriptor over a UNIX-domain
socket (SCM_RIGHTS); torch.distributed carries the socket path.  Creation is collective and its
failure is agreed on, like the IPC mappings of p2p.py.  Multicast needs distinct GPUs behind an
NVSwitch (one rank per device).
"""

from __future__ import annotations

import ctypes
import os
import socket
import tempfile
import time
import weakref

import torch

from . import _lib
from .errors import ConfigError
from .p2p import all_ranks_agree

__all__ = ["NvlsBuffer", "nvls_buffer_of", "nvls_available"]

_live: "weakref.WeakValueDictionary[int, NvlsBuffer]" = weakref.WeakValueDictionary()


def nvls_available(device: torch.device) -> bool:
    return bool(_lib.lib.cs_nvls_supported(torch.device(device).index or 0))


def nvls_buffer_of(t: torch.Tensor) -> "NvlsBuffer | None":
    return _live.get(t.data_ptr())


def _share_fd(fd: int, rank: int, world: int, timeout: float = 60.0) -> int:
    """Rank 0's file descriptor to every rank (returns this rank's own descriptor, -1 on failure;
    a failure is agreed on by the caller, so no rank waits for a peer that gave up)."""
    import torch.distributed as dist

    path = [None]
    server = None
    if rank == 0:
        d = tempfile.mkdtemp(prefix="cs_nvls_")
        path[0] = os.path.join(d, "fd.sock")
        server = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        server.bind(path[0])
        server.listen(world)
        server.settimeout(timeout)
    dist.broadcast_object_list(path, src=0)
    if rank == 0:
        try:
            for _ in range(world - 1):
                conn, _ = server.accept()
                with conn:
                    socket.send_fds(conn, [b"f"], [fd])
        except OSError:
            return -1
        finally:
            server.close()
            os.unlink(path[0])
            os.rmdir(os.path.dirname(path[0]))
        return fd
    deadline = time.monotonic() + timeout
    with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as sock:
        sock.settimeout(timeout)
        while True:
            try:
                sock.connect(path[0])
                break
            except (FileNotFoundError, ConnectionRefusedError):
                if time.monotonic() > deadline:
                    return -1
                time.sleep(0.01)
        try:
            _, fds, _, _ = socket.recv_fds(sock, 1, 1)
        except OSError:
            return -1
    return fds[0] if fds else -1


class NvlsBuffer:
    """`numel` fp32 elements per rank, bound to one multicast object across `world` ranks."""

    def __init__(self, numel: int, device: torch.device, rank: int, world: int):
        if numel <= 0:
            raise ValueError("numel must be > 0")
        self.device = torch.device(device)
        self.dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.numel = int(numel)
        self.rank, self.world = rank, world
        self.mc = 0
        self.phys = 0
        self.ptr = 0
        self.mc_ptr = 0
        gran = ctypes.c_size_t()
        error = ""
        if not _lib.lib.cs_nvls_supported(self.dev_index):
            error = f"rank {rank}: device {self.dev_index} has no NVSwitch multicast"
        elif _lib.lib.cs_nvls_granularity(world, self.numel * 4, ctypes.byref(gran)):
            error = f"rank {rank}: {_lib.lib.cs_last_error().decode()}"
        if not all_ranks_agree(not error):
            raise ConfigError("nvls unavailable on some rank" + (f" ({error})" if error else ""))
        self.gran = int(gran.value)
        self.size = (self.numel * 4 + self.gran - 1) // self.gran * self.gran
        with torch.cuda.device(self.dev_index):
            mc = ctypes.c_uint64()
            fd = ctypes.c_int(-1)
            if rank == 0 and _lib.lib.cs_nvls_create(world, self.size, ctypes.byref(mc), ctypes.byref(fd)):
                error = f"rank 0: {_lib.lib.cs_last_error().decode()}"
            if not all_ranks_agree(not error):
                raise ConfigError("nvls multicast object creation failed" + (f" ({error})" if error else ""))
            myfd = _share_fd(fd.value, rank, world)
            if myfd < 0:
                error = f"rank {rank}: passing the multicast handle over a UNIX socket failed"
            elif rank != 0 and _lib.lib.cs_nvls_import(myfd, ctypes.byref(mc)):
                error = f"rank {rank}: {_lib.lib.cs_last_error().decode()}"
            if myfd >= 0:
                os.close(myfd)
            elif rank == 0:
                os.close(fd.value)
            self.mc = int(mc.value)
            if not error and _lib.lib.cs_nvls_add_device(self.mc, self.dev_index):
                error = f"rank {rank}: {_lib.lib.cs_last_error().decode()}"
            if not all_ranks_agree(not error):            # every device added before any bind
                self.close()
                raise ConfigError("nvls multicast setup failed" + (f" ({error})" if error else ""))
            phys, uc, mcp = ctypes.c_uint64(), ctypes.c_void_p(), ctypes.c_void_p()
            if _lib.lib.cs_nvls_alloc_bind(self.mc, self.dev_index, self.size, self.gran, ctypes.byref(phys),
                                           ctypes.byref(uc), ctypes.byref(mcp)):
                error = f"rank {rank}: {_lib.lib.cs_last_error().decode()}"
            else:
                self.phys, self.ptr, self.mc_ptr = int(phys.value), int(uc.value), int(mcp.value)
            if not all_ranks_agree(not error):            # every rank bound before any multimem op
                self.close()
                raise ConfigError("nvls bind failed" + (f" ({error})" if error else ""))
        self.__cuda_array_interface__ = {"shape": (self.numel,), "typestr": "<f4",
                                         "data": (self.ptr, False), "version": 3, "strides": None}
        t = torch.as_tensor(self, device=self.device)
        self._tensor = weakref.ref(t)
        self._first = t
        _live[self.ptr] = self

    @property
    def tensor(self) -> torch.Tensor:
        first, self._first = self._first, None
        t = first if first is not None else self._tensor()
        if t is None:
            raise RuntimeError("NvlsBuffer: every tensor view was dropped")
        return t

    def close(self) -> None:
        """Unmap and release (collective use: call after every rank finished its multimem ops)."""
        if self.ptr or self.phys:
            _live.pop(self.ptr, None)
            self._first = None
            _lib.lib.cs_nvls_free(self.mc, self.dev_index, self.phys, self.ptr or None,
                                  self.mc_ptr or None, self.size)
            self.ptr = self.phys = self.mc_ptr = 0
        if self.mc:
            _lib.lib.cs_nvls_release(self.mc)
            self.mc = 0

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown
            pass
