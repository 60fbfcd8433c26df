"""Latency of the SM-free flag barrier: flags in host shared memory vs in IPC-mapped device memory.

    torchrun --nproc-per-node 2 tools/barrier_latency.py [--out f.json]

For each flag location: (a) back-to-back barriers on an idle GPU; (b) one barrier issued while the
compute stream runs a long spin kernel (cs_spin_ns) -- does the wait notice the peer's write while
another engine of the GPU is busy, or only at the next scheduling event?
"""
import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import Harness  # noqa: E402
from paper_2103_07974_b200 import _lib  # noqa: E402
from paper_2103_07974_b200.p2p import DeviceBuffer, FlagArray, exchange_peer_addresses  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--spin-ms", type=float, default=5.0)
    args = ap.parse_args()
    h = Harness()
    r, w, dev = h.rank, h.world, h.dev
    lo, hi = torch.cuda.Stream.priority_range()
    ms = torch.cuda.Stream(dev, priority=hi)
    cs = torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out = {}

    # flag rows: host shared memory (FlagArray) or device memory mapped into every rank
    fa = FlagArray(r, w)
    host_rows = (fa.peer_rows[0], fa.local_rows[0])
    dbuf = DeviceBuffer(64, dev)
    dbuf.tensor.zero_()
    dmap = exchange_peer_addresses(dbuf, r, w)
    dev_rows = (np.asarray([a + 0 for a in dmap.addresses], dtype=np.uint64), dbuf.ptr)

    def barrier(rows, stream):
        peers, local = rows
        _lib.check("cs_flag_barrier", _lib.lib.cs_flag_barrier(peers.ctypes.data, local, r, w,
                                                               stream.cuda_stream))

    for name, rows in (("host_shm", host_rows), ("device_ipc", dev_rows)):
        # (a) idle: 50 back-to-back barriers
        h.barrier()
        a, b = ev(), ev()
        a.record(ms)
        for _ in range(50):
            barrier(rows, ms)
        b.record(ms)
        b.synchronize()
        idle_us = a.elapsed_time(b) / 50 * 1e3
        # (b) busy: compute stream spins, then one barrier on the comm stream
        busy = []
        for _ in range(5):
            h.barrier()
            _lib.spin_ns(int(args.spin_ms * 1e6), cs.cuda_stream)
            a, b = ev(), ev()
            a.record(ms)
            barrier(rows, ms)
            b.record(ms)
            torch.cuda.synchronize()
            busy.append(a.elapsed_time(b) * 1e3)
        out[name] = {"idle_barrier_us": round(idle_us, 2),
                     "barrier_beside_spin_us": round(statistics.median(busy), 2),
                     "spin_ms": args.spin_ms}
        if r == 0:
            print(name, out[name], flush=True)
    h.barrier()
    dmap.close()
    fa.close()
    if r == 0 and args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))
    h.close()


if __name__ == "__main__":
    main()
