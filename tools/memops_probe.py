"""Single-GPU probe of the stream-memory-op flag barrier (cs_flag_barrier).

    python tools/memops_probe.py

Emulates rank 0 of 2 with both flag arrays local: the "peer" slot is pre-set, so the wait
returns immediately; prints whether the driver entry points resolved and the barrier's rc.
"""
import ctypes, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2103_07974_b200 import _lib
torch.cuda.init()
print("supported", _lib.lib.cs_stream_memops_supported(), _lib.lib.cs_last_error())
# single-rank self test: flag array local, nranks=1 -> no-op; use a 2-slot fake: write/wait on own memory
buf = torch.zeros(8, dtype=torch.int32, device="cuda")
import numpy as np
peers = np.asarray([buf.data_ptr(), buf.data_ptr()], dtype=np.uint64)
s = torch.cuda.current_stream().cuda_stream
# rank 0 of 2 ranks where 'peer 1' array is also buf: writes buf[0]=1 (slot rank0 in peer1's array), waits buf[1]>=1 -> would hang
# so instead emulate rank 1 writing first via torch
buf[1] = 1
rc = _lib.lib.cs_flag_barrier(peers.ctypes.data, buf.data_ptr(), 0, 2, 1, s)
torch.cuda.synchronize()
print("rc", rc, buf[:2].tolist())
