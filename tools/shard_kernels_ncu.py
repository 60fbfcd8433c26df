"""Single-GPU stand-ins of the W-rank shard kernels, for ncu --set full (DRAM traffic per launch).

    ncu --set full -k regex:"unpack_sgd|p2p_reduce|p2p_bulk" -c 4 -o prof python tools/shard_kernels_ncu.py
        [--world 4] [--p2p-ctas 32 [--registers]]

ncu cannot replay a multi-rank command, so the kernels of the `ce` and `p2p` transports are run
here on one GPU with the W ranks' buffers all local (same kernels, same launch shapes, same
shard size as ResNet-50's bucket at world W):
  * shard K2 (`ce`): cs_unpack_sgd over W shard-sized sources, SGD-momentum on the shard;
  * fused P2P kernel: cs_p2p_reduce_sgd_bcast with W local "peer" sources and destinations.
Each runs twice (the second launch is the one to read).  DRAM traffic from ncu then says whether
a kernel re-reads (wasted bytes); the NVLink half of the P2P kernel's traffic is local here.
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=4)
    ap.add_argument("--bucket-bytes", type=int, default=102_228_128)   # ResNet-50
    ap.add_argument("--p2p-ctas", type=int, default=0,
                    help="grid cap of the P2P launches (> 0: the crossover shape, TMA ring by default)")
    ap.add_argument("--registers", action="store_true", help="capped P2P launches on the register kernel")
    args = ap.parse_args()
    from paper_2103_07974_b200 import _lib

    W = args.world
    dev = torch.device("cuda", 0)
    total = -(-args.bucket_bytes // 4)
    total += (-total) % (32 * W)
    shard = total // W
    s = torch.cuda.current_stream().cuda_stream
    srcs = [torch.randn(shard, device=dev) for _ in range(W)]
    p = torch.randn(shard, device=dev)
    mom = torch.randn(shard, device=dev)
    h = _lib.SgdHyper(lr=0.05, momentum=0.9, dampening_complement=1.0, weight_decay=1e-4,
                      divisor=W, first_step=0, rounding=_lib.CS_ROUND_TORCH)

    upd = np.zeros(1, dtype=_lib.UPDATE_DESC)
    upd["param"], upd["momentum_buf"], upd["numel"] = p.data_ptr(), mom.data_ptr(), shard
    sources = np.asarray([x.data_ptr() for x in srcs], dtype=np.uint64)
    for _ in range(2):
        _lib.unpack_sgd(upd, sources, 0, h, s)

    dsts = [torch.zeros(shard, device=dev) for _ in range(W)]
    d = _lib.P2PDesc()
    for r in range(W):
        d.src[r], d.dst[r] = srcs[r].data_ptr(), dsts[r].data_ptr()
    d.param, d.momentum_buf, d.numel, d.nranks = p.data_ptr(), mom.data_ptr(), shard, W
    d.max_ctas = args.p2p_ctas
    _lib.tune("p2p_bulk", 0 if args.registers else 1)
    for _ in range(2):
        _lib.check("p2p", _lib.lib.cs_p2p_reduce_sgd_bcast(ctypes.byref(d), ctypes.byref(h), s))
    torch.cuda.synchronize()
    print(f"world {W}: shard {shard} elements; K2 algorithmic bytes {(W + 4) * shard * 4}, "
          f"P2P {(2 * W + 3) * shard * 4}")


if __name__ == "__main__":
    main()
