"""K2 beside a tensor-core GEMM chain: how much of the sync's SM time does the compute pay?

    python tools/k2_interference.py [--mb 300] [--gemm-n 4096] [--reps 40] [--out f.json]

One GPU.  A bf16 GEMM chain runs on a normal-priority stream while K2 (the fused update, momentum,
over an `mb` MB bucket) loops on a high-priority stream -- the crossover situation of the band /
sweep runs (tools/band.py) and of every app whose compute is GEMM-bound.  For every K2 launch shape
(cs_tune "reg_shape": unroll x CTAs/SM) and grid cap (max_ctas: 0 = one CTA per chunk, else a
persistent grid) it reports K2 alone, the GEMM chain alone, both together (GEMM slowdown, K2 time
while overlapped) and the fraction of K2's time the GEMM lost.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2103_07974_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=300)
    ap.add_argument("--gemm-n", type=int, default=4096)
    ap.add_argument("--gemm-reps", type=int, default=40)
    ap.add_argument("--k2-loops", type=int, default=8)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    n = args.mb * 2**20 // 4
    n -= n % 1024
    grad = torch.randn(n, device=dev) * 1e-3
    p = torch.randn(n, device=dev)
    m = torch.zeros(n, device=dev)
    upd = np.zeros(1, dtype=_lib.UPDATE_DESC)
    upd["param"] = p.data_ptr()
    upd["momentum_buf"] = m.data_ptr()
    upd["numel"] = n
    src = np.asarray([grad.data_ptr()], dtype=np.uint64)
    h = _lib.SgdHyper(lr=1e-4, momentum=0.9, dampening_complement=1.0, weight_decay=1e-4,
                      first_step=0, divisor=1, rounding=_lib.CS_ROUND_TORCH)
    gemm_s = torch.cuda.Stream(dev)
    lo, hi = torch.cuda.Stream.priority_range()
    comm_s = torch.cuda.Stream(dev, priority=hi)
    a = torch.randn(args.gemm_n, args.gemm_n, device=dev, dtype=torch.bfloat16)
    b = torch.randn(args.gemm_n, args.gemm_n, device=dev, dtype=torch.bfloat16) / args.gemm_n ** 0.5
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def gemm_chain():
        with torch.cuda.stream(gemm_s):
            x = a
            for _ in range(args.gemm_reps):
                x = x @ b

    def k2(cap, loops):
        for _ in range(loops):
            _lib.unpack_sgd(upd, src, 0, h, comm_s.cuda_stream, cap)

    def timed(fn, stream):
        s, e = ev(), ev()
        s.record(stream)
        fn()
        e.record(stream)
        return s, e

    # warm-up
    gemm_chain()
    k2(0, 2)
    torch.cuda.synchronize()
    bytes_k2 = 5 * n * 4
    rows = []
    g_alone = []
    for _ in range(3):
        s, e = timed(gemm_chain, gemm_s)
        torch.cuda.synchronize()
        g_alone.append(s.elapsed_time(e))
    g_alone = statistics.median(g_alone)
    for shape in range(5):
        _lib.tune("reg_shape", shape)
        for cap in (0, sms, 2 * sms, 64, 32):
            alone = []
            for _ in range(3):
                s, e = timed(lambda: k2(cap, args.k2_loops), comm_s)
                torch.cuda.synchronize()
                alone.append(s.elapsed_time(e) / args.k2_loops)
            alone = statistics.median(alone)
            gt, kt = [], []
            for _ in range(3):
                torch.cuda.synchronize()
                gs, ge = timed(gemm_chain, gemm_s)
                ks, ke = timed(lambda: k2(cap, args.k2_loops), comm_s)
                torch.cuda.synchronize()
                gt.append(gs.elapsed_time(ge))
                kt.append(ks.elapsed_time(ke) / args.k2_loops)
            g_with, k_with = statistics.median(gt), statistics.median(kt)
            k2_total = args.k2_loops * k_with
            row = {"reg_shape": shape, "max_ctas": cap, "k2_alone_ms": round(alone, 4),
                   "k2_alone_frac": round(bytes_k2 / (alone / 1e3) / 1e9 / 6547.5, 3),
                   "gemm_alone_ms": round(g_alone, 3), "gemm_with_k2_ms": round(g_with, 3),
                   "k2_overlapped_ms": round(k_with, 4),
                   "gemm_loss_per_k2_ms": round((g_with - g_alone) / args.k2_loops, 4),
                   "gemm_loss_over_k2_alone": round((g_with - g_alone) / args.k2_loops / alone, 3)}
            rows.append(row)
            print(json.dumps(row), flush=True)
    _lib.tune("reg_shape", 1)
    if args.out:
        Path(args.out).write_text(json.dumps({"mb": args.mb, "gemm_n": args.gemm_n, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
