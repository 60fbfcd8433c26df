"""C1 microbenchmark: the bucket collectives through libcrossover.so's NCCL communicator.

    torchrun --nproc-per-node N tools/c1bench.py [--sizes-mb 1,16,102,256,1024] [--out f.json]

Ranks barrier (device sync + gloo barrier) before every timed call so rank skew is not
measured; the time is the max over ranks of CUDA events around the call on the comm stream.
busbw = 2(W-1)/W * S / t (nccl-tests convention) against NVLink 5's 900 GB/s per direction.
Also times the fused P2P kernel (reduce + SGD + broadcast) on the same bucket size.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import Harness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,16,102,256,1024")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default="")
    ap.add_argument("--p2p-caps", default="0", help="comma list of p2p_ctas values to time (0 = default)")
    args = ap.parse_args()
    from paper_2103_07974_b200.fusion import FusedGradientSync, SgdSettings, flatten_parameters

    h = Harness()
    W = h.world
    s = torch.cuda.Stream(h.dev, priority=-1)
    rows = []
    for mb in [float(x) for x in args.sizes_mb.split(",")]:
        n = int(mb * 2**20) // 4
        n -= n % (32 * W)
        row = {"size_MB": mb, "world": W}
        buf = torch.randn(n, device=h.dev)
        for name, fn in (
            ("allreduce", lambda: h.comm.all_reduce_(buf.data_ptr(), n, s.cuda_stream)),
            ("reduce_scatter", lambda: h.comm.reduce_scatter(buf.data_ptr(), buf.data_ptr() + h.rank * n // W * 4, n // W, s.cuda_stream)),
            ("all_gather", lambda: h.comm.all_gather(buf.data_ptr() + h.rank * n // W * 4, buf.data_ptr(), n // W, s.cuda_stream)),
        ):
            ts = []
            for it in range(args.iters + 2):
                h.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s); fn(); b.record(s); b.synchronize()
                if it >= 2:
                    ts.append(h.max_over_ranks(a.elapsed_time(b)))
            t = statistics.median(ts)
            bus = (2.0 if name == "allreduce" else 1.0) * (W - 1) / W * n * 4
            row[name] = {"ms": round(t, 4), "busbw_GB/s": round(bus / (t / 1e3) / 1e9, 1)}
        # fused P2P reduce + SGD(momentum) + broadcast on an n-element flat parameter buffer
        p = [torch.nn.Parameter(torch.randn(n - 32 * W, device=h.dev))]
        flat, _ = flatten_parameters(p, 32, W, ipc=True)
        sync = FusedGradientSync(p, SgdSettings(0.01, momentum=0.9), h.comm, mode="p2p", flat_params=flat)
        g = [torch.randn_like(p[0])]
        from paper_2103_07974_b200 import _lib
        for cap in [int(c) for c in args.p2p_caps.split(",")]:
            _lib.tune("p2p_ctas", cap)
            ts = []
            for it in range(args.iters + 2):
                sync.pack([g], s.cuda_stream)
                h.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                sync._p2p_tail(s.cuda_stream, None, None)
                b.record(s); b.synchronize()
                if it >= 2:
                    ts.append(h.max_over_ranks(a.elapsed_time(b)))
            t = statistics.median(ts)
            nv = 2.0 * (W - 1) / W * n * 4
            row[f"p2p_fused_with_barriers[ctas={cap}]"] = {
                "ms": round(t, 4), "busbw_equiv_GB/s": round(nv / (t / 1e3) / 1e9, 1), "hbm_bytes": sync.k2_bytes()}
        _lib.tune("p2p_ctas", 0)
        sync.close()
        # the NVSwitch-multicast fused sync (multimem.ld_reduce / multimem.st), same bucket
        from paper_2103_07974_b200.nvls import nvls_available

        if all(x for x in [nvls_available(h.dev)]):
            pn = [torch.nn.Parameter(torch.randn(n - 32 * W, device=h.dev))]
            flatn, _ = flatten_parameters(pn, 32, W, ipc="nvls")
            for cap in [int(c) for c in args.p2p_caps.split(",")]:
                syn = FusedGradientSync(pn, SgdSettings(0.01, momentum=0.9), h.comm, mode="nvls",
                                        flat_params=flatn, p2p_ctas=cap)
                ts = []
                for it in range(args.iters + 2):
                    syn.pack([g], s.cuda_stream)
                    h.barrier()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    syn._nvls_tail(s.cuda_stream, None, None)
                    b.record(s); b.synchronize()
                    if it >= 2:
                        ts.append(h.max_over_ranks(a.elapsed_time(b)))
                t = statistics.median(ts)
                nv = 2.0 * (W - 1) / W * n * 4
                row[f"nvls_fused_with_barriers[ctas={cap}]"] = {
                    "ms": round(t, 4), "busbw_equiv_GB/s": round(nv / (t / 1e3) / 1e9, 1)}
                syn.close()
            del flatn, pn
        rows.append(row)
        if h.rank == 0:
            print(json.dumps(row), flush=True)
        del buf, flat, p, g, sync
        torch.cuda.empty_cache()
    if h.rank == 0 and args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))
    h.close()


if __name__ == "__main__":
    main()
