"""Copy-engine transport study: NVLink pulls by the DMA engines vs SM-driven collectives.

    torchrun --nproc-per-node N tools/cebench.py [--sizes-mb 128,512] [--out f.json]

A. Bandwidth: each rank pulls its 1/W shard of the bucket from every peer (the reduce-scatter
   half of a copy-engine sync), W-1 copies serialised on one stream or forked onto W-1 streams.
B. Interference: a bf16 GEMM chain on one stream while a communication op loops on another;
   reports the GEMM slowdown and the comm op's rate for: nothing, CE pulls, the fused P2P kernel
   (32 CTAs and full grid), and NCCL all-reduce.  The question the crossover schedule asks:
   what does overlapped communication cost the other app's compute?
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


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="128,512")
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--gemm-n", type=int, default=4096)
    ap.add_argument("--gemm-reps", type=int, default=60)
    ap.add_argument("--comm-loops", type=int, default=6, help="comm ops issued beside the GEMM chain")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2103_07974_b200 import _lib
    from paper_2103_07974_b200.fusion import FusedGradientSync, SgdSettings, flatten_parameters
    from paper_2103_07974_b200.p2p import DeviceBuffer, exchange_peer_addresses

    h = Harness()
    W, r, dev = h.world, h.rank, h.dev
    streams = [torch.cuda.Stream(dev, priority=-1) for _ in range(max(1, 4 * (W - 1)))]
    main_s = streams[0]
    gemm_s = torch.cuda.Stream(dev)
    out = {"world": W, "rows": []}

    def copy(dst, src, nbytes, s):
        _lib.check("cs_copy_async", _lib.lib.cs_copy_async(dst, src, nbytes, s.cuda_stream))

    for mb in [int(x) for x in args.sizes_mb.split(",")]:
        n = mb * 2**20 // 4
        n -= n % (32 * W)
        shard = n // W
        bucket = DeviceBuffer(n, dev)
        bucket.tensor.normal_()
        recv = DeviceBuffer(n, dev)
        peers = exchange_peer_addresses(bucket, r, W)
        rpeers = exchange_peer_addresses(recv, r, W)
        row = {"size_MB": mb}

        def pulls(concurrent: bool, push: bool = False, split: int = 1, rotated: bool = False):
            fork = ev()
            fork.record(main_s)
            joins = []
            others = ([(r + k) % W for k in range(1, W)] if rotated else [x for x in range(W) if x != r])
            part = shard // split
            k = 0
            for src in others:
                for c in range(split):
                    s = streams[k % len(streams)] if concurrent else main_s
                    k += 1
                    if s is not main_s:
                        s.wait_event(fork)
                    off = c * part * 4
                    if push:   # write my copy of peer src's shard into its recv slot for me
                        copy(rpeers.addresses[src] + r * shard * 4 + off,
                             bucket.ptr + src * shard * 4 + off, part * 4, s)
                    else:
                        copy(recv.ptr + src * shard * 4 + off,
                             peers.addresses[src] + r * shard * 4 + off, part * 4, s)
                    if s is not main_s:
                        j = ev()
                        j.record(s)
                        joins.append(j)
            for j in joins:
                main_s.wait_event(j)

        for name, conc, push, split, rot in (("ce_pull_serial", False, False, 1, False),
                                             ("ce_pull_serial_rotated", False, False, 1, True),
                                             ("ce_pull_concurrent", True, False, 1, False),
                                             ("ce_pull_concurrent_rotated", True, False, 1, True),
                                             ("ce_pull_concurrent_split4", True, False, 4, False),
                                             ("ce_push_serial", False, True, 1, False),
                                             ("ce_push_serial_rotated", False, True, 1, True),
                                             ("ce_push_concurrent", True, True, 1, False),
                                             ("ce_push_concurrent_split4", True, True, 4, False)):
            ts = []
            for it in range(args.iters + 2):
                h.barrier()
                a, b = ev(), ev()
                a.record(main_s)
                pulls(conc, push, split, rot)
                b.record(main_s)
                b.synchronize()
                if it >= 2:
                    ts.append(h.max_over_ranks(a.elapsed_time(b)))
            t = statistics.median(ts)
            nbytes = (W - 1) * shard * 4
            row[name] = {"ms": round(t, 4), "GB/s_in": round(nbytes / (t / 1e3) / 1e9, 1)}
        # correctness of one pull set
        pulls(True)
        torch.cuda.synchronize()
        h.barrier()

        # B: interference with a GEMM chain
        g_a = torch.randn(args.gemm_n, args.gemm_n, device=dev, dtype=torch.bfloat16)
        g_b = torch.randn(args.gemm_n, args.gemm_n, device=dev, dtype=torch.bfloat16) / args.gemm_n ** 0.5

        def gemm_chain():
            x = g_a
            for _ in range(args.gemm_reps):
                x = x @ g_b
            return x

        p = [torch.nn.Parameter(torch.randn(n - 32 * W, device=dev))]
        flat, _ = flatten_parameters(p, 32, W, ipc=True)
        syncs = {cap: FusedGradientSync(p, SgdSettings(0.01, momentum=0.9), h.comm, mode="p2p",
                                        flat_params=flat, p2p_ctas=cap) for cap in (32, 0)}
        for s_ in syncs.values():
            s_.pack([[torch.randn_like(p[0])]], main_s.cuda_stream)
        ar_buf = torch.randn(n, device=dev)

        ops = {
            "none": None,
            "ce_pull_concurrent": lambda: pulls(True),
            "ce_pull_serial_rotated": lambda: pulls(False, False, 1, True),
            "ce_push_concurrent": lambda: pulls(True, True),
            "p2p_kernel_32ctas": lambda: syncs[32]._p2p_tail(main_s.cuda_stream, None, None),
            "p2p_kernel_full": lambda: syncs[0]._p2p_tail(main_s.cuda_stream, None, None),
            "nccl_allreduce": lambda: h.comm.all_reduce_(ar_buf.data_ptr(), n, main_s.cuda_stream),
        }
        inter = {}
        for name, op in ops.items():
            gts, cts, counts = [], [], []
            for it in range(4):
                torch.cuda.synchronize()
                h.barrier()
                ga, gb = ev(), ev()
                ca, cb = ev(), ev()
                ga.record(gemm_s)
                with torch.cuda.stream(gemm_s):
                    gemm_chain()
                gb.record(gemm_s)
                k = 0
                if op is not None:
                    ca.record(main_s)
                    # keep the comm stream busy for about the GEMM's duration
                    for _ in range(args.comm_loops):
                        op()
                        k += 1
                    cb.record(main_s)
                torch.cuda.synchronize()
                if it >= 1:
                    gts.append(h.max_over_ranks(ga.elapsed_time(gb)))
                    if op is not None:
                        cts.append(h.max_over_ranks(ca.elapsed_time(cb)) / k)
            inter[name] = {"gemm_ms": round(statistics.median(gts), 4)}
            if cts:
                inter[name]["comm_op_ms"] = round(statistics.median(cts), 4)
        base = inter["none"]["gemm_ms"]
        for v in inter.values():
            v["gemm_slowdown"] = round(v["gemm_ms"] / base, 4)
        # each comm op alone (no GEMM) for reference
        for name, op in ops.items():
            if op is None:
                continue
            ts = []
            for it in range(args.iters + 2):
                h.barrier()
                a, b = ev(), ev()
                a.record(main_s)
                op()
                b.record(main_s)
                b.synchronize()
                if it >= 2:
                    ts.append(h.max_over_ranks(a.elapsed_time(b)))
            inter[name]["alone_ms"] = round(statistics.median(ts), 4)
        row["interference"] = inter
        out["rows"].append(row)
        for s_ in syncs.values():
            s_.close()
        peers.close()
        rpeers.close()
        torch.cuda.synchronize()
        h.barrier()
        bucket.close()
        recv.close()
        if r == 0:
            print(json.dumps(row), flush=True)
    if r == 0 and args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    h.close()


if __name__ == "__main__":
    main()
