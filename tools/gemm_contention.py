"""What slows a tensor-core GEMM chain when a sync runs beside it: SM sharing, HBM traffic or power?

    python tools/gemm_contention.py [--mb 300] [--gemm-n 4096] [--gemm-reps 200] [--out f.json]

One GPU.  A bf16 GEMM chain runs on a normal-priority stream; beside it, on a high-priority
stream, one kind of side work loops for about the chain's duration:

  none        the chain alone
  k2_hbm      K2 (fused update, momentum) over an `mb` MB bucket: SM time + HBM traffic
  k2_hbm_c32  the same at a 32-CTA persistent grid
  k2_l2       K2 over a 16 MB bucket that stays in L2: SM time + L2 traffic, no HBM
  ce_copy     device-to-device copies of `mb` MB by the copy engines: HBM traffic, no SM
  ce_copy_dN  the same copies with a 1-thread wait between them, at about 1/N of the full rate

Each arm is a CUDA graph replayed for about `--window` seconds (NVML averages board power over
about a second, so shorter windows read stale power and clocks).

For each it reports the chain's slowdown, the side work's bytes per second while overlapped, and
the SM clock, board power and clock-event reasons sampled by NVML during the overlapped window, so
the slowdown can be split between SM sharing (k2_l2), memory traffic (ce_copy) and power (clock).
"""
import argparse
import json
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2103_07974_b200 import _lib  # noqa: E402

REASONS = {0x1: "gpu_idle", 0x2: "app_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x20: "sw_thermal", 0x40: "hw_thermal", 0x80: "hw_power_brake", 0x100: "display_clocks"}


class Sampler:
    """NVML SM clock / power / clock-event reasons every `period` s while `on` is set."""

    def __init__(self, index: int, period: float = 0.002):
        import pynvml

        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.period = period
        self.on = threading.Event()
        self.stop = threading.Event()
        self.samples: list[tuple[int, float, int]] = []
        self.cap_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv, h = self.nv, self.h
        while not self.stop.is_set():
            if self.on.is_set():
                try:
                    clk = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((clk, pw, rs))
                except Exception:  # noqa: BLE001 - a failed sample is skipped
                    pass
            time.sleep(self.period)

    def window(self):
        self.samples = []
        self.on.set()

    def close_window(self) -> dict:
        self.on.clear()
        s = self.samples
        if not s:
            return {"samples": 0}
        bits = 0
        for _, _, r in s:
            bits |= r
        return {"samples": len(s), "sm_mhz_median": statistics.median(c for c, _, _ in s),
                "sm_mhz_min": min(c for c, _, _ in s),
                "power_w_median": round(statistics.median(p for _, p, _ in s), 1),
                "reasons": [n for b, n in REASONS.items() if bits & b]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=300)
    ap.add_argument("--gemm-n", type=int, default=4096)
    ap.add_argument("--gemm-reps", type=int, default=200)
    ap.add_argument("--window", type=float, default=1.5, help="seconds per measurement")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    sampler = Sampler(0)

    def bucket(mb):
        n = mb * 2**20 // 4
        n -= n % 1024
        grad = torch.randn(n, device=dev) * 1e-3
        p = torch.randn(n, device=dev)
        m = torch.zeros(n, device=dev)
        upd = np.zeros(1, dtype=_lib.UPDATE_DESC)
        upd["param"], upd["momentum_buf"], upd["numel"] = p.data_ptr(), m.data_ptr(), n
        src = np.asarray([grad.data_ptr()], dtype=np.uint64)
        return (grad, p, m), upd, src, 5 * n * 4

    big_keep, big_upd, big_src, big_bytes = bucket(args.mb)
    small_keep, small_upd, small_src, small_bytes = bucket(16)
    copy_src = torch.empty(args.mb * 2**20, dtype=torch.uint8, device=dev)
    copy_dst = torch.empty_like(copy_src)
    h = _lib.SgdHyper(lr=1e-4, momentum=0.9, dampening_complement=1.0, weight_decay=1e-4,
                      first_step=0, divisor=1, rounding=_lib.CS_ROUND_TORCH)
    gemm_s = torch.cuda.Stream(dev)
    _, hi = torch.cuda.Stream.priority_range()
    side_s = torch.cuda.Stream(dev, priority=hi)
    a = torch.randn(args.gemm_n, args.gemm_n, device=dev, dtype=torch.bfloat16)
    b = torch.randn(args.gemm_n, args.gemm_n, device=dev, dtype=torch.bfloat16) / args.gemm_n ** 0.5
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def gemm_chain():
        with torch.cuda.stream(gemm_s):
            x = a
            for _ in range(args.gemm_reps):
                x = x @ b

    sides = {
        "k2_hbm": (lambda: _lib.unpack_sgd(big_upd, big_src, 0, h, side_s.cuda_stream, 0), big_bytes),
        "k2_hbm_c32": (lambda: _lib.unpack_sgd(big_upd, big_src, 0, h, side_s.cuda_stream, 32), big_bytes),
        "k2_l2": (lambda: _lib.unpack_sgd(small_upd, small_src, 0, h, side_s.cuda_stream, 0), small_bytes),
    }

    def ce_copy():
        with torch.cuda.stream(side_s):
            copy_dst.copy_(copy_src, non_blocking=True)

    sides["ce_copy"] = (ce_copy, 2 * copy_src.numel())

    def timed(fn, stream, loops=1):
        s, e = ev(), ev()
        s.record(stream)
        for _ in range(loops):
            fn()
        e.record(stream)
        torch.cuda.synchronize()
        return s.elapsed_time(e)

    copy_ms = timed(ce_copy, side_s, 4) / 4
    for duty in (2, 4):
        def throttled(d=duty):
            ce_copy()
            _lib.spin_ns(int(copy_ms * (d - 1) * 1e6), side_s.cuda_stream)
        sides[f"ce_copy_d{duty}"] = (throttled, 2 * copy_src.numel())

    def graph_of(fn, stream, loops):
        """`loops` calls of fn captured as one graph on `stream`."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            fn()                                 # warm the allocator / lazy init outside capture
            torch.cuda.synchronize()
            g.capture_begin()
            for _ in range(loops):
                fn()
            g.capture_end()
        torch.cuda.synchronize()
        return g

    def replay_timed(graphs_streams, reps):
        """Replay each (graph, stream) `reps` times, all streams concurrently; ms per stream."""
        marks = []
        for g, st in graphs_streams:
            s, e = ev(), ev()
            with torch.cuda.stream(st):
                s.record(st)
            marks.append((s, e, g, st))
        for _ in range(reps):
            for _, _, g, st in marks:
                with torch.cuda.stream(st):
                    g.replay()
        for s, e, _, st in marks:
            e.record(st)
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e, _, _ in marks]

    gemm_g = graph_of(gemm_chain, gemm_s, 1)
    one = replay_timed([(gemm_g, gemm_s)], 3)[0] / 3
    reps = max(3, int(args.window * 1e3 / one))
    rows = []
    sampler.window()
    g_alone = replay_timed([(gemm_g, gemm_s)], reps)[0] / reps
    clk = sampler.close_window()
    rows.append({"side": "none", "gemm_ms": round(g_alone, 3), "reps": reps,
                 "gemm_tflops": round(2 * args.gemm_n ** 3 * args.gemm_reps / (g_alone / 1e3) / 1e12, 1),
                 **clk})
    print(json.dumps(rows[-1]), flush=True)
    for name, (fn, nbytes) in sides.items():
        one = timed(fn, side_s, 4) / 4
        loops = max(1, int(g_alone / one))
        side_g = graph_of(fn, side_s, loops)
        sampler.window()
        alone = replay_timed([(side_g, side_s)], reps)[0] / reps
        clk_alone = sampler.close_window()
        sampler.window()
        g_with, s_with = (t / reps for t in replay_timed([(gemm_g, gemm_s), (side_g, side_s)], reps))
        clk = sampler.close_window()
        row = {"side": name, "loops": loops, "side_alone_ms": round(alone, 3),
               "side_alone_GBps": round(loops * nbytes / (alone / 1e3) / 1e9, 1),
               "side_alone_clock": clk_alone,
               "gemm_alone_ms": round(g_alone, 3), "gemm_with_ms": round(g_with, 3),
               "gemm_slowdown": round(g_with / g_alone, 3),
               "side_with_ms": round(s_with, 3),
               "side_with_GBps": round(loops * nbytes / (s_with / 1e3) / 1e9, 1),
               "gemm_ms_lost_per_side_ms_alone": round((g_with - g_alone) / alone, 3),
               "gemm_ms_lost_per_GB": round((g_with - g_alone) / (loops * nbytes / 1e9), 4),
               **clk}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del side_g
    sampler.stop.set()
    if args.out:
        Path(args.out).write_text(json.dumps({"mb": args.mb, "gemm_n": args.gemm_n, "gemm_reps": args.gemm_reps,
                                              "power_limit_w": sampler.cap_w, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
