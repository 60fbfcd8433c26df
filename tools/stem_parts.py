"""Timing of the GEMM stem's parts at ResNet-50 bs 256: im2col, forward GEMM, weight-gradient GEMM.

    python tools/stem_parts.py
"""
import ctypes
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    from paper_2103_07974_b200 import _lib

    dev = torch.device("cuda", 0)
    n, h, w, c, oh, ow, kp = 256, 224, 224, 3, 112, 112, 152
    x = torch.randn(n, c, h, w, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    p = torch.empty((n * oh * ow, kp), dtype=torch.bfloat16, device=dev)
    wm = torch.randn(64, kp, device=dev, dtype=torch.bfloat16)
    dy = torch.randn(n * oh * ow, 64, device=dev, dtype=torch.bfloat16)
    y = torch.empty(n * oh * ow, 64, device=dev, dtype=torch.bfloat16)
    shape = (ctypes.c_int * 13)(n, h, w, c, oh, ow, 7, 7, 2, 2, 3, 3, kp)
    st = torch.cuda.current_stream().cuda_stream
    t_im = timeit(lambda: _lib.lib.cs_im2col_nhwc(x.data_ptr(), p.data_ptr(), shape, st))
    t_f = timeit(lambda: torch.mm(p, wm.t(), out=y))
    t_w = timeit(lambda: dy.t() @ p)
    t_w2 = timeit(lambda: p.t() @ dy)
    t_w3 = timeit(lambda: torch.mm(dy.t(), p, out_dtype=torch.float32) if hasattr(torch.mm, "__call__") else None)
    gb = lambda b, t: b / (t / 1e3) / 1e9  # noqa: E731
    print(f"im2col {t_im:.3f} ms ({gb(p.numel() * 2 + x.numel() * 2, t_im):.0f} GB/s)")
    print(f"fwd GEMM {t_f:.3f} ms ({gb(p.numel() * 2 + y.numel() * 2, t_f):.0f} GB/s)")
    print(f"wgrad GEMM {t_w:.3f} ms ({gb(p.numel() * 2 + dy.numel() * 2, t_w):.0f} GB/s)")
    print(f"wgrad GEMM as P^T.dy {t_w2:.3f} ms; fp32-out variant {t_w3:.3f} ms")


if __name__ == "__main__":
    main()
