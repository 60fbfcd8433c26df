"""ResNet-50 stem max-pool (3x3 / 2, pad 1) fwd + bwd at bs 256: libcrossover.so kernels vs ATen.

    python tools/pool_bench.py
"""
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
    from paper_2103_07974_b200.bn import CrossoverMaxPool2d

    dev = torch.device("cuda", 0)
    x = torch.randn(256, 64, 112, 112, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    x.requires_grad_(True)
    dy = torch.randn(256, 64, 56, 56, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    for name, mod in (("aten", torch.nn.MaxPool2d(3, 2, 1)), ("ours", CrossoverMaxPool2d(3, 2, 1))):
        fwd = timeit(lambda: mod(x))
        both = timeit(lambda: mod(x).backward(dy))
        print(f"{name}: fwd {fwd:.3f} ms, fwd+bwd {both:.3f} ms")
    # the kernels alone (no autograd, no gradient accumulation)
    import ctypes
    from paper_2103_07974_b200 import _lib
    xd = x.detach()
    y = torch.empty_like(dy)
    arg = torch.empty(dy.numel(), dtype=torch.uint8, device=dev)
    dx = torch.empty_like(xd)
    shape = (ctypes.c_int * 12)(256, 112, 112, 64, 56, 56, 3, 3, 2, 2, 1, 1)
    st = torch.cuda.current_stream().cuda_stream
    kf = timeit(lambda: _lib.lib.cs_maxpool2d_forward(xd.data_ptr(), y.data_ptr(), arg.data_ptr(), shape, st))
    kb = timeit(lambda: _lib.lib.cs_maxpool2d_backward(dy.data_ptr(), arg.data_ptr(), dx.data_ptr(), shape, st))
    print(f"kernels alone: fwd {kf:.3f} ms, bwd {kb:.3f} ms")
    # algorithmic bytes: fwd reads x, writes y + uint8 argmax; bwd reads dy + argmax, writes dx
    nx, ny = x.numel() * 2, dy.numel() * 2
    print(f"roofline @6.5 TB/s: fwd {(nx + ny + ny / 2) / 6.5e9:.3f} ms, bwd {(ny + ny / 2 + nx) / 6.5e9:.3f} ms")


if __name__ == "__main__":
    main()
