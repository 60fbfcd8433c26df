"""ResNet-50 stem convolution (7x7/2, 64 filters) fwd + wgrad at bs 256, channels_last bf16:
3 input channels (cuDNN pads internally and falls back to sm80-era kernels) vs the input and the
weight zero-padded to 4 / 8 channels (numerically the same convolution).

    python tools/stem_bench.py
"""
import statistics

import torch
import torch.nn.functional as F


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
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2103_07974_b200.stem import _StemGemm

    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    x3 = torch.randn(256, 3, 224, 224, device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    w3 = torch.randn(64, 3, 7, 7, device=dev, dtype=torch.float32, requires_grad=True)
    dy = torch.randn(256, 64, 112, 112, device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    for cin in (3, 4, 8):
        def step():
            if cin == 3:
                x, w = x3, w3
            else:
                x = x3.new_empty((256, 224, 224, cin)).permute(0, 3, 1, 2)
                x[:, 3:] = 0
                x[:, :3] = x3
                w = F.pad(w3, (0, 0, 0, 0, 0, cin - 3))
            with torch.autocast("cuda", dtype=torch.bfloat16):
                y = F.conv2d(x, w, stride=2, padding=3)
            y.backward(dy)
        ms = timeit(step)
        y = None
        with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
            ref = F.conv2d(x3, w3, stride=2, padding=3)
            x8 = x3.new_empty((256, 224, 224, cin)).permute(0, 3, 1, 2)
            x8[:, 3:] = 0
            x8[:, :3] = x3
            out = F.conv2d(x8, F.pad(w3, (0, 0, 0, 0, 0, cin - 3)), stride=2, padding=3)
        print(f"cin={cin}: fwd+wgrad {ms:.3f} ms  max|y - y3| = {float((out.float() - ref.float()).abs().max()):.3g}")

    def gemm_step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = _StemGemm.apply(x3, w3, None, (2, 2), (3, 3))
        y.backward(dy)
    ms = timeit(gemm_step)
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
        ref = F.conv2d(x3, w3, stride=2, padding=3)
        out = _StemGemm.apply(x3, w3, None, (2, 2), (3, 3))
    print(f"gemm stem: fwd+wgrad {ms:.3f} ms  max|y - y3| = {float((out.float() - ref.float()).abs().max()):.3g}")


if __name__ == "__main__":
    main()
