"""BN forward+backward of the small ResNet-50 layers, eager (launch- and finalize-bound shapes).

    python tools/finalize_bench.py
"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d

    dev = torch.device("cuda", 0)
    for shape in ((256, 64, 56, 56), (256, 256, 14, 14), (256, 512, 7, 7), (256, 2048, 7, 7)):
        x = torch.randn(shape, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        x.requires_grad_(True)
        dy = torch.randn_like(x)
        bn = CrossoverBatchNorm2d(shape[1]).to(dev)

        def step():
            bn(x).backward(dy)

        for _ in range(3):
            step()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); step(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        print(shape, f"{statistics.median(ts):.4f} ms")


if __name__ == "__main__":
    main()
