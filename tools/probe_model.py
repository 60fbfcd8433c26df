"""Probe the per-iteration forward+backward time of the apps' model compute (device-timed).

Variants: memory format (channels_last / NCHW), eager vs CUDA-graph capture.
"""
import statistics
import sys
import time
from pathlib import Path

import torch
import torch.nn.functional as F

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run(model_name="resnet50", batch=256, fmt="cl", graph=False, iters=10, fast_bn=False, fuse=False):
    import torchvision

    dev = torch.device("cuda", 0)
    torch.backends.cudnn.benchmark = True
    m = getattr(torchvision.models, model_name)()
    if fast_bn:
        from paper_2103_07974_b200.bn import fuse_resnet, swap_batchnorm
        swap_batchnorm(m)
        if fuse:
            fuse_resnet(m)
    m = m.to(dev)
    mf = torch.channels_last if fmt == "cl" else torch.contiguous_format
    m = m.to(memory_format=mf)
    params = [p for p in m.parameters()]
    x = torch.randn(batch, 3, 224, 224, device=dev, dtype=torch.bfloat16).contiguous(memory_format=mf)
    y = torch.randint(0, 1000, (batch,), device=dev)
    s = torch.cuda.Stream()

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=not graph):
            loss = F.cross_entropy(m(x), y)
        return torch.autograd.grad(loss, params)

    with torch.cuda.stream(s):
        for _ in range(3):
            g = step()
    torch.cuda.synchronize()
    if graph:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            g = step()
        fn = gr.replay
    else:
        fn = step
    ts = []
    cpu = []
    with torch.cuda.stream(s):
        for _ in range(iters):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            t0 = time.perf_counter()
            fn()
            cpu.append((time.perf_counter() - t0) * 1e3)
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b))
    return statistics.median(ts), statistics.median(cpu)


if __name__ == "__main__":
    for model in sys.argv[1:] or ["resnet50"]:
        for fmt, graph, fast, fuse in (("cl", True, False, False), ("cl", True, True, False), ("cl", True, True, True)):
                try:
                    gpu, cpu = run(model, fmt=fmt, graph=graph, fast_bn=fast, fuse=fuse)
                    print(f"{model} graph={graph} fast_bn={fast} fused={fuse}: {gpu:.2f} ms/iter GPU, {cpu:.2f} ms host issue, "
                          f"{256 / gpu * 1e3:.0f} img/s", flush=True)
                except Exception as e:  # noqa: BLE001
                    print(f"{model} fmt={fmt} graph={graph}: FAILED {type(e).__name__}: {str(e)[:200]}", flush=True)
