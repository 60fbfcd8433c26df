"""BatchNorm2d fwd+bwd: libcrossover.so NHWC kernels vs ATen, at ResNet-50 bs256 shapes."""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

SHAPES = [(256, 64, 112, 112), (256, 64, 56, 56), (256, 256, 56, 56), (256, 128, 28, 28),
          (256, 512, 28, 28), (256, 256, 14, 14), (256, 1024, 14, 14), (256, 512, 7, 7),
          (256, 2048, 7, 7)]


def timeit(fn, iters=10):
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
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d

    if "--no-pdl" in sys.argv:
        _lib.tune("bn_no_pdl", 1)
    for a in sys.argv[1:]:
        if a.startswith("--ctas-per-sm="):
            _lib.tune("bn_ctas_per_sm", int(a.split("=")[1]))

    dev = torch.device("cuda", 0)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    rows = []
    for shape in SHAPES:
        n, c, h, w = shape
        x = torch.randn(shape, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        dy = torch.randn_like(x)
        out = {"shape": shape}
        for name, mod in (("aten", torch.nn.BatchNorm2d(c)), ("ours", CrossoverBatchNorm2d(c))):
            mod = mod.to(dev)
            xr = x.detach().requires_grad_(True)

            def step():
                y = mod(xr)
                torch.autograd.grad(y, (xr, mod.weight, mod.bias), dy)
            # time the device work only: capture fwd+bwd in a CUDA graph
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for _ in range(3):
                    step()
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            out[name + "_ms"] = round(timeit(g.replay), 4)
        nbytes = x.numel() * 2 * 8      # fwd: read, read, write; bwd: read dy, x; read dy, x; write dx
        out["roofline_ms"] = round(nbytes / (peak * 1e9) * 1e3, 4)
        out["ours_frac_of_roofline"] = round(out["roofline_ms"] / out["ours_ms"], 3)
        out["speedup"] = round(out["aten_ms"] / out["ours_ms"], 2)
        rows.append(out)
        print(json.dumps(out), flush=True)
    outs = [a for a in sys.argv[1:] if not a.startswith("--")]
    if outs:
        Path(outs[0]).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
