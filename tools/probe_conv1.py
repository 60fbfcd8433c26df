"""Probe: ResNet stem conv (7x7/2, 64 out) fwd + wgrad with the input channels padded 3 -> 4 / 8."""
import statistics
import torch
import torch.nn.functional as F

dev = torch.device("cuda", 0)
torch.backends.cudnn.benchmark = True
cl = torch.channels_last
for cin in (3, 4, 8):
    x = torch.randn(256, cin, 224, 224, device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
    w = torch.randn(64, cin, 7, 7, device=dev, dtype=torch.bfloat16, requires_grad=True).contiguous(memory_format=cl)
    dy = torch.randn(256, 64, 112, 112, device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)

    def step():
        y = F.conv2d(x, w, stride=2, padding=3)
        torch.autograd.grad(y, w, dy)
    for _ in range(5):
        step()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    print(f"cin={cin}: conv1 fwd+wgrad {statistics.median(ts):.3f} ms", flush=True)
