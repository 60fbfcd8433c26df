"""NHWC BatchNorm kernels (apps' compute) vs torch.nn.functional.batch_norm in fp32."""

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

SHAPES = [(8, 64, 56, 56), (4, 256, 14, 14), (2, 2048, 7, 7), (16, 24, 5, 5), (3, 512, 9, 9),
          (2, 8, 1, 1), (64, 1024, 2, 3)]


@pytest.mark.parametrize("shape", SHAPES)
def test_bn_forward_backward_matches_torch(cuda_device, shape):
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d

    torch.manual_seed(sum(shape))
    n, c, h, w = shape
    x = (torch.randn(shape, device=cuda_device) * 3 + 1.5).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    dy = torch.randn(shape, device=cuda_device).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    bn = CrossoverBatchNorm2d(c).to(cuda_device)
    with torch.no_grad():
        bn.weight.copy_(torch.rand(c) + 0.5)
        bn.bias.copy_(torch.randn(c))
        bn.running_var.fill_(2.0)
    ref = torch.nn.BatchNorm2d(c).to(cuda_device)
    ref.load_state_dict(bn.state_dict())
    xa = x.detach().clone().requires_grad_(True)
    xb = x.detach().float().clone().requires_grad_(True)
    y = bn(xa)
    yr = ref(xb)
    assert y.dtype == torch.bfloat16 and y.is_contiguous(memory_format=torch.channels_last)
    torch.testing.assert_close(y.float(), yr.to(torch.bfloat16).float(), rtol=2e-2, atol=3e-2)
    y.backward(dy)
    yr.backward(dy.float())
    scale = xb.grad.abs().max().item()
    torch.testing.assert_close(xa.grad.float(), xb.grad, rtol=2e-2, atol=2e-2 * scale + 1e-6)
    for a, b in ((bn.weight.grad, ref.weight.grad), (bn.bias.grad, ref.bias.grad)):
        torch.testing.assert_close(a, b, rtol=2e-3, atol=1e-3 * b.abs().max().item() + 1e-4)
    torch.testing.assert_close(bn.running_mean, ref.running_mean, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(bn.running_var, ref.running_var, rtol=1e-4, atol=1e-5)
    assert int(bn.num_batches_tracked) == int(ref.num_batches_tracked) == 1


def test_bn_deterministic_and_graph_capturable(cuda_device):
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d

    bn = CrossoverBatchNorm2d(128).to(cuda_device)
    x = torch.randn(32, 128, 28, 28, device=cuda_device).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    y1 = bn(x)
    y2 = bn(x)
    assert torch.equal(y1, y2)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        bn(x)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        yg = bn(x)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(yg, y1)


def test_bn_fallbacks(cuda_device):
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d, swap_batchnorm

    bn = CrossoverBatchNorm2d(20).to(cuda_device)          # C % 8 != 0 -> ATen path
    x = torch.randn(4, 20, 6, 6, device=cuda_device).to(torch.bfloat16)
    ref = torch.nn.BatchNorm2d(20).to(cuda_device)
    torch.testing.assert_close(bn(x).float(), ref(x).float(), rtol=1e-2, atol=1e-2)
    bn.eval()
    assert bn(x).shape == x.shape
    import torchvision

    m = torchvision.models.resnet50()
    assert swap_batchnorm(m) == 53
    assert isinstance(m.bn1, CrossoverBatchNorm2d)
    assert sum(p.numel() for p in m.parameters()) == 25_557_032


def test_resnet50_fast_bn_graphed_pipeline(cuda_device):
    from paper_2103_07974_b200.apps import resnet50_app
    from paper_2103_07974_b200.engine import validate_trace
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    s = CrossoverScheduler(Policy.CROSSOVER)
    for k in range(2):
        s.register(resnet50_app(f"b{k}", 16, 3, cuda_device, seed=k, graphed=True, fast_bn=True))
    tr = s.run()
    assert validate_trace(tr) == []
    losses = [float(l) for st in s.states for l in st.losses]
    assert all(0 < l < 20 for l in losses)


@pytest.mark.parametrize("relu,residual", [(True, False), (True, True), (False, True)])
def test_bn_fused_epilogues_match_torch(cuda_device, relu, residual):
    from paper_2103_07974_b200.bn import CrossoverBatchNorm2d

    torch.manual_seed(3)
    shape = (8, 256, 14, 14)
    c = shape[1]
    cl = dict(memory_format=torch.channels_last)
    x = torch.randn(shape, device=cuda_device).to(torch.bfloat16).contiguous(**cl)
    r = torch.randn(shape, device=cuda_device).to(torch.bfloat16).contiguous(**cl)
    dy = torch.randn(shape, device=cuda_device).to(torch.bfloat16).contiguous(**cl)
    bn = CrossoverBatchNorm2d(c).to(cuda_device)
    ref = torch.nn.BatchNorm2d(c).to(cuda_device)
    xa, ra = x.clone().requires_grad_(True), r.clone().requires_grad_(True)
    xb, rb = x.float().requires_grad_(True), r.float().requires_grad_(True)
    y = bn.forward_fused(xa, relu=relu, residual=ra if residual else None)
    yr = ref(xb) + (rb if residual else 0)
    if relu:
        yr = torch.relu(yr)
    torch.testing.assert_close(y.float(), yr.to(torch.bfloat16).float(), rtol=2e-2, atol=3e-2)
    y.backward(dy)
    yr.backward(dy.float())
    sc = xb.grad.abs().max().item()
    torch.testing.assert_close(xa.grad.float(), xb.grad, rtol=2e-2, atol=2e-2 * sc + 1e-6)
    if residual:
        torch.testing.assert_close(ra.grad.float(), rb.grad, rtol=1e-2, atol=1e-2)
    torch.testing.assert_close(bn.weight.grad, ref.weight.grad, rtol=5e-3,
                               atol=2e-3 * ref.weight.grad.abs().max().item() + 1e-4)


def test_fused_resnet_no_less_accurate_than_aten(cuda_device):
    """Whole ResNet-50 in bf16: a random-init net's early-layer gradients are ill-conditioned
    (ATen bf16 itself is O(1) off the fp32 gradients there), so the bar is relative: our
    swapped and fused BN models must be as close to the fp32 reference as ATen's bf16 run."""
    import copy

    import torchvision

    from paper_2103_07974_b200.bn import fuse_resnet, swap_batchnorm

    torch.manual_seed(0)
    m_swap = torchvision.models.resnet50()
    swap_batchnorm(m_swap)
    m_fused = copy.deepcopy(m_swap)
    assert fuse_resnet(m_fused) == 16
    from paper_2103_07974_b200.bn import CrossoverMaxPool2d
    assert isinstance(m_fused.maxpool, CrossoverMaxPool2d)
    aten = torchvision.models.resnet50()
    aten.load_state_dict(m_swap.state_dict())
    aten32 = copy.deepcopy(aten)
    x = torch.randn(16, 3, 224, 224, device=cuda_device).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    keys = ["conv1.weight", "layer1.0.conv1.weight", "layer3.0.bn1.weight", "layer4.2.bn3.weight",
            "fc.weight", "fc.bias"]
    res = []
    for m, amp in ((aten32, False), (aten, True), (m_swap, True), (m_fused, True)):
        m = m.to(cuda_device).to(memory_format=torch.channels_last)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=amp):
            loss = m(x if amp else x.float()).float().square().mean()
        named = dict(m.named_parameters())
        g = torch.autograd.grad(loss, [named[k] for k in keys])
        res.append((loss.item(), g))
    for k in range(len(keys)):
        ref = res[0][1][k].float()
        sc = ref.abs().max().item()
        err = [((r[1][k].float() - ref).abs().max().item()) / sc for r in res[1:]]
        assert err[1] <= 1.5 * err[0] + 0.05 and err[2] <= 1.5 * err[0] + 0.05, (keys[k], err)
    assert abs(res[2][0] - res[0][0]) <= 2 * abs(res[1][0] - res[0][0]) + 1e-3
    assert abs(res[3][0] - res[0][0]) <= 2 * abs(res[1][0] - res[0][0]) + 1e-3


@pytest.mark.parametrize("shape,k,s,p", [((8, 64, 112, 112), 3, 2, 1), ((2, 64, 9, 7), 3, 2, 1),
                                         ((2, 64, 10, 12), 3, 2, 1),
                                         ((4, 16, 9, 7), 3, 2, 1),
                                         ((2, 8, 10, 10), 2, 2, 0), ((3, 24, 11, 13), 3, 1, 1)])
def test_maxpool_matches_aten_exactly(cuda_device, shape, k, s, p):
    from paper_2103_07974_b200.bn import CrossoverMaxPool2d

    torch.manual_seed(1)
    x = torch.randn(shape, device=cuda_device).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    x[0, 0, 0, :4] = 0.0          # ties: the first maximum in scan order wins (ATen's rule)
    x[0, 1, :3, :3] = 1.0
    dy = torch.randn((shape[0], shape[1], (shape[2] + 2 * p - k) // s + 1, (shape[3] + 2 * p - k) // s + 1),
                     device=cuda_device).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    xa, xb = x.clone().requires_grad_(True), x.clone().requires_grad_(True)
    ya = CrossoverMaxPool2d(k, s, p)(xa)
    yb = torch.nn.functional.max_pool2d(xb, k, s, p)
    assert torch.equal(ya, yb)
    ya.backward(dy)
    yb.backward(dy)
    torch.testing.assert_close(xa.grad.float(), xb.grad.float(), rtol=1e-2, atol=1e-2)
    assert torch.equal(xa.grad != 0, xb.grad != 0)      # same selected positions


@pytest.mark.parametrize("cfg", [dict(k=7, s=2, p=3, bias=False, hw=32),    # ResNet stem
                                 dict(k=7, s=2, p=3, bias=False, hw=33),    # rows not 16-B multiple
                                 dict(k=3, s=1, p=1, bias=True, hw=24),     # VGG stem
                                 dict(k=5, s=3, p=2, bias=True, hw=17)])    # generic shape path
def test_gemm_stem_matches_conv(cuda_device, cfg):
    """The RGB stem as im2col + GEMMs (stem.py) vs F.conv2d in fp32: output at bf16 rounding,
    weight / bias gradients at the tolerance of a bf16 GEMM over N*OH*OW terms."""
    import torch.nn.functional as F

    from paper_2103_07974_b200.stem import gemm_stem

    torch.manual_seed(0)
    conv = torch.nn.Conv2d(3, 64, cfg["k"], stride=cfg["s"], padding=cfg["p"], bias=cfg["bias"]).to(cuda_device)
    ref = torch.nn.Conv2d(3, 64, cfg["k"], stride=cfg["s"], padding=cfg["p"], bias=cfg["bias"]).to(cuda_device)
    ref.load_state_dict(conv.state_dict())
    assert gemm_stem(conv) == 1
    x = torch.randn(4, 3, cfg["hw"], cfg["hw"], device=cuda_device).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        y = conv(x)
    y_ref = F.conv2d(x.float(), ref.weight, ref.bias, stride=cfg["s"], padding=cfg["p"])
    assert y.shape == y_ref.shape and y.dtype == torch.bfloat16
    assert y.is_contiguous(memory_format=torch.channels_last)
    torch.testing.assert_close(y.float(), y_ref, rtol=2e-2, atol=2e-2)
    dy = torch.randn_like(y_ref).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    y.backward(dy)
    y_ref.backward(dy.float())
    torch.testing.assert_close(conv.weight.grad, ref.weight.grad, rtol=2e-2, atol=0.5)
    if cfg["bias"]:
        torch.testing.assert_close(conv.bias.grad, ref.bias.grad, rtol=1e-2, atol=0.1)
    assert conv.weight.grad.dtype == torch.float32
    # the output is a base tensor: an in-place consumer (VGG's ReLU(inplace=True)) is legal
    with torch.autocast("cuda", dtype=torch.bfloat16):
        z = torch.relu_(conv(x))
    z.float().sum().backward()


def test_side_gradient_replaces_autograd_add(cuda_device):
    """ResNet-50 with the identity gradients delivered to the producing BN (cs_bn_backward2, dy +
    dy2 summed in fp32) vs the same model where autograd sums them (one bf16 add per block): the
    same forward, and gradients no further from an fp32 model's than the autograd-add run's
    (early-layer gradients of a random-init bf16 ResNet are ill-conditioned, so the bar is
    relative, as in test_fused_resnet_no_less_accurate_than_aten)."""
    import copy

    import torchvision

    from paper_2103_07974_b200 import bn as bnmod

    torch.manual_seed(0)
    ref = torchvision.models.resnet50()
    m = copy.deepcopy(ref)
    bnmod.swap_batchnorm(m)
    assert bnmod.fuse_resnet(m) == 16
    m2 = copy.deepcopy(m)
    x = torch.randn(8, 3, 64, 64, device=cuda_device).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    ref = ref.to(cuda_device).to(memory_format=torch.channels_last)
    g_ref = torch.autograd.grad(ref(x.float()).float().square().mean(), list(ref.parameters()))
    out = []
    saved = bnmod._SIDE_GRADS
    for model, side in ((m, True), (m2, False)):
        bnmod._SIDE_GRADS = side
        try:
            model = model.to(cuda_device).to(memory_format=torch.channels_last)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = model(x).float().square().mean()
            out.append((loss.item(), torch.autograd.grad(loss, list(model.parameters()))))
        finally:
            bnmod._SIDE_GRADS = saved
    (l1, g1), (l2, g2) = out
    assert l1 == l2                                  # the forward is unchanged
    for a, b, r in zip(g1, g2, g_ref):
        sc = r.abs().max().item() + 1e-12
        ea, eb = (a - r).abs().max().item() / sc, (b - r).abs().max().item() / sc
        assert ea <= 1.5 * eb + 0.05, (ea, eb)
