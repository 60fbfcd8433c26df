"""Config-2 update parity: the ResNet-50 bucket through K2 vs torch.optim.SGD, bit for bit.

Reference: the update rule is equivalence.sgd_step (equivalence.py:163-168) extended with
torch.optim.SGD's momentum / weight decay (SgdSettings, fusion.py); the payload is the fused
gradient of workload.fuse_gradients (workload.py:94-101).  The bucket here is the real config-2
one: 161 tensors, channels_last conv weights, CUDA-graph static gradients (or eager autograd
gradients through the GEMM stem, whose dW layout once differed from the weight's), updated in
place by K2 (direct mode: straight from the gradient tensors; bucket mode: K1 pack first).
After every slot the test reads the app's gradients and parameters and replays
torch.optim.SGD(foreach=False) on the CPU: parameters and momentum buffers must be identical.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _replay_and_compare(sched, apps, sgd, world_grads=None):
    before = {a.job_id: [p.detach().cpu().clone() for p in a.params] for a in apps}
    bufs = {a.job_id: None for a in apps}
    mism = {}
    while True:
        st = sched._next_with_work()
        if st is None:
            break
        sched.step()
        torch.cuda.synchronize()     # graphed grads are rewritten by the app's next replay
        grads = [g.detach().cpu().clone() for g in st.held[0]]
        after = [p.detach().cpu().clone() for p in st.app.params]
        params = [torch.nn.Parameter(p.clone()) for p in before[st.job_id]]
        opt = torch.optim.SGD(params, lr=sgd.lr, momentum=sgd.momentum, weight_decay=sgd.weight_decay,
                              foreach=False)
        if bufs[st.job_id] is not None:
            for p, b in zip(params, bufs[st.job_id]):
                opt.state[p]["momentum_buffer"] = b
        for p, g in zip(params, grads):
            p.grad = g.clone()
        opt.step()
        bufs[st.job_id] = [opt.state[p]["momentum_buffer"] for p in params]
        key = f"{st.job_id}_t{st.next_iteration - 1}"
        mism[key] = sum(int((a.view(torch.int32) != p.detach().view(torch.int32)).sum())
                        for a, p in zip(after, params))
        # K2's momentum buffers (direct / bucket modes keep one per parameter)
        mb = st.sync.momentum_bufs
        if mb is not None and len(mb) == len(params):
            mism[key + "_momentum"] = sum(
                int((m.cpu().view(torch.int32) != b.view(torch.int32)).sum())
                for m, b in zip(mb, bufs[st.job_id]))
        before[st.job_id] = after
    sched.drain()
    return mism


@pytest.mark.parametrize("mode", ["direct", "bucket"])
def test_resnet50_graphed_update_bitwise_torch_sgd(cuda_device, mode):
    from paper_2103_07974_b200.apps import DEFAULT_IMAGE_SGD, resnet50_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    apps = [resnet50_app(f"r{j}", 32, 3, cuda_device, seed=j, graphed=True, fast_bn=True)
            for j in range(2)]
    assert len(apps[0].params) == 161
    s = CrossoverScheduler(Policy.CROSSOVER, sync_mode=mode)
    for a in apps:
        s.register(a)
    assert {st.sync.mode for st in s.states} == {mode}
    mism = _replay_and_compare(s, apps, DEFAULT_IMAGE_SGD)
    assert len(mism) >= 6 and all(v == 0 for v in mism.values()), mism


def test_resnet50_eager_gemm_stem_update_bitwise_torch_sgd(cuda_device):
    """Eager autograd gradients (the GEMM stem's dW included) through direct-mode K2."""
    from paper_2103_07974_b200.apps import DEFAULT_IMAGE_SGD, resnet50_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    apps = [resnet50_app(f"e{j}", 16, 3, cuda_device, seed=10 + j, graphed=False, fast_bn=True,
                         stem="gemm") for j in range(2)]
    w = apps[0].model.conv1.weight
    s = CrossoverScheduler(Policy.CROSSOVER)
    for a in apps:
        s.register(a)
    mism = _replay_and_compare(s, apps, DEFAULT_IMAGE_SGD)
    assert all(v == 0 for v in mism.values()), mism
    # the stem's gradient now comes back in the weight's own layout (no re-layout copy in K2's path)
    x = torch.randn(2, 3, 64, 64, device=cuda_device, dtype=torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        y = apps[0].model.conv1(x)
    (g,) = torch.autograd.grad(y.float().sum(), [w])
    assert g.stride() == w.stride()


def test_resnet50_eager_crossover_equals_sequential_bitwise(cuda_device):
    """Crossover adds no staleness on the eager config-2 path (GEMM stem, NHWC BN, deterministic
    cuDNN): the weights after 3 iterations of both apps equal the sequential baseline's bit for
    bit -- any stream race on the gradients (e.g. a gradient freed to the next app's forward
    before the comm stream read it) would show up here."""
    from paper_2103_07974_b200.apps import resnet50_app
    from paper_2103_07974_b200.scheduler import CrossoverScheduler, Policy

    old = torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
    try:
        out = {}
        for pol in (Policy.CROSSOVER, Policy.SEQUENTIAL):
            apps = [resnet50_app(f"e{j}", 16, 3, cuda_device, seed=20 + j, graphed=False, fast_bn=True,
                                 stem="gemm") for j in range(2)]
            s = CrossoverScheduler(pol)
            for a in apps:
                s.register(a)
            s.run()
            out[pol] = [torch.cat([p.detach().reshape(-1) for p in a.params]).cpu() for a in apps]
        for a, b in zip(out[Policy.CROSSOVER], out[Policy.SEQUENTIAL]):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    finally:
        torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = old
