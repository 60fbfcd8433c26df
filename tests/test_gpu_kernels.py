"""Parity of the sm_100a kernels (K1 pack, K2 reduce+average+SGD, K3 stats) -- ladder L0/L1.

Every comparison is BIT-EXACT (int32 views), against the CPU oracle
(oracle/fusion.py) for the reference rounding and against torch.optim.SGD on
the CPU for the torch (momentum) rounding.
"""

import numpy as np
import pytest
import torch

from oracle import fusion as ofusion

pytestmark = pytest.mark.gpu

RAGGED = [0, 1, 3, 4, 5, 17, 64, 4095, 4096, 4097, 12345, 200704, 256, 2560, 10]


@pytest.fixture(autouse=True)
def _needs_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _bits(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float32).view(np.int32)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _sync_obj(params, **kw):
    from paper_2103_07974_b200.fusion import FusedGradientSync, SgdSettings

    sgd = kw.pop("sgd", SgdSettings(0.05))
    return FusedGradientSync(params, sgd, **kw)


@pytest.mark.parametrize("align", [1, 4, 32])
def test_pack_bitexact_ragged(cuda_device, align):
    torch.manual_seed(0)
    grads = [torch.randn(n, device=cuda_device) for n in RAGGED]
    params = [torch.zeros(n, device=cuda_device) for n in RAGGED]
    s = _sync_obj(params, local_workers=2, align=align, mode="bucket")
    grads2 = [torch.randn(n, device=cuda_device) for n in RAGGED]
    s.pack([grads, grads2], _stream())
    torch.cuda.synchronize()
    want0 = ofusion.pack([g.cpu().numpy() for g in grads], align)
    want1 = ofusion.pack([g.cpu().numpy() for g in grads2], align)
    got = s.bucket.view(2, -1)
    assert np.array_equal(_bits(got[0]), _bits(want0))
    assert np.array_equal(_bits(got[1]), _bits(want1))
    if align == 1:  # exact reference layout == torch.cat
        assert torch.equal(got[0][:sum(RAGGED)], torch.cat(grads))


def test_pack_many_tensors_and_misaligned_sources(cuda_device):
    torch.manual_seed(1)
    sizes = [int(x) for x in np.random.default_rng(3).integers(0, 3000, 700)]
    big = torch.randn(sum(sizes) + 700, device=cuda_device)
    grads, cur = [], 1                               # offset 1 element -> not 16B aligned
    for n in sizes:
        grads.append(big[cur:cur + n])
        cur += n + 1
    params = [torch.zeros(n, device=cuda_device) for n in sizes]
    s = _sync_obj(params, local_workers=2, align=4, mode="bucket")
    aligned = [torch.randn(n, device=cuda_device) for n in sizes]
    s.pack([grads, aligned], _stream())             # > 512 descriptors -> several launches
    torch.cuda.synchronize()
    got = s.bucket.view(2, -1)
    assert np.array_equal(_bits(got[0]), _bits(ofusion.pack([g.cpu().numpy() for g in grads], 4)))
    assert np.array_equal(_bits(got[1]), _bits(ofusion.pack([g.cpu().numpy() for g in aligned], 4)))


@pytest.mark.parametrize("nsrc", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("align", [1, 32])
def test_reduce_update_reference_rounding(cuda_device, nsrc, align):
    torch.manual_seed(nsrc)
    params = [torch.randn(n, device=cuda_device) for n in RAGGED]
    p0 = [p.cpu().numpy().copy() for p in params]
    s = _sync_obj(params, local_workers=nsrc, align=align, mode="bucket")
    grads = [[torch.randn(n, device=cuda_device) * (w + 1) for n in RAGGED] for w in range(nsrc)]
    s.pack(grads, _stream())
    rows = s.bucket.view(nsrc, -1).cpu().numpy()
    s.update(_stream())
    torch.cuda.synchronize()
    want = ofusion.reduce_update(p0, list(rows), s.layout.offsets, 0.05, nsrc)
    for got, w in zip(params, want):
        assert np.array_equal(_bits(got), _bits(w))


def test_direct_mode_equals_bucket_mode(cuda_device):
    torch.manual_seed(7)
    base = [torch.randn(n, device=cuda_device) for n in RAGGED]
    pa = [b.clone() for b in base]
    pb = [b.clone() for b in base]
    grads = [torch.randn(n, device=cuda_device) for n in RAGGED]
    a = _sync_obj(pa, mode="bucket")
    b = _sync_obj(pb, mode="direct")
    a.sync([grads], _stream())
    b.sync([grads], _stream())
    torch.cuda.synchronize()
    for x, y in zip(pa, pb):
        assert torch.equal(x, y)


@pytest.mark.parametrize("momentum,dampening,wd,nesterov", [
    (0.9, 0.0, 0.0, False), (0.9, 0.0, 1e-4, False), (0.9, 0.0, 5e-4, True),
    (0.5, 0.1, 0.0, False), (0.0, 0.0, 1e-2, False)])
def test_torch_rounding_matches_torch_sgd(cuda_device, momentum, dampening, wd, nesterov):
    """K2 (torch rounding) == torch.optim.SGD (fp32, CPU, single-tensor) bit for bit."""
    from paper_2103_07974_b200.fusion import SgdSettings

    sizes = [1024, 4096, 4112, 65536, 160]            # multiples of 16: fully vectorised on CPU too
    torch.manual_seed(11)
    ref = [torch.nn.Parameter(torch.randn(n)) for n in sizes]
    dev = [p.detach().to(cuda_device).clone() for p in ref]
    opt = torch.optim.SGD(ref, lr=0.05, momentum=momentum, dampening=dampening,
                          weight_decay=wd, nesterov=nesterov, foreach=False)
    sgd = SgdSettings(0.05, momentum=momentum, dampening=dampening, weight_decay=wd,
                      nesterov=nesterov, rounding="torch")
    s = _sync_obj(dev, sgd=sgd, mode="direct")
    for step in range(3):
        g = [torch.randn(n) for n in sizes]
        for p, gi in zip(ref, g):
            p.grad = gi.clone()
        opt.step()
        s.sync([[gi.to(cuda_device) for gi in g]], _stream())
        torch.cuda.synchronize()
        for r, d in zip(ref, dev):
            assert np.array_equal(_bits(r), _bits(d)), f"step {step}"


def test_snapshot_rows_capture_weights(cuda_device):
    params = [torch.randn(n, device=cuda_device) for n in [10, 33, 4096]]
    s = _sync_obj(params, mode="direct", snapshot_rows=2, align=4)
    for row in range(2):
        s.update(_stream(), [torch.randn_like(p) for p in params], snapshot_row=row)
        torch.cuda.synchronize()
        for p, o in zip(params, s.layout.offsets):
            assert torch.equal(s.snapshot[row, o:o + p.numel()], p)


def test_channels_last_parameters(cuda_device):
    w = torch.randn(8, 3, 5, 5, device=cuda_device).contiguous(memory_format=torch.channels_last)
    g = torch.randn_like(w)                        # preserves channels_last strides
    w0 = w.clone()
    s = _sync_obj([w], mode="bucket")
    s.sync([[g]], _stream())
    torch.cuda.synchronize()
    f = np.float32
    want = w0.cpu().numpy() - f(0.05) * (g.cpu().numpy() / f(1))
    assert np.array_equal(_bits(w.cpu().numpy()), _bits(want))


def test_gradient_stats(cuda_device):
    from paper_2103_07974_b200 import _lib

    x = torch.randn(1_000_003, device=cuda_device)
    x[17] = float("nan")
    x[99] = float("inf")
    ws = torch.zeros(_lib.gradient_stats_workspace_bytes(x.numel()), dtype=torch.uint8,
                     device=cuda_device)
    outs = []
    for view in (x, x[1:]):                        # aligned and misaligned base
        out = torch.zeros(2, dtype=torch.float64, device=cuda_device)
        _lib.gradient_stats(view.data_ptr(), view.numel(), out.data_ptr(), ws.data_ptr(), _stream())
        torch.cuda.synchronize()
        v = view.cpu().numpy().astype(np.float64)
        fin = np.isfinite(v)
        assert out[1].item() == float((~fin).sum())
        assert out[0].item() == pytest.approx(float(np.sum(v[fin] ** 2)), rel=1e-12)
        outs.append(out.cpu())
    out2 = torch.zeros(2, dtype=torch.float64, device=cuda_device)
    _lib.gradient_stats(x.data_ptr(), x.numel(), out2.data_ptr(), ws.data_ptr(), _stream())
    torch.cuda.synchronize()
    assert torch.equal(out2.cpu(), outs[0])        # deterministic


def test_guard_bands_untouched(cuda_device):
    """Out-of-bounds write detector (compute-sanitizer is closed on this pool): every tensor,
    the bucket and the momentum buffers live inside one sentinel-filled arena with gaps; after
    K1 + K2 the gaps must still hold the sentinel bit pattern."""
    from paper_2103_07974_b200.fusion import FusedGradientSync, SgdSettings

    sizes = [1, 3, 5, 4095, 4097, 12345, 10, 0, 7]
    gap = 37
    total = sum(sizes) * 4 + gap * (4 * len(sizes) + 2)
    arena = torch.full((total,), float("nan"), device=cuda_device)
    sentinel = arena.clone()
    views, cur = {"p": [], "g": []}, gap
    for kind in ("p", "g"):
        for n in sizes:
            v = arena[cur:cur + n]
            v.copy_(torch.randn(n, device=cuda_device))
            views[kind].append(v)
            cur += n + gap
    used = torch.zeros(total, dtype=torch.bool, device=cuda_device)
    for kind in ("p", "g"):
        for v in views[kind]:
            off = (v.data_ptr() - arena.data_ptr()) // 4
            used[off:off + v.numel()] = True
    s = FusedGradientSync(views["p"], SgdSettings(0.01, momentum=0.9, weight_decay=1e-3), mode="direct")
    for _ in range(2):
        s.sync([views["g"]], _stream())
    sb = FusedGradientSync(views["p"], SgdSettings(0.01), mode="bucket", align=1)
    sb.sync([views["g"]], _stream())
    torch.cuda.synchronize()
    a = arena.view(torch.int32)[~used]
    b = sentinel.view(torch.int32)[~used]
    assert torch.equal(a, b)
    assert torch.isfinite(torch.cat([v for v in views["p"] if v.numel()])).all()


@pytest.mark.parametrize("variant", ["registers", "bulk"])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_p2p_kernel_emulated_ranks(cuda_device, world, momentum, variant):
    """The fused P2P kernel with every 'peer' address pointing at local memory (one GPU emulates
    W ranks): rank-order sum, /W, SGD, and the broadcast into all W destinations, bit-exact
    against the same arithmetic (reference rounding) / torch-SGD rounding on the CPU.  "bulk" is
    the capped-grid variant that streams tiles through shared memory with cp.async.bulk (TMA)."""
    import ctypes

    from paper_2103_07974_b200 import _lib

    torch.manual_seed(world)
    shard = 4096 * 3 + 8                                  # not a multiple of the chunk: tail path
    srcs = [torch.randn(shard, device=cuda_device) for _ in range(world)]
    p = torch.randn(shard, device=cuda_device)
    dsts = [torch.zeros(shard, device=cuda_device) for _ in range(world)]
    mom = torch.randn(shard, device=cuda_device) if momentum else None
    d = _lib.P2PDesc()
    for r in range(world):
        d.src[r] = srcs[r].data_ptr()
        d.dst[r] = dsts[r].data_ptr()
    d.param, d.numel, d.nranks = p.data_ptr(), shard, world
    d.momentum_buf = mom.data_ptr() if mom is not None else None
    h = _lib.SgdHyper(lr=0.05, momentum=momentum, dampening_complement=1.0, divisor=world,
                      first_step=0, rounding=_lib.CS_ROUND_TORCH if momentum else _lib.CS_ROUND_REFERENCE)
    p0, m0 = p.cpu().clone(), (mom.cpu().clone() if mom is not None else None)
    d.max_ctas = 1                                        # one CTA walks every tile: the stage ring wraps
    _lib.tune("p2p_bulk", 1 if variant == "bulk" else 0)
    try:
        _lib.check("p2p", _lib.lib.cs_p2p_reduce_sgd_bcast(ctypes.byref(d), ctypes.byref(h), _stream()))
        torch.cuda.synchronize()
    finally:
        _lib.tune("p2p_bulk", 1)
    acc = torch.zeros(shard)
    for sr in srcs:
        acc = acc + sr.cpu()                              # rank order, fp32, one rounding per add
    avg = acc / world
    if momentum:
        # torch.optim.SGD itself on the CPU (foreach=False): buf = 0.9 buf + g, p -= lr buf
        q = torch.nn.Parameter(p0.clone())
        opt = torch.optim.SGD([q], lr=0.05, momentum=0.9, foreach=False)
        opt.state[q]["momentum_buffer"] = m0.clone()
        q.grad = avg
        opt.step()
        assert torch.equal(mom.cpu(), opt.state[q]["momentum_buffer"])
        assert torch.equal(dsts[0].cpu(), q.detach())
    else:
        want = p0 - torch.tensor(0.05, dtype=torch.float32) * avg
        assert torch.equal(dsts[0].cpu(), want)
    for r in range(1, world):
        assert torch.equal(dsts[r], dsts[0])              # the fused all-gather wrote every rank


def test_pack_by_copy_engines_equals_kernel(cuda_device):
    """K1 by the copy engines (one DMA per tensor, pack_engine='ce') == the pack kernel, bitwise,
    including ragged / misaligned tensors (the bucket's padding stays zero either way)."""
    from paper_2103_07974_b200.fusion import FusedGradientSync, SgdSettings

    torch.manual_seed(5)
    params = [torch.randn(n, device=cuda_device) for n in RAGGED if n]
    grads = [torch.randn_like(p) for p in params]
    out = {}
    for eng in ("sm", "ce"):
        s = FusedGradientSync(params, SgdSettings(0.1), mode="bucket", local_workers=1, pack_engine=eng)
        s.pack([grads], _stream())
        torch.cuda.synchronize()
        out[eng] = s.bucket.clone()
    assert torch.equal(out["sm"].view(torch.int32), out["ce"].view(torch.int32))
