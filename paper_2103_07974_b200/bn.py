"""channels_last BatchNorm2d for the apps' forward/backward, on libcrossover.so's BN kernels.

``swap_batchnorm(model)`` replaces every ``nn.BatchNorm2d`` by :class:`CrossoverBatchNorm2d`
(same parameters and buffers, same training semantics: batch statistics, biased variance for
normalisation, unbiased variance in the running estimate, ``momentum``, ``num_batches_tracked``).
In training mode on a bf16 CUDA input whose channel count the kernels support it runs
``cs_bn_forward`` / ``cs_bn_backward``; everything else (eval mode, fp32 inputs, odd channel
counts) goes through ``torch.nn.functional.batch_norm`` unchanged.  The kernels are graph-safe
(no host synchronisation; the per-module workspace keeps a fixed address).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

__all__ = ["CrossoverBatchNorm2d", "CrossoverMaxPool2d", "swap_batchnorm", "fuse_resnet",
           "bn_supported"]


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def bn_supported(x: torch.Tensor) -> bool:
    c = x.shape[1] if x.dim() == 4 else 0
    return (x.is_cuda and x.dtype == torch.bfloat16 and x.dim() == 4 and c % 8 == 0
            and (c <= 256 or c % 256 == 0))


CS_BN_RELU = 1
CS_BN_RESIDUAL = 2


class _SideGrad:
    """A gradient of a BN output delivered outside autograd.

    A bottleneck block's input x feeds both conv1 (an autograd edge) and the identity path into
    the block's bn3.  Autograd would sum the two gradients of x with one elementwise add per
    block; instead the identity edge is cut (``residual.detach()``), bn3's backward stores its
    residual gradient here, and the BN that produced x reads it as a second incoming gradient
    (``cs_bn_backward2``: dy + dy2 summed in fp32 inside its kernels).  The producer's backward
    always runs after bn3's (it needs conv1's input gradient, which bn3's backward precedes)."""

    __slots__ = ("grad",)

    def __init__(self):
        self.grad = None


class _BnFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, running_mean, running_var, momentum, eps, ws, residual, flags,
                side_in=None, side_out=None):
        n, c, h, w = x.shape
        m = n * h * w
        x = x.contiguous(memory_format=torch.channels_last)
        if residual is not None:
            residual = residual.contiguous(memory_format=torch.channels_last)
        y = torch.empty_like(x)
        f32 = dict(dtype=torch.float32, device=x.device)
        save_mean = torch.empty(c, **f32)
        save_invstd = torch.empty(c, **f32)
        scale_shift = torch.empty(2 * c, **f32)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check("cs_bn_forward", _lib.lib.cs_bn_forward(
            x.data_ptr(), _ptr(residual), m, c, _ptr(weight), _ptr(bias), _ptr(running_mean),
            _ptr(running_var), ctypes.c_float(momentum), ctypes.c_float(eps), save_mean.data_ptr(),
            save_invstd.data_ptr(), scale_shift.data_ptr(), y.data_ptr(), ws.data_ptr(), flags, stream))
        keep_res = residual if (flags & CS_BN_RELU and flags & CS_BN_RESIDUAL) else None
        ctx.save_for_backward(x, weight, save_mean, save_invstd, scale_shift, keep_res)
        ctx.ws, ctx.flags = ws, flags
        ctx.has_bias = bias is not None
        ctx.side_in, ctx.side_out = side_in, side_out
        return y

    @staticmethod
    def backward(ctx, dy):
        x, weight, save_mean, save_invstd, scale_shift, res = ctx.saved_tensors
        n, c, h, w = x.shape
        dy = dy.contiguous(memory_format=torch.channels_last)
        dy2 = None
        if ctx.side_in is not None and ctx.side_in.grad is not None:
            dy2 = ctx.side_in.grad.contiguous(memory_format=torch.channels_last)
            ctx.side_in.grad = None
        dx = torch.empty_like(x)
        dres = torch.empty_like(x) if ctx.flags & CS_BN_RESIDUAL else None
        f32 = dict(dtype=torch.float32, device=x.device)
        gw = torch.empty(c, **f32) if weight is not None else None
        gb = torch.empty(c, **f32) if ctx.has_bias else None
        coef = torch.empty(3 * c, **f32)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check("cs_bn_backward", _lib.lib.cs_bn_backward2(
            dy.data_ptr(), _ptr(dy2), x.data_ptr(), _ptr(res), n * h * w, c, save_mean.data_ptr(),
            save_invstd.data_ptr(), scale_shift.data_ptr(), _ptr(weight), _ptr(gw), _ptr(gb),
            coef.data_ptr(), dx.data_ptr(), _ptr(dres), ctx.ws.data_ptr(), ctx.flags, stream))
        if ctx.side_out is not None:      # identity-path gradient goes to the producer's BN
            ctx.side_out.grad = dres
            dres = None
        return dx, gw, gb, None, None, None, None, None, dres, None, None, None


class CrossoverBatchNorm2d(torch.nn.BatchNorm2d):
    """nn.BatchNorm2d whose training-mode bf16 path runs the fused NHWC kernels.

    ``forward_fused(x, relu, residual)`` also fuses the ReLU and the residual add that follow
    the BN in ResNet blocks into the same passes (forward and backward).
    """

    def _workspace(self, x: torch.Tensor) -> torch.Tensor:
        n, c, h, w = x.shape
        need = int(_lib.lib.cs_bn_workspace_bytes(n * h * w, c))
        ws = getattr(self, "_cs_ws", None)
        if ws is None or ws.numel() < need or ws.device != x.device:
            ws = torch.zeros(need, dtype=torch.uint8, device=x.device)
            self._cs_ws = ws
        return ws

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return self.forward_fused(x)

    def forward_fused(self, x: torch.Tensor, relu: bool = False,
                      residual: torch.Tensor | None = None,
                      residual_side: "_SideGrad | None" = None) -> torch.Tensor:
        fast = self.training and bn_supported(x) and (
            residual is None or (residual.shape == x.shape and residual.dtype == x.dtype))
        if not fast:
            y = super().forward(x)
            if residual is not None:
                y = y + residual
            return torch.relu(y) if relu else y
        momentum = self.momentum
        if self.track_running_stats and self.num_batches_tracked is not None:
            self.num_batches_tracked.add_(1)
            if momentum is None:   # cumulative moving average, as nn.BatchNorm2d
                raise NotImplementedError("momentum=None is not supported by the fused kernels")
        rm = self.running_mean if self.track_running_stats else None
        rv = self.running_var if self.track_running_stats else None
        flags = (CS_BN_RELU if relu else 0) | (CS_BN_RESIDUAL if residual is not None else 0)
        side_out = None
        if residual is not None and residual_side is not None:
            residual, side_out = residual.detach(), residual_side
        side_in = _SideGrad() if (relu and residual is not None) else None
        y = _BnFunction.apply(x, self.weight, self.bias, rm, rv, float(momentum or 0.0),
                              float(self.eps), self._workspace(x), residual, flags, side_in, side_out)
        if side_in is not None:
            y._cs_side = side_in
        return y


def _bn_relu_forward(self, x):
    return self.forward_fused(x, relu=True)


def _bottleneck_forward(self, x):
    # torchvision Bottleneck.forward with bn+relu and bn3+residual+relu fused; when x came out
    # of the previous block's fused bn3, the identity gradient is handed to that BN directly
    # (_SideGrad) instead of being summed with conv1's input gradient by an autograd add
    identity = x if self.downsample is None else self.downsample(x)
    side = getattr(x, "_cs_side", None) if (self.downsample is None and _SIDE_GRADS) else None
    out = self.bn1.forward_fused(self.conv1(x), relu=True)
    out = self.bn2.forward_fused(self.conv2(out), relu=True)
    return self.bn3.forward_fused(self.conv3(out), relu=True, residual=identity, residual_side=side)


# Measured on B200 (bench.py --side-grads A/B): the two-input backward kernels (one more input
# stream in both the partial and the apply kernel, +16 registers) cost more than the add kernel
# they remove (-1.9 % on the N = 1 bench), so autograd keeps summing by default.
_SIDE_GRADS = False


class _MaxPoolFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, s, p):
        n, c, h, w = x.shape
        oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        x = x.contiguous(memory_format=torch.channels_last)
        y = torch.empty((n, c, oh, ow), dtype=x.dtype, device=x.device,
                        memory_format=torch.channels_last)
        arg = torch.empty(n * oh * ow * c, dtype=torch.uint8, device=x.device)
        shape = (ctypes.c_int * 12)(n, h, w, c, oh, ow, k, k, s, s, p, p)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check("cs_maxpool2d_forward", _lib.lib.cs_maxpool2d_forward(
            x.data_ptr(), y.data_ptr(), arg.data_ptr(), shape, stream))
        ctx.save_for_backward(arg)
        ctx.meta = (n, c, h, w, oh, ow, k, s, p)
        return y

    @staticmethod
    def backward(ctx, dy):
        (arg,) = ctx.saved_tensors
        n, c, h, w, oh, ow, k, s, p = ctx.meta
        dy = dy.contiguous(memory_format=torch.channels_last)
        dx = torch.empty((n, c, h, w), dtype=dy.dtype, device=dy.device,
                         memory_format=torch.channels_last)
        shape = (ctypes.c_int * 12)(n, h, w, c, oh, ow, k, k, s, s, p, p)
        stream = torch.cuda.current_stream(dy.device).cuda_stream
        _lib.check("cs_maxpool2d_backward", _lib.lib.cs_maxpool2d_backward(
            dy.data_ptr(), arg.data_ptr(), dx.data_ptr(), shape, stream))
        return dx, None, None, None


class CrossoverMaxPool2d(torch.nn.MaxPool2d):
    """nn.MaxPool2d (square kernel, no dilation / ceil mode) with the NHWC kernels on bf16 CUDA input."""

    def forward(self, x):
        k, s, p = self.kernel_size, self.stride, self.padding
        simple = (isinstance(k, int) and isinstance(s, int) and isinstance(p, int)
                  and self.dilation == 1 and not self.ceil_mode and not self.return_indices)
        if not (simple and x.is_cuda and x.dtype == torch.bfloat16 and x.dim() == 4
                and x.shape[1] % 8 == 0 and k * k <= 256):
            return super().forward(x)
        return _MaxPoolFunction.apply(x, k, s, p)


def fuse_resnet(model: torch.nn.Module) -> int:
    """Fuse BN+ReLU (and the bottleneck residual add) in a torchvision ResNet; returns #blocks.

    Call after swap_batchnorm.  Parameters, buffers and state_dict keys are unchanged.
    """
    import types

    from torchvision.models.resnet import Bottleneck

    if isinstance(getattr(model, "bn1", None), CrossoverBatchNorm2d) and hasattr(model, "relu"):
        model.bn1.forward = types.MethodType(_bn_relu_forward, model.bn1)   # stem BN + ReLU
        model.relu = torch.nn.Identity()
    mp = getattr(model, "maxpool", None)
    if type(mp) is torch.nn.MaxPool2d:
        model.maxpool = CrossoverMaxPool2d(mp.kernel_size, mp.stride, mp.padding, mp.dilation,
                                           mp.return_indices, mp.ceil_mode)
    n = 0
    for m in model.modules():
        if isinstance(m, Bottleneck) and isinstance(m.bn3, CrossoverBatchNorm2d):
            m.forward = types.MethodType(_bottleneck_forward, m)
            n += 1
    return n


def swap_batchnorm(module: torch.nn.Module) -> int:
    """Replace nn.BatchNorm2d children in place (parameters and buffers are shared); returns count."""
    count = 0
    for name, child in list(module.named_children()):
        if type(child) is torch.nn.BatchNorm2d:
            new = CrossoverBatchNorm2d(child.num_features, child.eps, child.momentum, child.affine,
                                       child.track_running_stats, device=None)
            new.weight, new.bias = child.weight, child.bias
            new.running_mean, new.running_var = child.running_mean, child.running_var
            new.num_batches_tracked = child.num_batches_tracked
            new.train(child.training)
            setattr(module, name, new)
            count += 1
        else:
            count += swap_batchnorm(child)
    return count
