"""The models' RGB stem convolution as two tensor-core GEMMs (apps' compute, not the sync path).

cuDNN runs the ResNet-50 stem (7x7 / 2, 3 -> 64, channels_last bf16, batch 256) at ~46 TFLOP/s:
with 3 input channels it pads the input and falls back to sm80-era fprop / wgrad kernels (about
2.6 ms of a ~24 ms iteration; tools/stem_bench.py).  Here the stem is

    forward   P = im2col(x)          (cs_im2col_nhwc: [N*OH*OW, KP] bf16, KP = K rounded up to 8)
              y = P . W^T            (cuBLAS bf16 GEMM; [N*OH*OW, O] is already the NHWC output)
    backward  dW = dy^T . P          (cuBLAS, K = N*OH*OW; P is kept from the forward)
              db = sum(dy)

The input gradient is not formed: the stem's input is the data.  The weight keeps its
[O, C, KH, KW] fp32 parameter; the GEMMs run in bf16 with fp32 accumulation like autocast's
convolution (the weight gradient is returned in fp32 straight from the accumulator), so the
result matches `F.conv2d` to bf16 rounding (tests/test_gpu_bn.py).
"""

from __future__ import annotations

import ctypes
import types

import torch

from . import _lib

__all__ = ["gemm_stem", "stem_supported"]


def stem_supported(conv: torch.nn.Conv2d, x: torch.Tensor) -> bool:
    return (x.is_cuda and x.dtype == torch.bfloat16 and x.dim() == 4 and conv.groups == 1
            and tuple(conv.dilation) == (1, 1) and conv.padding_mode == "zeros"
            and isinstance(conv.padding, tuple) and not x.requires_grad)


class _StemGemm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, stride, padding):
        n, c, h, w = x.shape
        o, _, kh, kw = weight.shape
        (sh, sw), (ph, pw) = stride, padding
        oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        k = kh * kw * c
        kp = (k + 7) // 8 * 8
        x = x.contiguous(memory_format=torch.channels_last)
        p = torch.empty((n * oh * ow, kp), dtype=torch.bfloat16, device=x.device)
        shape = (ctypes.c_int * 13)(n, h, w, c, oh, ow, kh, kw, sh, sw, ph, pw, kp)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check("cs_im2col_nhwc", _lib.lib.cs_im2col_nhwc(x.data_ptr(), p.data_ptr(), shape, stream))
        # the output is allocated channels_last and the GEMM writes its NHWC storage through a
        # 2-D view, so the Function returns a base tensor (consumers such as VGG's in-place
        # ReLU may modify it) without a layout copy
        y = torch.empty((n, o, oh, ow), dtype=torch.bfloat16, device=x.device,
                        memory_format=torch.channels_last)
        y2d = y.permute(0, 2, 3, 1).view(n * oh * ow, o)
        with torch.autocast("cuda", enabled=False):
            wm = torch.zeros((o, kp), dtype=torch.bfloat16, device=x.device)
            wm[:, :k] = weight.detach().permute(0, 2, 3, 1).reshape(o, k)
            if bias is not None:
                torch.addmm(bias.detach().to(torch.bfloat16), p, wm.t(), out=y2d)
            else:
                torch.mm(p, wm.t(), out=y2d)
        ctx.save_for_backward(p)
        fmt = (torch.channels_last if weight.is_contiguous(memory_format=torch.channels_last)
               and not weight.is_contiguous() else torch.contiguous_format)
        ctx.meta = (o, c, kh, kw, k, weight.dtype, bias is not None, fmt)
        return y

    @staticmethod
    def backward(ctx, dy):
        (p,) = ctx.saved_tensors
        o, c, kh, kw, k, wdt, has_bias, fmt = ctx.meta
        dy = dy.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        dym = dy.permute(0, 2, 3, 1).reshape(-1, o)
        with torch.autocast("cuda", enabled=False):
            # fp32 output straight from the bf16 GEMM's fp32 accumulator (no bf16 rounding of dW)
            dwm = torch.mm(dym.t(), p, out_dtype=torch.float32)
            # dW in the weight's own layout (a [o, kp] slice would carry the padded row stride),
            # so the fused update reads it in place without a re-layout copy
            dw = dwm[:, :k].reshape(o, kh, kw, c).permute(0, 3, 1, 2).to(wdt).contiguous(
                memory_format=fmt)
            db = dym.sum(0, dtype=torch.float32).to(wdt) if has_bias else None
        return None, dw, db, None, None


def _gemm_stem_forward(self, x):
    if not stem_supported(self, x):
        return self._conv_forward(x, self.weight, self.bias)
    return _StemGemm.apply(x, self.weight, self.bias, tuple(self.stride), tuple(self.padding))


def gemm_stem(model: torch.nn.Module) -> int:
    """Route every Conv2d with 3 input channels (the RGB stem) through the GEMM path; returns
    the number patched.  Parameters, buffers and state_dict keys are unchanged."""
    n = 0
    for m in model.modules():
        if isinstance(m, torch.nn.Conv2d) and m.in_channels == 3 and m.groups == 1:
            m.forward = types.MethodType(_gemm_stem_forward, m)
            n += 1
    return n
