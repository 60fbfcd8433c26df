"""Bucket pack and fused average+update in numpy fp32 -- TEST INFRASTRUCTURE ONLY.

Restates, with the rounding sequence the device kernels promise:
  pack            workload.fuse_gradients (workload.py:94-101): tensors laid out back to
                  back in registration order at element offsets `offsets` (padding = 0)
  reduce_update   equivalence.average_gradients (equivalence.py:150-160) then
                  equivalence.sgd_step (equivalence.py:163-168):
                      acc = 0; acc = acc + g_s (s = 0..S-1); avg = acc / W; p - lr * avg
                  every operation rounded to fp32 (numpy fp32 arithmetic never fuses).
The torch-rounding (momentum) variant is checked against torch.optim.SGD on the
CPU directly in the tests, because numpy has no fused multiply-add.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


def layout(numels: Sequence[int], align: int):
    offs, cur = [], 0
    for n in numels:
        cur = -(-cur // align) * align
        offs.append(cur)
        cur += int(n)
    return offs, -(-cur // align) * align


def pack(tensors: Sequence[np.ndarray], align: int) -> np.ndarray:
    offs, total = layout([t.size for t in tensors], align)
    out = np.zeros(total, dtype=np.float32)
    for t, o in zip(tensors, offs):
        out[o:o + t.size] = t.reshape(-1)
    return out


def reduce_update(params: Sequence[np.ndarray], sources: Sequence[np.ndarray], offsets,
                  lr: float, divisor: int) -> list[np.ndarray]:
    """New fp32 parameters from fp32 bucket rows `sources` (reference rounding)."""
    f = np.float32
    out = []
    for p, o in zip(params, offsets):
        n = p.size
        acc = np.zeros(n, dtype=f)
        for s in sources:
            acc = acc + s[o:o + n]
        avg = acc / f(divisor)
        out.append((p.reshape(-1) - f(lr) * avg).reshape(p.shape))
    return out
