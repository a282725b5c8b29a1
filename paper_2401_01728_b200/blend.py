"""Delayed-update blend.

In the reference, batches in flight during an averaging cycle computed
their gradients on parameters stashed at forward time (pipeline.py:353) and
apply them to the LIVE, post-average parameters (pipeline.py:384-411 ->
modelcore.apply_update, modelcore.py:357-371).  On the GPU the cycle averages
a snapshot ``snap`` while training keeps updating ``live``; at the next step
boundary ``blend_`` folds the updates made since the snapshot onto the mean:

    live <- mean + (live - snap)      (exactly ``mean`` where live == snap bitwise)

One HBM-bound kernel per cluster (rv_blend), on the training stream.
"""

from __future__ import annotations

import ctypes

from . import _native as N
from .errors import LayoutError
from .plan import _dtype_code, _stream_handle


def blend_(live, snap, mean, stream=None):
    """In place on ``live`` (CUDA tensors of one dtype and size)."""
    import torch

    for t in (live, snap, mean):
        if not t.is_cuda or not t.is_contiguous():
            raise LayoutError("blend_ needs contiguous CUDA tensors")
        if t.numel() != live.numel() or t.dtype != live.dtype:
            raise LayoutError("blend_ tensors differ in size or dtype")
    st = stream if stream is not None else torch.cuda.current_stream(live.device)
    lib = N.load()
    N.check(lib.rv_blend(live.device.index, _dtype_code(live.dtype), ctypes.c_void_p(live.data_ptr()),
                         ctypes.c_void_p(snap.data_ptr()), ctypes.c_void_p(mean.data_ptr()),
                         live.numel(), ctypes.c_void_p(_stream_handle(st))), "rv_blend")
    return live
