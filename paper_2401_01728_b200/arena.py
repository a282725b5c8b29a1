"""Zero-copy flat parameter arena.

The reference keeps each peer's parameters in one flat float64 vector laid
out layer by layer (modelcore.ParameterVector, modelcore.py:75-108) and
copies them into a cluster vector for every averaging (assemble_full /
peer_vector, modelcore.py:403-418; pipeline.full_values/load_values,
pipeline.py:445-452).  Here a torch module's parameters become views into
ONE contiguous device buffer, in registration order: the averaging kernel
reads and writes that buffer in place, so no gather, scatter or copy runs
around a cycle, and optimizers keep working on the views.

Ring layout: submodels are cut at tensor boundaries by walking the tensors
in order and closing a submodel before a tensor that would push it past
total / R (the split behind SURVEY.md §8a's ResNet-50 / BERT-base /
GPT-2-medium ring lengths, reproduced exactly by ``tensor_boundary_rings``).
Every cluster uses the same split, so ``build_ring_schedule`` gives one ring
per submodel.
"""

from __future__ import annotations

from typing import Sequence

from .schedule import ParamRange, RingSchedule, build_ring_schedule


def tensor_boundary_rings(sizes: Sequence[int], n_rings: int) -> list[int]:
    """Ring lengths from per-tensor element counts (contiguous, in order)."""
    if n_rings < 1:
        raise ValueError("n_rings must be >= 1")
    target = sum(sizes) / n_rings
    out, cur = [], 0
    for n in sizes:
        if cur > 0 and cur + n > target and len(out) < n_rings - 1:
            out.append(cur)
            cur = 0
        cur += int(n)
    out.append(cur)
    return out


def layout_from_lengths(lengths: Sequence[int]) -> list[ParamRange]:
    out, start = [], 0
    for n in lengths:
        out.append(ParamRange(start, int(n)))
        start += int(n)
    return out


def ring_schedule(cluster_ids: Sequence[int], lengths: Sequence[int]) -> RingSchedule:
    """Every cluster split the same way -> one ring per submodel."""
    lay = layout_from_lengths(lengths)
    return build_ring_schedule({int(c): list(lay) for c in cluster_ids})


class ParamArena:
    """All parameters of ``module`` as views into one flat buffer.

    ``flat`` is the buffer the averaging path binds (DistRingGroup /
    AsyncAverager / ring_mean_).  ``grads=True`` also gives every parameter a
    ``.grad`` view into a second flat buffer (one fused optimizer step)."""

    def __init__(self, module, device=None, dtype=None, grads: bool = False):
        import torch

        params = [p for p in module.parameters()]
        if not params:
            raise ValueError("module has no parameters")
        device = torch.device(device) if device is not None else params[0].device
        dtype = dtype or params[0].dtype
        self.sizes = [p.numel() for p in params]
        self.names = [n for n, _ in module.named_parameters()]
        total = sum(self.sizes)
        self.flat = torch.empty(total, device=device, dtype=dtype)
        self.grad = torch.zeros(total, device=device, dtype=dtype) if grads else None
        off = 0
        with torch.no_grad():
            for p, n in zip(params, self.sizes):
                view = self.flat[off:off + n].view_as(p)
                view.copy_(p.detach().to(device=device, dtype=dtype))
                p.data = view
                if grads:
                    p.grad = self.grad[off:off + n].view_as(p)
                off += n
        self.offsets = [sum(self.sizes[:i]) for i in range(len(self.sizes))]

    @property
    def numel(self) -> int:
        return self.flat.numel()

    def ring_lengths(self, n_rings: int) -> list[int]:
        return tensor_boundary_rings(self.sizes, n_rings)

    def schedule(self, cluster_ids: Sequence[int], n_rings: int) -> RingSchedule:
        return ring_schedule(cluster_ids, self.ring_lengths(n_rings))
