"""NCCL comparison path for the multi-ring average (measurement only; not
parity-exact -- NCCL's reduction order differs from the reference ring).

Two variants, both ncclAllReduce(avg) over each ring's slice of the
parameter vector:

* ``sequential`` -- one communicator, the rings issued back to back on one
  stream (what a straightforward port would do);
* ``concurrent`` -- one communicator per ring, every ring on
  its own stream, all in flight together.

Timed with CUDA events, max over ranks.
"""

from __future__ import annotations

import os


_GROUPS: list = []  # one NCCL communicator per ring index, created once per process


def _ring_groups(n: int) -> list:
    import torch.distributed as dist

    while len(_GROUPS) < n:
        _GROUPS.append(dist.new_group(backend="nccl"))
    return _GROUPS[:n]


def _busbw(total_params: int, c: int, seconds: float) -> float:
    return total_params * 4 / seconds * 2 * (c - 1) / c / 1e9


class NcclRings:
    def __init__(self, x, lens):
        import torch
        import torch.distributed as dist

        self.world = dist.get_world_size()
        self.lens = list(lens)
        self.y = x.clone()
        starts, s = [], 0
        for n in self.lens:
            starts.append(s)
            s += n
        self.views = [self.y[a:a + n] for a, n in zip(starts, self.lens)]
        self.groups = _ring_groups(len(self.lens))
        self.streams = [torch.cuda.Stream() for _ in self.lens]

    def sequential(self):
        import torch.distributed as dist

        for v in self.views:
            dist.all_reduce(v, op=dist.ReduceOp.AVG)

    def concurrent(self):
        import torch
        import torch.distributed as dist

        main = torch.cuda.current_stream()
        for v, g, st in zip(self.views, self.groups, self.streams):
            st.wait_stream(main)
            with torch.cuda.stream(st):
                dist.all_reduce(v, op=dist.ReduceOp.AVG, group=g)
        for st in self.streams:
            main.wait_stream(st)

    def time(self, fn, steps: int) -> float:
        import torch
        import torch.distributed as dist

        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s = torch.cuda.current_stream()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(steps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def report(self, steps: int) -> dict:
        out = {"algo": os.environ.get("NCCL_ALGO", "default"),
               "nvls": os.environ.get("NCCL_NVLS_ENABLE", "default")}
        for name, fn in (("sequential", self.sequential), ("concurrent", self.concurrent)):
            ms = self.time(fn, steps)
            out[name] = {"ms_per_step": round(ms, 4),
                         "bus_gbps_per_gpu": round(_busbw(sum(self.lens), self.world, ms * 1e-3), 3)}
        # headline comparison: the faster NCCL variant
        best = min(("sequential", "concurrent"), key=lambda k: out[k]["ms_per_step"])
        out["ms_per_step"] = out[best]["ms_per_step"]
        out["bus_gbps_per_gpu"] = out[best]["bus_gbps_per_gpu"]
        out["best"] = best
        return out
