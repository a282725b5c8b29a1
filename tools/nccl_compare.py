"""NCCL comparison path for the multi-ring average (measurement only; not
parity-exact -- NCCL's reduction order differs from the reference ring).

Two variants, both ncclAllReduce(avg) over each ring's slice of the
parameter vector:

* ``sequential`` -- one communicator, the rings issued back to back on one
  stream (what a straightforward port would do);
* ``coalesced`` -- all rings' all-reduces in one NCCL group
  (ncclGroupStart/End via torch's coalescing manager), so they run
  concurrently on one communicator.

A communicator and stream per ring was measured too
(profiles/r01/sweep_n4_nccl_multicomm.jsonl: 645-668 GB/s at >= 256 MiB at 4
GPUs), but concurrent collectives on separate communicators can deadlock --
it did, at 256 MiB x 2 rings -- so it is not part of the default paths.

Timed with CUDA events, max over ranks.
"""

from __future__ import annotations

import os


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
        self.device = x.device

    def sequential(self):
        import torch.distributed as dist

        for v in self.views:
            dist.all_reduce(v, op=dist.ReduceOp.AVG)

    def coalesced(self):
        import torch.distributed as dist

        with dist._coalescing_manager(device=self.device):
            for v in self.views:
                dist.all_reduce(v, op=dist.ReduceOp.AVG)

    def time(self, fn, steps: int, flush=None) -> float:
        """Mean ms per call; with `flush` (bench.L2Flush), L2 is flushed
        before every call, outside its events."""
        import torch
        import torch.distributed as dist

        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s = torch.cuda.current_stream()
        if flush is None:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(steps):
                fn()
            b.record(s)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / steps
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for a, b in evs:
                flush(s)
                a.record(s)
                fn()
                b.record(s)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def report(self, steps: int, flush=None) -> dict:
        out = {"algo": os.environ.get("NCCL_ALGO", "default"),
               "nvls": os.environ.get("NCCL_NVLS_ENABLE", "default"), "l2_flushed": flush is not None}
        for name, fn in (("sequential", self.sequential), ("coalesced", self.coalesced)):
            ms = self.time(fn, steps, flush)
            out[name] = {"ms_per_step": round(ms, 4),
                         "bus_gbps_per_gpu": round(_busbw(sum(self.lens), self.world, ms * 1e-3), 3)}
        # headline comparison: the faster NCCL variant
        best = min(("sequential", "coalesced"), key=lambda k: out[k]["ms_per_step"])
        out["ms_per_step"] = out[best]["ms_per_step"]
        out["bus_gbps_per_gpu"] = out[best]["bus_gbps_per_gpu"]
        out["best"] = best
        return out
