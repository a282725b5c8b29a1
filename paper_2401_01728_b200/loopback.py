"""The multi-rank transports with every rank on ONE device.

``LoopbackGroup`` builds C rank plans (``DevicePlan`` with ``n_ranks = C``,
``rank = position``) on a single GPU: the same pull / push / LL kernels,
barrier flags, staging areas and mean-delivered flags that
``dist.DistRingGroup`` drives across processes and GPUs, but with the peers'
buffers as plain device pointers instead of CUDA IPC mappings.  Each rank
launches on its own stream with an SM budget of 1/C of the device, so all C
kernels are resident at once (the transports spin on each other's flags).

Launch order matters on one device: rank kernels wait on each other, so no
launch that depends on an unfinished rank kernel may sit in a hardware queue
ahead of another rank's kernel (streams share the device's hardware queues,
CUDA_DEVICE_MAX_CONNECTIONS of them).  ``run`` therefore issues lane by lane
across all ranks, one stream per rank, and the separate blend launches of the
pull / LL transports only after every cycle kernel.

What it is for: the transports' arithmetic, work order and flag protocol run
-- and are checked bit for bit against the oracle -- on a one-GPU box, and
the same launch sequence is what every rank of an N-GPU job issues
(multiring.py:302-333 semantics; the reference has no transport code, its
rings exchange numpy payloads over simnet, multiring.py:185-225).  The
NVLink timing is of course not reproduced; bandwidth numbers come from the
multi-GPU bench.
"""

from __future__ import annotations

from typing import Mapping, Sequence

from . import _native as N
from .errors import ConfigError, LayoutError
from .blend import blend_
from .plan import DevicePlan, _dtype_code

TRANSPORTS = ("pull", "push", "ll")


class LoopbackGroup:
    """C ranks of one averaging group, all on ``device`` -- or spread over
    ``devices`` (rank m on devices[m]; several ranks may share a GPU), which
    drives an 8-rank group over the NVLink of a 4-GPU box from one process.

    Position m (the m-th smallest cluster id) is rank m.  ``bind_tensors``
    takes the C member buffers (rank m averages buffer m in place, or
    src[m] -> dst[m]); ``bind_live`` fuses the delayed-update blend as
    ``DistRingGroup.bind_live`` does.
    """

    def __init__(self, starts: Sequence[int], lens: Sequence[int], total: int, n_ranks: int, dtype,
                 protocol: str = "push", device: int = 0, acc: str = "f64", lanes: int = 1,
                 options: Mapping[str, int] | None = None, timeout_s: float | None = None,
                 blocks_per_rank: int | None = None, devices: Sequence[int] | None = None):
        if protocol not in TRANSPORTS:
            raise ConfigError(f"unknown protocol {protocol!r} (one of {TRANSPORTS})")
        if n_ranks < 2 or n_ranks > N.RV_MAX_RANKS:
            raise ConfigError(f"a loopback group needs 2..{N.RV_MAX_RANKS} ranks, got {n_ranks}")
        self.starts = [int(s) for s in starts]
        self.lens = [int(n) for n in lens]
        self.total = int(total)
        self.C = int(n_ranks)
        # rank m lives on devices[m] (default: all on `device`); ranks on
        # different devices reach each other's buffers, flags and staging
        # through peer access over NVLink, like DistRingGroup's IPC mappings
        self.devices = [int(device)] * self.C if devices is None else [int(d) for d in devices]
        if len(self.devices) != self.C:
            raise ConfigError(f"{len(self.devices)} devices for {self.C} ranks")
        self.device = self.devices[0]
        self.protocol = protocol
        self.lanes = int(lanes)
        lib = N.load()
        for a in set(self.devices):
            for b in set(self.devices):
                if a != b:
                    N.check(lib.rv_enable_peer_access(a, b), "rv_enable_peer_access")
        self.plans = []
        try:
            for m in range(self.C):
                dev = self.devices[m]
                # every rank's kernels must be resident together: the cycle
                # kernels run <= 2 blocks per SM (__launch_bounds__(256, 2)),
                # so 2*SMs / (ranks on the device) blocks per rank leave room
                budget = blocks_per_rank or max(1, 2 * lib.rv_device_sm_count(dev) // self.devices.count(dev))
                p = DevicePlan(dev, self.C, self.starts, self.lens, self.total, _dtype_code(dtype), acc)
                self.plans.append(p)
                p.set_options(options)
                if self.lanes != 1:
                    p.set_lanes(self.lanes)
                if timeout_s is not None:
                    p.set_timeout(timeout_s)
                p.set_max_blocks(budget)
                p.set_protocol(protocol)
            flags = [p.flag_area()[0] for p in self.plans]
            push = [p.push_area()[0] for p in self.plans] if protocol in ("push", "ll") else None
            for m, p in enumerate(self.plans):
                p.set_local([m])
                p.set_peers(m, self.C, flags)
                if push is not None:
                    p.set_push_peers(push)
        except BaseException:
            for p in self.plans:  # no half-built group keeps device memory
                p.close()
            self.plans = []
            raise
        import torch

        # one stream per rank (torch's pool holds 32 per device: more would alias)
        self.streams = [torch.cuda.Stream(device=d) for d in self.devices]
        self._bound = None
        self._lives = None

    def bind_tensors(self, srcs: Sequence, dsts: Sequence | None = None) -> None:
        dsts = srcs if dsts is None else dsts
        if len(srcs) != self.C or len(dsts) != self.C:
            raise LayoutError(f"expected {self.C} member buffers")
        for m, (s, d) in enumerate(zip(srcs, dsts)):
            for t in (s, d):
                if not t.is_cuda or t.device.index != self.devices[m] or not t.is_contiguous() or \
                        t.numel() != self.total:
                    raise LayoutError(f"member buffer {m} must be a contiguous cuda:{self.devices[m]} tensor "
                                      f"of {self.total} elements")
        for p in self.plans:
            for m, (s, d) in enumerate(zip(srcs, dsts)):
                p.bind(m, s.data_ptr(), d.data_ptr())
        self._bound = (list(srcs), list(dsts))  # plans hold raw pointers: keep the tensors alive
        self._agree()

    def bind_live(self, lives: Sequence | None) -> None:
        """Delayed-update blend: live <- mean + (live - src) every cycle.  The
        push transport fuses it into its kernel (rv_plan_bind_live); for pull
        and LL the group launches rv_blend per rank after all cycle kernels
        (the C ABI would launch it right behind each lane's kernel)."""
        if self.protocol == "push":
            for m, p in enumerate(self.plans):
                p.bind_live(m, None if lives is None else lives[m].data_ptr())
        self._lives = None if lives is None else list(lives)
        self._agree()

    def _agree(self) -> None:
        # the ranks must derive one layout (DistRingGroup checks the same
        # across processes); on one device they do by construction
        layouts = set()
        for p in self.plans:
            p.prepare()
            layouts.add(p.layout())
        if len(layouts) != 1:
            raise ConfigError(f"loopback ranks derived different layouts: {sorted(layouts)}")

    def run(self, after=None) -> None:
        """One cycle: every rank's launches on its own stream, lane by lane
        across the ranks, ordered after ``after`` (default: the current
        stream), which then waits for all."""
        import torch

        cur = after or torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(cur)
        for lane in range(self.lanes):
            for p, s in zip(self.plans, self.streams):
                p.run_lanes(lane, 1, [s])
        if self._lives is not None and self.protocol != "push":
            srcs, dsts = self._bound
            for m, s in enumerate(self.streams):
                blend_(self._lives[m], srcs[m], dsts[m], s)
        for s in self.streams:
            cur.wait_stream(s)

    def failed(self) -> bool:
        return any(p.failed() for p in self.plans)

    def check(self) -> None:
        for p in self.plans:
            p.check_status()

    def close(self) -> None:
        import torch

        for d in set(self.devices):
            torch.cuda.synchronize(d)
        for p in self.plans:
            p.close()
        self.plans = []
