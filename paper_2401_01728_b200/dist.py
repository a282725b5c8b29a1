"""One process per GPU: the multi-ring average across ranks of a torch.distributed group.

Each rank hosts one cluster (its live parameter vector on its own GPU).  At
construction the ranks exchange CUDA IPC handles of their parameter buffers
and barrier-flag areas over torch.distributed (plumbing only; gloo or nccl),
so every rank can address every peer's buffer over NVLink.  A cycle is then
one kernel per rank with no host round trip and no NCCL call: rank k folds
chunk k of every ring from all C buffers in ring order, divides by C, and
stores the mean into all C buffers (multiring.py:302-333 arithmetic).

Ring member order is ascending cluster id (multiring.py:95): ranks are sorted
by the ``cluster_id`` they pass (default: their rank).
"""

from __future__ import annotations

import ctypes
from typing import Sequence

from . import _native as N
from .errors import ConfigError, LayoutError
from .plan import DevicePlan, _dtype_code
from .schedule import ring_arrays


def _export(ptr: int) -> tuple[bytes, int]:
    lib = N.load()
    size = lib.rv_ipc_handle_size()
    buf = ctypes.create_string_buffer(size)
    off = ctypes.c_uint64()
    N.check(lib.rv_ipc_export(ctypes.c_void_p(int(ptr)), buf, ctypes.byref(off)), "rv_ipc_export")
    return buf.raw, int(off.value)


def _import(device: int, handle: bytes, offset: int) -> int:
    lib = N.load()
    out = ctypes.c_void_p()
    N.check(lib.rv_ipc_import(int(device), handle, ctypes.c_uint64(int(offset)), ctypes.byref(out)),
            "rv_ipc_import")
    return int(out.value)


def _close(device: int, ptr: int) -> None:
    N.load().rv_ipc_close(int(device), ctypes.c_void_p(int(ptr)))


PUSH_MIN_BYTES = 32 << 20       # 3 or more ranks
PUSH_MIN_BYTES_C2 = 192 << 20   # 2 ranks
LL_MAX_BYTES = 4 << 20


def choose_protocol(protocol: str, bytes_per_cluster: int, fp32: bool = True, n_ranks: int | None = None) -> str:
    """'auto': the LL transport for fp32 sets up to 4 MiB per cluster
    (latency-bound: no fences or barriers), store-only push from 32 MiB (its
    per-unit flags pay off and NVLink stores outrun loads) -- from 192 MiB
    with 2 ranks, where pull stays ahead longer -- and pull in between.
    Round-2 sweep (profiles/r02/sweep_r02_n{2,4}.jsonl): at 4 GPUs push
    leads from 32 MiB; at 2 GPUs pull leads up to 128 MiB (ResNet-50, 102 MB:
    pull 552.7 vs push 546 GB/s; BERT, 438 MB: push 671 vs pull 647,
    profiles/r02/proto_crossover_n2.txt).  Depends only on the schedule,
    dtype and rank count, so every rank picks the same."""
    if protocol == "auto":
        if fp32 and bytes_per_cluster <= LL_MAX_BYTES:
            return "ll"
        push_min = PUSH_MIN_BYTES_C2 if n_ranks == 2 else PUSH_MIN_BYTES
        return "push" if bytes_per_cluster >= push_min else "pull"
    if protocol not in ("pull", "push", "ll"):
        raise ConfigError(f"unknown protocol {protocol!r} (auto, pull, push or ll)")
    return protocol


def rendezvous(mine: dict, group=None) -> tuple[list, list[int], int]:
    """All-gather each rank's descriptor (cluster id + IPC handles) and order
    ranks by ascending cluster id -- the ring member order (multiring.py:95).
    Returns (descriptors by rank, rank of each position, this rank's position)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    everyone: list = [None] * world
    dist.all_gather_object(everyone, mine, group=group)
    cids = [e["cid"] for e in everyone]
    if len(set(cids)) != len(cids):
        raise ConfigError(f"duplicate cluster ids across ranks: {cids}")
    order = sorted(range(world), key=lambda r: cids[r])
    return everyone, order, order.index(dist.get_rank(group))


def agree_layouts(mine, group=None) -> None:
    """Collective: every rank's (vectors per unit, staging stride, unit slots,
    work items) must be identical -- push and LL writers compute the owners'
    staging addresses and unit flags locally, so a rank with another SM count
    or option set would corrupt the means or hang.  Raises ConfigError on
    every rank when they differ."""
    import torch.distributed as dist

    everyone: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(everyone, tuple(mine), group=group)
    if any(e != tuple(mine) for e in everyone):
        raise ConfigError(f"ranks derived different cycle layouts (unit vectors, stride, unit slots, "
                          f"work items): {everyone}; use the same options on every rank "
                          f"(e.g. layout_sms for GPUs with different SM counts)")


def agree_bind_live(err: str | None, bound: bool, group=None) -> None:
    """Collective vote of bind_live: every rank learns every rank's verdict,
    so all raise together (LayoutError for a bad buffer anywhere, ConfigError
    when some ranks bind and others do not) instead of leaving the others
    blocked in the next collective or, worse, spinning on mean-delivered
    flags nobody raises."""
    import torch.distributed as dist

    votes: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(votes, (err, bool(bound)), group=group)
    errs = [(r, e) for r, (e, _) in enumerate(votes) if e]
    if errs:
        raise LayoutError("; ".join(f"rank {r}: {e}" for r, e in errs))
    if len({b for _, b in votes}) != 1:
        raise ConfigError(f"bind_live is collective: ranks disagree on the fused blend ({[b for _, b in votes]})")


class DistRingGroup:
    """Collective multi-ring averaging of one CUDA buffer per rank.

    ``src`` is read and ``dst`` (default: ``src``, i.e. in place) written;
    both must stay allocated while the group lives.  With ``live`` (and a
    separate ``dst``), every cycle also applies the delayed-update blend
    live <- mean + (live - src) (``bind_live``).  All ranks must call
    ``average`` the same number of times in the same order, as with any
    collective.
    """

    def __init__(self, schedule=None, src=None, dst=None, *, starts: Sequence[int] | None = None,
                 lens: Sequence[int] | None = None, cluster_id: int | None = None, acc: str = "f64",
                 lanes: int = 1, group=None, timeout_s: float | None = None, protocol: str = "auto",
                 max_blocks: int = 0, live=None, options: dict | None = None):
        import torch.distributed as dist

        if src is None:
            raise ConfigError("DistRingGroup needs the rank's parameter buffer")
        if schedule is not None:
            starts, lens = ring_arrays(schedule)
            total = int(schedule.total_params)
        else:
            if starts is None or lens is None:
                raise ConfigError("pass a schedule or ring starts/lens")
            starts, lens = [int(s) for s in starts], [int(n) for n in lens]
            total = sum(lens)
        dst = src if dst is None else dst
        for t in (src, dst):
            if not t.is_cuda or not t.is_contiguous():
                raise LayoutError("DistRingGroup buffers must be contiguous CUDA tensors")
            if t.numel() != total:
                raise LayoutError(f"buffer has {t.numel()} elements, schedule expects {total}")
        if dst.dtype != src.dtype:
            raise LayoutError("src and dst dtypes differ")
        if total == 0:
            raise LayoutError("DistRingGroup needs a non-empty parameter vector")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world < 2:
            raise ConfigError("all-reduce needs at least 2 clusters")
        if self.world > N.RV_MAX_RANKS:
            raise ConfigError(f"at most {N.RV_MAX_RANKS} ranks")
        self.device = src.device.index
        self.src, self.dst = src, dst
        self.total = total
        self.starts, self.lens = starts, lens
        cid = self.rank if cluster_id is None else int(cluster_id)

        self.plan = DevicePlan(self.device, self.world, starts, lens, total, _dtype_code(src.dtype), acc)
        self.plan.set_options(options)
        if lanes != 1:
            self.plan.set_lanes(lanes)
        if timeout_s is not None:
            self.plan.set_timeout(timeout_s)
        if max_blocks:
            self.plan.set_max_blocks(max_blocks)
        protocol = choose_protocol(protocol, total * src.element_size(), src.element_size() == 4, self.world)
        self.protocol = protocol
        self.plan.set_protocol(protocol)
        flag_ptr, _ = self.plan.flag_area()
        mine = {
            "cid": cid,
            "src": _export(src.data_ptr()),
            "dst": _export(dst.data_ptr()),
            "flags": _export(flag_ptr),
        }
        push_ptr = 0
        if protocol in ("push", "ll"):
            push_ptr, _ = self.plan.push_area()
            mine["push"] = _export(push_ptr)
        everyone, order, self.position = rendezvous(mine, group)
        self._imported: list[int] = []
        areas = [0] * self.world
        push_areas = [0] * self.world
        for pos, r in enumerate(order):
            e = everyone[r]
            if r == self.rank:
                self.plan.bind(pos, src.data_ptr(), dst.data_ptr())
                areas[pos] = flag_ptr
                push_areas[pos] = push_ptr
                continue
            s = _import(self.device, *e["src"])
            d = s if e["dst"] == e["src"] else _import(self.device, *e["dst"])
            f = _import(self.device, *e["flags"])
            self._imported += [s, f] + ([d] if d != s else [])
            if protocol in ("push", "ll"):
                push_areas[pos] = _import(self.device, *e["push"])
                self._imported.append(push_areas[pos])
            self.plan.bind(pos, s, d)
            areas[pos] = f
        self.plan.set_local([self.position])
        self.plan.set_peers(self.position, self.world, areas)
        if protocol in ("push", "ll"):
            self.plan.set_push_peers(push_areas)
        self.live = None
        if live is not None:
            self.bind_live(live)
        else:
            self._agree()
        dist.barrier(group=group)

    def _agree(self) -> None:
        """Build the tables and check every rank derived the same layout:
        push and LL writers compute the owners' staging addresses and unit
        flags locally, so a rank with another SM count or option set would
        corrupt the means or hang.  Raises ConfigError on a mismatch."""
        self.plan.prepare()
        agree_layouts(self.plan.layout(), self.group)

    def bind_live(self, live) -> None:
        """Fuse the delayed-update blend into every cycle: ``live`` (this
        rank's live parameters) ends each cycle as mean + (live - src), the
        snapshot ``src`` having been averaged into ``dst``.  ``None`` unbinds.
        Collective: every rank must bind (or unbind) together -- the push
        kernel then blends unit by unit as the means land and skips the depart
        barrier, so a rank without the blend would wait for flags nobody
        raises.  Raises ConfigError when the ranks disagree."""
        err = None
        if live is not None:
            if not live.is_cuda or not live.is_contiguous() or live.numel() != self.total:
                err = "live must be a contiguous CUDA tensor shaped like the parameter vector"
            elif live.dtype != self.src.dtype or live.device.index != self.device:
                err = "live must match the parameter buffer's dtype and device"
            elif self.dst.data_ptr() == self.src.data_ptr():
                err = "the fused blend needs a separate mean buffer (dst) besides the snapshot (src)"
        agree_bind_live(err, live is not None, self.group)
        self.plan.bind_live(self.position, None if live is None else live.data_ptr())
        self.live = live
        self._agree()

    def failed(self) -> bool:
        """Non-blocking: a cycle of this rank stalled (see ``check``)."""
        return self.plan.failed()

    def average(self, streams=None) -> None:
        """Launch one cycle on ``streams`` (default: the current stream)."""
        import torch

        if streams is None:
            self.plan.run((torch.cuda.current_stream(self.device).cuda_stream,))
            return
        self.plan.run(streams if isinstance(streams, (list, tuple)) else [streams])

    def average_host(self, host_src, host_dst, streams=None) -> None:
        """Cycle from/to pinned HOST tensors: H2D, average, D2H, pipelined
        per lane (rv_allreduce_mean_host)."""
        import torch

        st = streams if streams is not None else [torch.cuda.current_stream(self.device)]
        st = st if isinstance(st, (list, tuple)) else [st]
        with torch.cuda.nvtx.range("ravnest_b200.cycle_host"):
            self.plan.run_host([host_src.data_ptr()], [host_dst.data_ptr()], st)

    def check(self) -> None:
        self.plan.check_status()

    def close(self, barrier: bool = True) -> None:
        """Release the plan and the peer mappings.  Collective by default:
        every rank finishes its cycles (device sync) and meets the others
        before anything is unmapped, so no kernel still touches a peer's
        buffer or this rank's staging when it goes away."""
        import torch
        import torch.distributed as dist

        if self.plan is None:
            return
        torch.cuda.synchronize(self.device)
        if barrier and dist.is_initialized():
            dist.barrier(group=self.group)
        for p in self._imported:
            _close(self.device, p)
        self._imported = []
        self.plan.close()
        self.plan = None
