"""Drop-in replacements for the reference's averaging entry points.

Signatures follow /root/reference/pkg/src/ravnest/multiring.py:

* ``apply_ring_mean(schedule, cluster_params)``      -- multiring.py:302-333
* ``run_allreduce(schedule, cluster_params, network=None, node_of=..., max_events=None)``
                                                     -- multiring.py:254-299
* ``AllReduceController(schedule, working, network, node_of)``
                                                     -- multiring.py:154-247

They accept what the reference accepts (``{cluster_id: np.ndarray}``) and
return what it returns (new float64 arrays; ``working`` mutated in place for
the controller), bit for bit: float64 inputs run the float64 kernel, whose
fold order is the reference's.  ``dict[int, torch.Tensor]`` of CUDA tensors
is the fast path: the cycle runs where the tensors live (one GPU ->
co-resident kernel, several GPUs -> NVLink peer kernel), in the tensors'
dtype, and ``ring_mean_`` averages them in place.

There is no CPU fallback: without a CUDA device these raise RavnestError.
"""

from __future__ import annotations

import collections
import os
import sys
from concurrent.futures import ThreadPoolExecutor
from typing import Callable

import numpy as np

from . import _native as N
from .errors import ConfigError, LayoutError, ProtocolError, RavnestError, StallError
from .plan import LocalRingGroup
from .schedule import RingStats, chunk_bounds, ring_arrays, schedule_stats

_GROUPS: "collections.OrderedDict[tuple, LocalRingGroup]" = collections.OrderedDict()
_MAX_GROUPS = 8


def default_node_name(cluster_id: int, peer: int) -> str:
    return f"c{cluster_id}.p{peer}"


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RavnestError("no CUDA device visible: the B200 averaging path has no CPU fallback")
    return torch


def group_for(schedule, devices, dtype, acc: str = "f64", lanes: int = 1) -> LocalRingGroup:
    """Cached LocalRingGroup for (schedule, placement, dtype, accumulation)."""
    starts, lens = ring_arrays(schedule)
    key = (tuple(starts), tuple(lens), int(schedule.total_params), tuple(devices), str(dtype), acc, lanes)
    g = _GROUPS.get(key)
    if g is None:
        g = LocalRingGroup(starts, lens, schedule.total_params, devices, dtype, acc=acc, lanes=lanes)
        _GROUPS[key] = g
        while len(_GROUPS) > _MAX_GROUPS:
            _, old = _GROUPS.popitem(last=False)
            old.close()
    else:
        _GROUPS.move_to_end(key)
    return g


def _check_shapes(schedule, cluster_params, cids) -> None:
    # multiring.py:270-275
    for cid in cids:
        shape = tuple(cluster_params[cid].shape)
        if shape != (schedule.total_params,):
            raise LayoutError(
                f"cluster {cid} vector has {shape}, schedule expects ({schedule.total_params},)"
            )


def ring_mean_(schedule, tensors: dict, acc: str = "f64", lanes: int = 1, streams=None,
               sync: bool = True) -> dict:
    """Average ``{cluster_id: cuda tensor}`` IN PLACE (the B200 fast path).

    Every tensor ends holding, for chunk k of every ring, the fold
    x_k + x_{k+1} + ... + x_{k+C-1} divided by C (apply_ring_mean's bits when
    ``acc="f64"``; float32 storage is rounded once from the float64 fold).
    """
    torch = _torch()
    cids = sorted(tensors)
    if len(cids) < 2:
        raise ConfigError("all-reduce needs at least 2 clusters")
    _check_shapes(schedule, tensors, cids)
    ts = [tensors[c] for c in cids]
    dtype = ts[0].dtype
    for t in ts:
        if not t.is_cuda:
            raise LayoutError("ring_mean_ needs CUDA tensors; use apply_ring_mean for host arrays")
        if t.dtype != dtype:
            raise LayoutError(f"mixed dtypes {t.dtype} and {dtype}")
    if schedule.total_params == 0:
        return tensors  # nothing to average (all rings empty)
    devices = [t.device.index for t in ts]
    g = group_for(schedule, devices, dtype, acc=acc, lanes=lanes)
    g.bind_tensors(ts)
    g.run(streams)
    if sync:
        for d in g.device_order:
            torch.cuda.synchronize(d)
        g.check()
    return tensors


# ---------------------------------------------------------------------------
# numpy in, numpy out: the reference's own calling convention


_COPY_POOL: ThreadPoolExecutor | None = None
_COPY_PIECE = 1 << 21  # elements per copy task (16 MB of float64)


def _copy_pool() -> ThreadPoolExecutor:
    global _COPY_POOL
    if _COPY_POOL is None:
        try:
            cpus = len(os.sched_getaffinity(0))
        except Exception:
            cpus = os.cpu_count() or 1
        _COPY_POOL = ThreadPoolExecutor(max_workers=max(1, min(16, cpus)), thread_name_prefix="ravnest-copy")
    return _COPY_POOL


def _copy_ranges(pairs, lo: int, hi: int) -> None:
    """dst[lo:hi] = src[lo:hi] for every (dst, src) pair, widening to the
    destination dtype like np.array(x, dtype=float64) (multiring.py:309).
    Large ranges are split across the copy pool (numpy releases the GIL
    inside the copy loop)."""
    n = hi - lo
    if n <= 0:
        return
    if n * len(pairs) <= 2 * _COPY_PIECE:
        for d, s in pairs:
            np.copyto(d[lo:hi], s[lo:hi], casting="unsafe")
        return
    pool = _copy_pool()
    futs = [pool.submit(np.copyto, d[a:min(hi, a + _COPY_PIECE)], s[a:min(hi, a + _COPY_PIECE)], casting="unsafe")
            for d, s in pairs for a in range(lo, hi, _COPY_PIECE)]
    for f in futs:
        f.result()


class _HostCycle:
    """One cycle for numpy inputs: the reference's float64 copy-in goes into
    pinned staging arrays, and lane by lane the staging is copied to the GPU,
    averaged by the float64 kernel (bitwise apply_ring_mean) and copied back
    into the same staging arrays -- while the host fills the next lane.  The
    staging arrays are what ``apply_ring_mean`` returns (new float64 arrays,
    inputs untouched, as multiring.py:309 promises)."""

    MIN_LANE_BYTES = 16 << 20  # per cluster; below it one lane (launch-bound sizes)
    MAX_LANES = 16

    def __init__(self, schedule, n_clusters: int):
        torch = _torch()
        self.torch = torch
        self.total = int(schedule.total_params)
        self.n = n_clusters
        dev = torch.cuda.current_device()
        lanes = max(1, min(self.MAX_LANES, self.total * 8 // self.MIN_LANE_BYTES))
        lanes = min(lanes, max(64, len(schedule.rings)))
        self.group = group_for(schedule, [dev] * n_clusters, torch.float64, lanes=lanes)
        g = self.group
        # device buffers and streams live with the cached group
        if getattr(g, "_host_bufs", None) is None:
            g._host_bufs = [torch.empty(self.total, dtype=torch.float64, device=f"cuda:{dev}")
                            for _ in range(n_clusters)]
            g._host_streams = [torch.cuda.Stream(device=dev) for _ in range(min(lanes, 4))]
        g.bind_tensors(g._host_bufs)
        self.plan = g.plans[dev]
        starts, lens = ring_arrays(schedule)
        self.ranges = N.lane_ranges(starts, lens, lanes)
        self.streams = g._host_streams
        self.dev = dev
        self.done_event = None

    def launch(self, inputs) -> list:
        """Start the cycle; returns the pinned float64 staging arrays that
        will hold the means once ``wait`` returns."""
        torch = self.torch
        cur = torch.cuda.current_stream(self.dev)
        for st in self.streams:
            st.wait_stream(cur)
        stage = [torch.empty(self.total, dtype=torch.float64, pin_memory=True).numpy() for _ in range(self.n)]
        ptrs = [a.ctypes.data for a in stage]
        pairs = list(zip(stage, inputs))
        for lane, (lo, hi) in enumerate(self.ranges):
            _copy_ranges(pairs, int(lo), int(hi))
            self.plan.run_host_lanes(lane, 1, ptrs, ptrs, self.streams)
        for st in self.streams:
            cur.wait_stream(st)
        self.done_event = torch.cuda.Event()
        self.done_event.record(cur)
        return stage

    def ready(self) -> bool:
        return self.done_event is None or self.done_event.query()

    def wait(self) -> None:
        if self.done_event is not None:
            self.done_event.synchronize()
        if self.plan.failed():
            self.group.check()


def _as_arrays(cluster_params, cids) -> list:
    return [a if isinstance(a, np.ndarray) else np.asarray(a) for a in (cluster_params[c] for c in cids)]


def apply_ring_mean(schedule, cluster_params: dict, acc: str = "f64") -> dict:
    """Synchronous cycle with the reference's contract: inputs untouched,
    new arrays returned (multiring.py:302-333).

    numpy inputs are widened to float64 exactly as the reference does
    (multiring.py:309) -- into pinned staging, lane by lane, overlapped with
    the transfers -- and averaged co-resident on the current GPU by the
    float64 kernel; the result is float64 and bitwise equal to the reference.
    CUDA tensors are cloned and averaged where they live.
    """
    cids = sorted(cluster_params)
    if not cids:
        return {}
    first = cluster_params[cids[0]]
    is_torch = type(first).__module__.startswith("torch")
    if is_torch and first.is_cuda:
        clones = {c: cluster_params[c].clone() for c in cids}
        if len(cids) < 2:
            return clones
        return ring_mean_(schedule, clones, acc=acc)
    arrays = _as_arrays(cluster_params, cids)
    if len(cids) < 2 or schedule.total_params == 0:
        return {c: np.array(a, dtype=np.float64) for c, a in zip(cids, arrays)}
    _check_shapes(schedule, dict(zip(cids, arrays)), cids)
    cyc = _HostCycle(schedule, len(cids))
    stage = cyc.launch(arrays)
    cyc.wait()
    return dict(zip(cids, stage))


def _ideal_network_progress(schedule, n_clusters: int, budget: int,
                            node_of: Callable[[int, int], str] = default_node_name):
    """Replay, without data, how far the reference's cycle gets on its ideal
    network within ``budget`` events: every link has bandwidth 1e18 B/s and
    zero latency (multiring.py:278-285), so a chunk of n float64 values is
    delivered n*8/1e18 s after its link frees up (simnet.py:165-187), ties by
    send order (simnet.py:70-113).  Returns AllReduceController._expected."""
    import heapq

    expected = {r.ring_id: [0] * n_clusters for r in schedule.rings}
    last = 2 * (n_clusters - 1)
    rings = {r.ring_id: r for r in schedule.rings}
    bounds = {r.ring_id: chunk_bounds(r.start, r.length, n_clusters) for r in schedule.rings}
    busy: dict = {}
    heap: list = []
    seq = 0

    def send(rid, pos, rnd, chunk, now):
        nonlocal seq
        ring = rings[rid]
        link = (node_of(*ring.members[pos]), node_of(*ring.members[(pos + 1) % n_clusters]))
        lo, hi = bounds[rid][chunk]
        start = max(now, busy.get(link, 0.0))
        done = start + (hi - lo) * 8 / 1e18
        busy[link] = done
        heapq.heappush(heap, (done + 0.0, seq, (rid, (pos + 1) % n_clusters, rnd, chunk)))
        seq += 1

    for r in schedule.rings:
        for pos in range(n_clusters):
            send(r.ring_id, pos, 0, pos % n_clusters, 0.0)
    now, done_events = 0.0, 0
    while heap and done_events < budget:
        t, _, (rid, to_pos, rnd, chunk) = heapq.heappop(heap)
        now = max(now, t)
        expected[rid][to_pos] = rnd + 1
        done_events += 1
        if rnd + 1 < last:
            send(rid, to_pos, rnd + 1, chunk, now)
    return expected


def _stall_text(schedule, expected, n_clusters: int) -> str:
    stuck = []
    members = {r.ring_id: r.members for r in schedule.rings}
    for rid in sorted(expected):
        for pos, exp in enumerate(expected[rid]):
            if exp < 2 * (n_clusters - 1):
                stuck.append(f"(ring={rid}, round={exp}, member={tuple(members[rid][pos])})")
    return "waiting on: " + ", ".join(stuck) if stuck else "no ring is stalled"


def run_allreduce(schedule, cluster_params: dict, network=None,
                  node_of: Callable[[int, int], str] = default_node_name,
                  max_events: int | None = None) -> tuple[dict, list[RingStats]]:
    """One full cycle; every cluster ends with the global mean
    (multiring.py:254-299).  Without a network the rings run over the
    reference's ideal links, whose timing never shapes the arithmetic
    (test_multiring.py:173-205): the GPU cycle runs directly, and an event
    budget smaller than the cycle's message count raises StallError naming
    the blocked (ring, round, member), as the reference does under FIFO
    delivery.  With a caller's network the controller below replays the
    ring's messages over it (same virtual time and trace as the reference)
    while the GPU computes the means."""
    cids = sorted(cluster_params)
    if len(cids) < 2:
        raise ConfigError("all-reduce needs at least 2 clusters")
    _check_shapes(schedule, cluster_params, cids)
    c = len(cids)
    if network is not None:
        working = {cid: np.array(cluster_params[cid], dtype=np.float64) for cid in cids}
        ctl = AllReduceController(schedule, working, network, node_of)
        ctl.kickoff(network.now)
        budget = max_events
        if budget is None:
            budget = 10 * sum(2 * (len(r.members) - 1) * len(r.members) for r in schedule.rings) + 1000
        network.run_until(predicate=ctl.done, max_events=budget, diagnostics=ctl.stall_report)
        if not ctl.done():
            raise StallError("all-reduce incomplete: " + ctl.stall_report())
        return working, ctl.stats()
    needed = sum(2 * (c - 1) * c for _ in schedule.rings)
    if max_events is not None and max_events < needed:
        expected = _ideal_network_progress(schedule, c, max_events, node_of)
        raise StallError(
            f"event budget of {max_events} exhausted\n"
            + "all-reduce incomplete: " + _stall_text(schedule, expected, c)
        )
    out = apply_ring_mean(schedule, cluster_params)
    return out, schedule_stats(schedule, c)


_NO_DATA = np.zeros(1)


class AllReduceController:
    """Drain-barrier seam (orchestrator.py:339-363, multiring.py:154-247).

    ``kickoff`` starts the GPU cycle asynchronously (float64 copy-in, H2D,
    kernel, D2H on side streams) and then plays the reference's ring
    protocol over the caller's network message for message: the same
    sender, receiver, round and chunk, and a payload of the chunk's size
    that carries no data (a zero-stride float64 view, so the network's
    serialisation delay, trace bytes and event order are the reference's).
    ``handle`` enforces the reference's round order (ProtocolError) and
    forwards the next round.  ``done`` is true once every ring member has
    seen all 2(C-1) rounds AND the GPU cycle has landed; at that moment
    ``working`` (the caller's dict, mutated in place as the reference does)
    receives the means.  Virtual time, stats and stall reports therefore
    match the reference exactly, and the arithmetic is bitwise its own.
    """

    def __init__(self, schedule, working: dict, network, node_of: Callable[[int, int], str]):
        self.schedule = schedule
        self.working = working
        self.network = network
        self.node_of = node_of
        self._cids = sorted(working)
        self._c = len(self._cids)
        self._bounds = {r.ring_id: chunk_bounds(r.start, r.length, len(r.members)) for r in schedule.rings}
        self._expected = {r.ring_id: [0] * len(r.members) for r in schedule.rings}
        self._messages = {r.ring_id: 0 for r in schedule.rings}
        self._rings = {r.ring_id: r for r in schedule.rings}
        self._cycle = None
        self._stage = None
        self._landed = False
        self._message_cls = None

    def kickoff(self, now: float) -> None:
        arrays = [self.working[c] for c in self._cids]
        if self._c >= 2 and self.schedule.total_params > 0:
            _check_shapes(self.schedule, self.working, self._cids)
            self._cycle = _HostCycle(self.schedule, self._c)
            self._stage = self._cycle.launch(arrays)
        else:
            self._landed = True  # nothing to average (multiring.py:302-333 with C < 2)
        if self.network is None:  # no network to play the rounds over: finish now
            self._land()
            for rid, exps in self._expected.items():
                c = len(self._rings[rid].members)
                exps[:] = [2 * (c - 1)] * len(exps)
                self._messages[rid] = 2 * (c - 1) * c
            return
        self._message_cls = getattr(sys.modules.get(type(self.network).__module__), "Message", None)
        if self._message_cls is None:
            raise RavnestError(f"network {type(self.network).__name__} exposes no Message class")
        for ring in self.schedule.rings:
            for pos in range(len(ring.members)):
                self._send(ring, pos, 0, pos % len(ring.members), now)

    def _send(self, ring, pos: int, round_idx: int, chunk_idx: int, now: float) -> None:
        c = len(ring.members)
        dst_pos = (pos + 1) % c
        lo, hi = self._bounds[ring.ring_id][chunk_idx]
        msg = self._message_cls(
            "ring_chunk",
            sender=self.node_of(*ring.members[pos]),
            receiver=self.node_of(*ring.members[dst_pos]),
            step_tag=ring.ring_id,
            payload=np.broadcast_to(_NO_DATA, (hi - lo,)),  # the chunk's float64 size, no data
            extra={"ring": ring.ring_id, "round": round_idx, "chunk": chunk_idx, "to_pos": dst_pos},
        )
        self.network.send(msg, now)

    def handle(self, msg, now: float) -> None:
        rid = msg.extra["ring"]
        ring = self._rings.get(rid)
        if ring is None:
            raise ProtocolError(f"ring {rid}: unknown ring")
        pos = msg.extra["to_pos"]
        round_idx = msg.extra["round"]
        c = len(ring.members)
        if round_idx != self._expected[rid][pos]:
            raise ProtocolError(
                f"ring {rid} member {pos}: got round {round_idx}, expected {self._expected[rid][pos]}"
            )
        self._expected[rid][pos] = round_idx + 1
        self._messages[rid] += 1
        if round_idx + 1 < 2 * (c - 1):
            self._send(ring, pos, round_idx + 1, msg.extra["chunk"], now)

    def _rounds_done(self) -> bool:
        return all(exp == 2 * (len(self._rings[rid].members) - 1)
                   for rid, exps in self._expected.items() for exp in exps)

    def _land(self) -> None:
        if self._landed:
            return
        self._cycle.wait()
        _copy_ranges([(self.working[c], st) for c, st in zip(self._cids, self._stage)], 0,
                     int(self.schedule.total_params))
        self._stage = None
        self._landed = True

    def gpu_ready(self) -> bool:
        """Non-blocking: the GPU cycle has finished (the means may not have
        been copied into ``working`` yet)."""
        return self._landed or (self._cycle is not None and self._cycle.ready())

    def done(self) -> bool:
        if not self._rounds_done():
            return False
        self._land()
        return True

    def stats(self) -> list[RingStats]:
        return [RingStats(rid, min(self._expected[rid]), self._messages[rid]) for rid in sorted(self._expected)]

    def stall_report(self) -> str:
        stuck = []
        for rid in sorted(self._expected):
            c = len(self._rings[rid].members)
            for pos, exp in enumerate(self._expected[rid]):
                if exp < 2 * (c - 1):
                    stuck.append(f"(ring={rid}, round={exp}, member={self._rings[rid].members[pos]})")
        return "waiting on: " + ", ".join(stuck) if stuck else "no ring is stalled"
