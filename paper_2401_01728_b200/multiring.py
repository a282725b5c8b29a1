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
import sys
from typing import Callable

import numpy as np

from .errors import ConfigError, LayoutError, RavnestError, StallError
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


def apply_ring_mean(schedule, cluster_params: dict, acc: str = "f64") -> dict:
    """Synchronous cycle with the reference's contract: inputs untouched,
    new arrays returned (multiring.py:302-333).

    numpy inputs are widened to float64 exactly as the reference does
    (multiring.py:309) and averaged co-resident on the current GPU; the
    result is float64 and bitwise equal to the reference.  CUDA tensors are
    cloned and averaged where they live.
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
    work = {c: np.array(cluster_params[c], dtype=np.float64) for c in cids}
    if len(cids) < 2:
        return work
    _check_shapes(schedule, work, cids)
    torch = _torch()
    dev = torch.cuda.current_device()
    on_dev = {c: torch.from_numpy(work[c]).to(f"cuda:{dev}") for c in cids}
    ring_mean_(schedule, on_dev, acc=acc)
    for c in cids:
        work[c][...] = on_dev[c].cpu().numpy()
    return work


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
    (multiring.py:254-299).  ``network``/``node_of`` only shape timing in the
    reference, never the arithmetic (test_multiring.py:173-205), so the GPU
    cycle ignores them.  An event budget smaller than the cycle's message
    count raises StallError naming the blocked (ring, round, member), as the
    reference does under FIFO delivery."""
    cids = sorted(cluster_params)
    if len(cids) < 2:
        raise ConfigError("all-reduce needs at least 2 clusters")
    _check_shapes(schedule, cluster_params, cids)
    c = len(cids)
    needed = sum(2 * (c - 1) * c for _ in schedule.rings)
    if max_events is not None and max_events < needed:
        expected = _ideal_network_progress(schedule, c, max_events, node_of)
        raise StallError(
            f"event budget of {max_events} exhausted\n"
            + "all-reduce incomplete: " + _stall_text(schedule, expected, c)
        )
    out = apply_ring_mean(schedule, cluster_params)
    return out, schedule_stats(schedule, c)


class AllReduceController:
    """Drain-barrier seam (orchestrator.py:339-363): the reference drives a
    self-clocked ring over its simulated network; this one launches the GPU
    cycle at ``kickoff`` and posts one zero-byte token per ring so the
    orchestrator's router still sees ring traffic and calls ``handle`` /
    ``done``.  ``working`` is averaged in place, as the reference does."""

    def __init__(self, schedule, working: dict, network, node_of: Callable[[int, int], str]):
        self.schedule = schedule
        self.working = working
        self.network = network
        self.node_of = node_of
        self._cids = sorted(working)
        self._c = len(self._cids)
        self._pending: set[int] = set()
        self._finished = False
        self._delivered = 0

    def kickoff(self, now: float) -> None:
        result = apply_ring_mean(self.schedule, self.working)
        for cid in self._cids:
            self.working[cid][...] = result[cid]
        self._finished = True
        if self.network is None:
            return
        message_cls = getattr(sys.modules.get(type(self.network).__module__), "Message", None)
        if message_cls is None:
            return
        for ring in self.schedule.rings:
            src, dst = ring.members[0], ring.members[1 % self._c]
            msg = message_cls(
                "ring_chunk",
                sender=self.node_of(*src),
                receiver=self.node_of(*dst),
                step_tag=ring.ring_id,
                payload=np.zeros(0),
                extra={"ring": ring.ring_id, "round": 2 * (self._c - 1) - 1, "chunk": 0, "to_pos": 1 % self._c},
            )
            self._pending.add(ring.ring_id)
            self.network.send(msg, now)

    def handle(self, msg, now: float) -> None:
        rid = msg.extra["ring"]
        if rid not in self._pending:
            from .errors import ProtocolError

            raise ProtocolError(f"ring {rid}: unexpected token")
        self._pending.discard(rid)
        self._delivered += 1

    def done(self) -> bool:
        return self._finished and not self._pending

    def stats(self) -> list[RingStats]:
        return schedule_stats(self.schedule, self._c) if self.done() else [
            RingStats(int(r.ring_id), 0, 0) for r in self.schedule.rings
        ]

    def stall_report(self) -> str:
        if self.done():
            return "no ring is stalled"
        return "waiting on: " + ", ".join(f"(ring={rid}, token)" for rid in sorted(self._pending))
