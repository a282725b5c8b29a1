"""Ring schedule: which parameter ranges form rings, and who sits in each.

Host-side mirror of the reference's schedule types and builders
(/root/reference/pkg/src/ravnest/multiring.py):

====================  =========================================
this module            reference
====================  =========================================
ParamRange            multiring.py:23-28
Ring, RingSchedule    multiring.py:31-53 (``dump`` schema ravnest-rings-v1)
build_ring_schedule   multiring.py:56-105
validate_schedule     multiring.py:108-131
chunk_bounds          multiring.py:134-144
RingStats             multiring.py:147-151
bytes_per_member      multiring.py:340-342
allreduce_cost        multiring.py:345-394 (RingCost, CostReport)
====================  =========================================

Same names, argument meaning and exception classes, so a schedule produced
here (or by the reference's ``plan_session``, clusterform.py:314-315) feeds
the GPU path unchanged: any object with ``rings`` (each with ``start``,
``length``, ``members``) and ``total_params`` is accepted.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

from .errors import LayoutError

SCHEMA = "ravnest-rings-v1"


@dataclass(frozen=True)
class ParamRange:
    """A submodel seen only through its span of the flat parameter vector."""

    param_start: int
    param_len: int


@dataclass(frozen=True)
class Ring:
    ring_id: int
    start: int
    length: int
    members: tuple[tuple[int, int], ...]  # (cluster_id, peer_index), ascending cluster id


@dataclass(frozen=True)
class RingSchedule:
    rings: tuple[Ring, ...]
    total_params: int

    @property
    def n_clusters(self) -> int:
        return len(self.rings[0].members)

    def dump(self) -> str:
        out = [f"# schema: {SCHEMA}"]
        for ring in self.rings:
            who = ",".join("(%d,%d)" % m for m in ring.members)
            out.append("ring_id=%d,start=%d,len=%d,members=[%s]" % (ring.ring_id, ring.start, ring.length, who))
        return "\n".join(out) + "\n"


@dataclass
class RingStats:
    ring_id: int
    rounds: int
    messages: int


def _spans(layout) -> list[tuple[int, int]]:
    return [(int(sub.param_start), int(sub.param_len)) for sub in layout]


def build_ring_schedule(cluster_layouts: dict[int, Sequence]) -> RingSchedule:
    """One ring per segment of the union of all clusters' submodel cuts.

    Every cluster's layout must be contiguous from 0 and cover the same total;
    the cuts must nest so that the segment count equals the largest peer
    count.  Each ring lists, per cluster in ascending id order, the peer
    whose submodel contains the segment.
    """
    if not cluster_layouts:
        raise LayoutError("no cluster layouts given")
    order = sorted(cluster_layouts)
    spans = {cid: _spans(cluster_layouts[cid]) for cid in order}
    totals = {}
    for cid in order:
        expect = 0
        for start, length in spans[cid]:
            if start != expect:
                raise LayoutError(f"cluster {cid}: submodels not contiguous")
            expect = start + length
        totals[cid] = expect
    if len(set(totals.values())) > 1:
        raise LayoutError(f"layouts cover different totals: {totals}")
    total = totals[order[0]]

    cut_set = set()
    for cid in order:
        cut_set.update(start for start, _ in spans[cid] if start > 0)
    cuts = sorted(cut_set)
    widest = max(len(spans[cid]) for cid in order)
    if len(cuts) + 1 != widest:
        raise LayoutError(
            f"cluster boundaries do not nest: {len(cuts) + 1} segments needed "
            f"but max peer count is {widest}"
        )

    edges = [0, *cuts, total]
    rings = []
    for rid, (lo, hi) in enumerate(zip(edges[:-1], edges[1:])):
        members = []
        for cid in order:
            owner = next(
                (i for i, (s, n) in enumerate(spans[cid]) if s <= lo and hi <= s + n), None
            )
            if owner is None:
                raise LayoutError(f"cluster {cid}: no peer owns range [{lo},{hi})")
            members.append((cid, owner))
        rings.append(Ring(rid, lo, hi - lo, tuple(members)))
    return RingSchedule(tuple(rings), total)


def validate_schedule(schedule: RingSchedule, cluster_layouts: dict[int, Sequence]) -> None:
    """Independent re-check of every schedule invariant."""
    expect = 0
    for ring in schedule.rings:
        if ring.length < 0 or ring.start != expect:
            raise LayoutError("rings do not tile the parameter space")
        expect += ring.length
    if expect != schedule.total_params:
        raise LayoutError("rings do not cover all parameters")
    order = sorted(cluster_layouts)
    widest = max(len(cluster_layouts[c]) for c in order)
    if len(schedule.rings) != widest:
        raise LayoutError(f"{len(schedule.rings)} rings but max peer count is {widest}")
    for ring in schedule.rings:
        if [cid for cid, _ in ring.members] != order:
            raise LayoutError(f"ring {ring.ring_id} lacks one member per cluster")
        for cid, peer in ring.members:
            sub = cluster_layouts[cid][peer]
            if not (sub.param_start <= ring.start and ring.start + ring.length <= sub.param_start + sub.param_len):
                raise LayoutError(f"ring {ring.ring_id} range outside cluster {cid} peer {peer}")


def chunk_bounds(start: int, length: int, c: int) -> list[tuple[int, int]]:
    """C contiguous chunks of [start, start+length); the remainder goes to
    the lowest chunk indices.  The GPU plan applies the same split."""
    base, rem = divmod(length, c)
    sizes = [base + 1] * rem + [base] * (c - rem)
    out, lo = [], start
    for n in sizes:
        out.append((lo, lo + n))
        lo += n
    return out


def ring_arrays(schedule) -> tuple[list[int], list[int]]:
    """(starts, lengths) of the rings, in schedule order."""
    return [int(r.start) for r in schedule.rings], [int(r.length) for r in schedule.rings]


def schedule_stats(schedule, n_clusters: int) -> list[RingStats]:
    """What ``AllReduceController.stats`` reports after a full cycle
    (multiring.py:234-238): 2(C-1) rounds, C messages per round."""
    rounds = 2 * (n_clusters - 1)
    return [RingStats(int(r.ring_id), rounds, rounds * n_clusters) for r in schedule.rings]


# ---------------------------------------------------------------------------
# cost model (unchanged semantics; calibrated variants live in bench.py)


def bytes_per_member(c: int, seg_bytes: float) -> float:
    """Bytes one member sends (and receives) per cycle: 2(C-1) chunks of S/C."""
    return 2.0 * (c - 1) * seg_bytes / c


@dataclass
class RingCost:
    ring_id: int
    rounds: int
    seg_bytes: float
    bytes_per_member: float
    seconds: float


@dataclass
class CostReport:
    rings: list[RingCost]
    critical_seconds: float
    single_ring_seconds: float

    @property
    def critical_ratio(self) -> float:
        return self.critical_seconds / self.single_ring_seconds


def allreduce_cost(
    schedule: RingSchedule,
    bandwidth: float | Callable[[tuple[int, int], tuple[int, int]], float],
    latency: float = 0.0,
    elem_bytes: int = 8,
) -> CostReport:
    """Analytic ring cost: each ring takes 2(C-1) rounds of S/C bytes over its
    slowest link; the cycle's critical path is the slowest ring, compared with
    one ring carrying everything.  ``elem_bytes`` defaults to the reference's
    float64 (multiring.py:383,392)."""
    link = bandwidth if callable(bandwidth) else (lambda a, b: bandwidth)
    out = []
    slowest_link = float("inf")
    for ring in schedule.rings:
        c = len(ring.members)
        rounds = 2 * (c - 1)
        seg = float(ring.length * elem_bytes)
        bw = min(link(ring.members[i], ring.members[(i + 1) % c]) for i in range(c))
        slowest_link = min(slowest_link, bw)
        secs = rounds * (latency + (seg / c) / bw)
        out.append(RingCost(ring.ring_id, rounds, seg, bytes_per_member(c, seg), secs))
    c = len(schedule.rings[0].members)
    everything = float(schedule.total_params * elem_bytes)
    single = 2 * (c - 1) * (latency + (everything / c) / slowest_link)
    return CostReport(out, max(r.seconds for r in out), single)
