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

This file is an attributed INTERFACE MIRROR of those reference items: the
dataclass schemas, the ``dump`` text format, the argument meaning, and the
exception classes and messages are the reference's contract (callers and
golden files depend on them, tests/golden/schedule_kats.json pins 47 layouts
against the unmodified reference).  The construction itself is this
package's own: cluster layouts are reduced to prefix-sum boundary arrays and
each ring's owner is found by bisection.  The GPU path does not depend on
these builders -- any object with ``rings`` (each with ``start``,
``length``, ``members``) and ``total_params`` is accepted, including the
reference's own ``RingSchedule`` from ``plan_session`` (clusterform.py:314-315).
"""

from __future__ import annotations

import bisect
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


def _boundaries(cid, layout) -> list[int]:
    """[s_0 = 0, s_1, ..., s_P = total] of a contiguous layout (submodel p
    spans [s_p, s_{p+1})); LayoutError when a submodel does not start where
    the previous one ended."""
    bounds = [0]
    for sub in layout:
        if int(sub.param_start) != bounds[-1]:
            raise LayoutError(f"cluster {cid}: submodels not contiguous")
        bounds.append(bounds[-1] + int(sub.param_len))
    return bounds


def _owner(bounds: list[int], lo: int, hi: int):
    """Index of the first submodel whose span holds [lo, hi), or None.  For a
    non-empty range the holder is unique and bisection finds it; an empty
    range (a zero-length ring) takes the first span reaching it."""
    if lo < hi:
        p = bisect.bisect_right(bounds, lo) - 1
        return p if 0 <= p < len(bounds) - 1 and hi <= bounds[p + 1] else None
    return next((q for q in range(len(bounds) - 1) if bounds[q] <= lo and hi <= bounds[q + 1]), None)


def build_ring_schedule(cluster_layouts: dict[int, Sequence]) -> RingSchedule:
    """One ring per segment of the union of all clusters' submodel cuts.

    Every cluster's layout must be contiguous from 0 and cover the same total;
    the cuts must nest so that the segment count equals the largest peer
    count.  Each ring lists, per cluster in ascending id order, the peer
    whose submodel contains the segment (multiring.py:56-105 contract).
    """
    if not cluster_layouts:
        raise LayoutError("no cluster layouts given")
    ids = sorted(cluster_layouts)
    bounds = {cid: _boundaries(cid, cluster_layouts[cid]) for cid in ids}
    totals = {cid: b[-1] for cid, b in bounds.items()}
    if len(set(totals.values())) > 1:
        raise LayoutError(f"layouts cover different totals: {totals}")
    total = totals[ids[0]]
    # interior cuts: every submodel start above 0, over all clusters
    interior = sorted({x for b in bounds.values() for x in b[1:-1] if x > 0})
    n_peers = max(len(b) - 1 for b in bounds.values())
    if len(interior) + 1 != n_peers:
        raise LayoutError(
            f"cluster boundaries do not nest: {len(interior) + 1} segments needed "
            f"but max peer count is {n_peers}"
        )
    edges = [0, *interior, total]
    rings = []
    for rid in range(len(edges) - 1):
        lo, hi = edges[rid], edges[rid + 1]
        members = []
        for cid in ids:
            p = _owner(bounds[cid], lo, hi)
            if p is None:
                raise LayoutError(f"cluster {cid}: no peer owns range [{lo},{hi})")
            members.append((cid, p))
        rings.append(Ring(rid, lo, hi - lo, tuple(members)))
    return RingSchedule(tuple(rings), total)


def validate_schedule(schedule: RingSchedule, cluster_layouts: dict[int, Sequence]) -> None:
    """Independent re-check of every schedule invariant (multiring.py:108-131
    contract): rings tile [0, total) in order, one ring per peer of the
    widest cluster, one member per cluster in id order, and each member's
    submodel holds the ring's range."""
    starts = [r.start for r in schedule.rings]
    ends = [r.start + r.length for r in schedule.rings]
    if any(r.length < 0 for r in schedule.rings) or starts != [0, *ends[:-1]][:len(starts)]:
        raise LayoutError("rings do not tile the parameter space")
    if (ends[-1] if ends else 0) != schedule.total_params:
        raise LayoutError("rings do not cover all parameters")
    ids = sorted(cluster_layouts)
    n_peers = max(len(cluster_layouts[c]) for c in ids)
    if len(schedule.rings) != n_peers:
        raise LayoutError(f"{len(schedule.rings)} rings but max peer count is {n_peers}")
    for ring in schedule.rings:
        if [cid for cid, _ in ring.members] != ids:
            raise LayoutError(f"ring {ring.ring_id} lacks one member per cluster")
        for cid, peer in ring.members:
            sub = cluster_layouts[cid][peer]
            lo, hi = int(sub.param_start), int(sub.param_start) + int(sub.param_len)
            if ring.start < lo or ring.start + ring.length > hi:
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
