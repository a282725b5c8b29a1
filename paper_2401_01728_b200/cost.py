"""NVLink-aware cost model of one averaging cycle.

The reference's model (multiring.py:365-394, ``allreduce_cost``) prices each
ring as 2(C-1) rounds over its own slowest link and takes the slowest ring as
the critical path -- rings are assumed to use independent links.  On one
NVSwitch box every ring of a GPU shares the same NVLink ports, and the B200
cycle is one kernel that moves all rings at once, so the cycle costs

    t = alpha + B / beta,     B = 2(C-1)/C * S_total  (bytes per GPU per direction)

with alpha the fixed cost (launch + arrive/depart barriers) and beta the
sustained per-GPU, per-direction NVLink rate of the transport.  ``fit``
calibrates (alpha, beta) by least squares on relative error from sweep rows
(tools/sweep.py output); ``CALIBRATED`` holds the values fitted on
profiles/r02/sweep_r02_n4.jsonl (4 x B200, round-2 kernels, 24 shard-size x
ring-count points from 1 MiB to 8 GiB per cluster; max relative error 4 % for
pull, 15 % for push, 3 % for LL, under 2.1 % above 32 MiB per cluster).  At
2 GPUs the same fit gives pull 18.3 us / 676.5 GB/s, push 26.6 us / 697.6
GB/s (profiles/r02/sweep_r02_n2.jsonl).
"""

from __future__ import annotations

from dataclasses import dataclass

from .schedule import CostReport, RingCost, bytes_per_member


@dataclass(frozen=True)
class NvlinkModel:
    alpha_s: float      # fixed seconds per cycle
    beta_Bps: float     # bytes per second per GPU per direction
    source: str = ""

    def cycle_seconds(self, total_bytes_per_cluster: float, n_clusters: int) -> float:
        return self.alpha_s + bytes_per_member(n_clusters, total_bytes_per_cluster) / self.beta_Bps


CALIBRATED = {
    "pull": NvlinkModel(26.25e-6, 652.1e9, "profiles/r02/sweep_r02_n4.jsonl (4 GPUs)"),
    "push": NvlinkModel(31.30e-6, 689.3e9, "profiles/r02/sweep_r02_n4.jsonl (4 GPUs, adaptive units)"),
    "ll": NvlinkModel(10.42e-6, 298.2e9, "profiles/r02/sweep_r02_n4.jsonl (4 GPUs, <= 16 MiB per cluster)"),
    "nccl": NvlinkModel(3.16e-6, 606.2e9, "profiles/r01/sweep_n4.jsonl; + 23.3 us per ring call"),
}


def fit(rows, key: str) -> tuple[NvlinkModel, float]:
    """Least-squares (relative error) fit of alpha, beta to sweep rows for
    transport ``key``; returns the model and its max relative error."""
    import numpy as np

    x, y = [], []
    for r in rows:
        c = r["n_gpus"]
        x.append([1.0, bytes_per_member(c, r["bytes_per_cluster"])])
        y.append(r[key]["ms"] * 1e-3)
    x, y = np.array(x), np.array(y)
    w = 1.0 / y
    coef, *_ = np.linalg.lstsq(x * w[:, None], y * w, rcond=None)
    model = NvlinkModel(float(coef[0]), float(1.0 / coef[1]), f"fit on {len(rows)} rows")
    err = float(np.max(np.abs(x @ coef - y) / y))
    return model, err


def allreduce_cost_nvlink(schedule, elem_bytes: int = 4, protocol: str = "pull",
                          model: NvlinkModel | None = None) -> CostReport:
    """The reference's CostReport shape, priced for one B200 box.  Per-ring
    entries give each ring's share of the cycle (rings share the links, so
    the cycle -- not the slowest ring -- is the critical path); the
    single-ring baseline is the same bytes in one ring (identical here: the
    one-shot kernel makes ring count irrelevant to the byte count)."""
    m = model or CALIBRATED[protocol]
    c = len(schedule.rings[0].members)
    total = float(schedule.total_params * elem_bytes)
    cycle = m.cycle_seconds(total, c)
    rings = []
    for r in schedule.rings:
        seg = float(r.length * elem_bytes)
        share = bytes_per_member(c, seg) / m.beta_Bps
        rings.append(RingCost(r.ring_id, 2 * (c - 1), seg, bytes_per_member(c, seg), share))
    return CostReport(rings, cycle, cycle)
