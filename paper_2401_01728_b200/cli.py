"""Command line for the averaging path.

    python -m paper_2401_01728_b200.cli allreduce-bench --clusters 8 --rings 4 --shard-mib 105
    python -m paper_2401_01728_b200.cli allreduce-bench --plan plan.txt
    python -m paper_2401_01728_b200.cli rings --plan plan.txt

``allreduce-bench`` mirrors the reference's subcommand (cli.py:158-187),
which prints only its analytic per-ring model (multiring.py:365-394), and
adds the NVLink-calibrated model of the B200 cycle (cost.py).  Measured
numbers come from ``bench.py`` / ``tools/sweep.py`` (real kernels, torchrun).
"""

from __future__ import annotations

import argparse
import json
import sys

from . import cost, formats
from .schedule import Ring, RingSchedule, allreduce_cost


def _equal_schedule(clusters: int, rings: int, params_per_ring: int) -> RingSchedule:
    out, start = [], 0
    for rid in range(rings):
        out.append(Ring(rid, start, params_per_ring, tuple((c, rid) for c in range(clusters))))
        start += params_per_ring
    return RingSchedule(tuple(out), start)


def cmd_allreduce_bench(args) -> int:
    if args.plan:
        sched = formats.read_plan_file(args.plan).schedule
    else:
        sched = _equal_schedule(args.clusters, args.rings, args.shard_mib * (1 << 20) // 4)
    c = len(sched.rings[0].members)
    ref = allreduce_cost(sched, bandwidth=args.bandwidth, latency=args.latency, elem_bytes=4)
    rows = {
        "clusters": c, "rings": len(sched.rings), "params": sched.total_params,
        "reference_model": {"critical_s": ref.critical_seconds, "single_ring_s": ref.single_ring_seconds,
                            "assumes": f"independent links of {args.bandwidth:.3g} B/s per ring"},
    }
    for proto in ("ll", "pull", "push", "nccl"):
        m = cost.CALIBRATED[proto]
        t = m.cycle_seconds(sched.total_params * 4.0, c)
        if proto == "nccl":
            t += 23.3e-6 * (len(sched.rings) - 1)
        rows[f"b200_{proto}"] = {"cycle_s": t, "bus_GBps": sched.total_params * 4.0 / t * 2 * (c - 1) / c / 1e9,
                                 "calibration": m.source}
    print(json.dumps(rows, indent=1))
    return 0


def cmd_rings(args) -> int:
    plan = formats.read_plan_file(args.plan)
    sys.stdout.write(plan.schedule.dump())
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2401_01728_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("allreduce-bench")
    b.add_argument("--plan")
    b.add_argument("--clusters", type=int, default=8)
    b.add_argument("--rings", type=int, default=4)
    b.add_argument("--shard-mib", type=int, default=105)
    b.add_argument("--bandwidth", type=float, default=770e9)
    b.add_argument("--latency", type=float, default=0.0)
    b.set_defaults(fn=cmd_allreduce_bench)
    r = sub.add_parser("rings")
    r.add_argument("--plan", required=True)
    r.set_defaults(fn=cmd_rings)
    args = ap.parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
