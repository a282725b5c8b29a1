"""Where the time of the numpy drop-in goes (BERT-base C=8, float64 in/out):
the threaded float64 copy-in alone, the pinned H2D / kernel / D2H pipeline
alone, and the whole ``apply_ring_mean`` call.  Host wall times, median of 5.

    python tools/e2e_seam_probe.py [workload]
"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, host_inputs, ring_starts  # noqa: E402
from paper_2401_01728_b200 import multiring as mr  # noqa: E402
from paper_2401_01728_b200.schedule import ParamRange, build_ring_schedule  # noqa: E402

lens = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "bert"]
c = 8
total = sum(lens)
sched = build_ring_schedule({m: [ParamRange(s, n) for s, n in zip(ring_starts(lens), lens)] for m in range(c)})
xs = [x.astype(np.float64) for x in host_inputs(total, c)]
vals = dict(enumerate(xs))


def med(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


stage = [torch.empty(total, dtype=torch.float64, pin_memory=True).numpy() for _ in range(c)]
pairs = list(zip(stage, xs))
print(f"copy-in (pool {mr._copy_pool()._max_workers} threads): "
      f"{med(lambda: mr._copy_ranges(pairs, 0, total)):.1f} ms for {c * total * 8 / 1e9:.1f} GB")
for k in (1, 4, 8, 16, 24):
    pool = mr.ThreadPoolExecutor(max_workers=k)
    old = mr._COPY_POOL
    mr._COPY_POOL = pool
    print(f"  copy-in with {k} threads: {med(lambda: mr._copy_ranges(pairs, 0, total)):.1f} ms")
    mr._COPY_POOL = old
    pool.shutdown()

cyc = mr._HostCycle(sched, c)
ptrs = [a.ctypes.data for a in stage]


def pipeline():
    for lane in range(len(cyc.ranges)):
        cyc.plan.run_host_lanes(lane, 1, ptrs, ptrs, cyc.streams)
    torch.cuda.synchronize()


print(f"H2D+kernel+D2H pipeline ({len(cyc.ranges)} lanes, {len(cyc.streams)} streams): {med(pipeline):.1f} ms")
print(f"apply_ring_mean (numpy float64 in/out): {med(lambda: mr.apply_ring_mean(sched, vals)):.1f} ms")
out = mr.apply_ring_mean(sched, vals)
print("members agree:", all(np.array_equal(out[0], out[m]) for m in range(1, c)))
