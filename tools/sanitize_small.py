"""Small single-process workload for compute-sanitizer (one tool per run):
co-resident cycles through every kernel family (TMA, register path with
misaligned buffers, scalar path, fp64, native fold, blend) on small sizes,
each checked against the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ring_oracle  # noqa: E402
import paper_2401_01728_b200 as rv  # noqa: E402
from paper_2401_01728_b200.blend import blend_  # noqa: E402
from paper_2401_01728_b200.schedule import Ring, RingSchedule  # noqa: E402


def sched(lens, c):
    rings, s = [], 0
    for i, n in enumerate(lens):
        rings.append(Ring(i, s, n, tuple((m, 0) for m in range(c))))
        s += n
    return RingSchedule(tuple(rings), s)


def check(lens, c, dtype, acc, offsets):
    sc = sched(lens, c)
    npdt = np.float32 if dtype == torch.float32 else np.float64
    rng = np.random.Generator(np.random.Philox(key=c * 7 + len(lens)))
    rows = [rng.normal(0, 1, sc.total_params).astype(npdt) for _ in range(c)]
    want = ring_oracle.ring_mean([r.start for r in sc.rings], lens, rows, acc=acc)
    views = {}
    for m in range(c):
        buf = torch.empty(sc.total_params + offsets[m] + 2, dtype=dtype, device="cuda")
        v = buf[offsets[m]:offsets[m] + sc.total_params]
        v.copy_(torch.from_numpy(rows[m]))
        views[m] = v
    rv.ring_mean_(sc, views, acc=acc)
    for m in range(c):
        got = views[m].cpu().numpy()
        assert np.array_equal(got, want[m].astype(npdt)), (lens, c, dtype, acc, offsets)


def main():
    torch.cuda.set_device(0)
    for c in (2, 3, 8):
        for lens in ([1, 0, 4099, 77], [65536 + 3, 5]):
            check(lens, c, torch.float32, "f64", [0] * c)          # TMA path
            check(lens, c, torch.float32, "f64", [1] * c)          # register path, congruent misalignment
            check(lens, c, torch.float32, "f64", [m % 3 for m in range(c)])  # scalar path
            check(lens, c, torch.float64, "f64", [0] * c)
            check(lens, c, torch.float32, "native", [0] * c)
    n = 10001
    live, snap, mean = (torch.randn(n, device="cuda") for _ in range(3))
    want = ring_oracle.blend(mean.cpu().numpy(), live.cpu().numpy(), snap.cpu().numpy())
    blend_(live, snap, mean)
    assert np.array_equal(live.cpu().numpy(), want)
    torch.cuda.synchronize()
    print("sanitize_small ok")


if __name__ == "__main__":
    main()
