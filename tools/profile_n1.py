"""Small program for ncu: C=8 BERT-size clusters co-resident on cuda:0,
2 warm-up cycles + 3 profiled cycles of the ring kernel (lanes=1).
A fourth argument "blend" binds live buffers (the fused-blend kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, ring_starts, synth  # noqa: E402
from paper_2401_01728_b200.plan import LocalRingGroup  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "bert"
c = int(sys.argv[2]) if len(sys.argv) > 2 else 8
acc = sys.argv[3] if len(sys.argv) > 3 else "f64"
blend = len(sys.argv) > 4 and sys.argv[4] == "blend"
lens = WORKLOADS[wl]
total = sum(lens)
xs = [synth(total, m, torch.device("cuda:0")) for m in range(c)]
g = LocalRingGroup(ring_starts(lens), lens, total, [0] * c, torch.float32, acc=acc)
if blend:
    means = [torch.empty_like(x) for x in xs]  # held: the plan keeps raw pointers
    lives = [x + 1e-3 for x in xs]
    g.bind_tensors(xs, means)
    g.bind_live(lives)
else:
    g.bind_tensors(xs)
for _ in range(5):
    g.run()
torch.cuda.synchronize()
g.check()
print("profile_n1 done", wl, c, acc, "blend" if blend else "")
