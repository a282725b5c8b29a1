"""Small program for ncu: C=8 BERT-size clusters co-resident on cuda:0,
2 warm-up cycles + 3 profiled cycles of the ring kernel (lanes=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, ring_starts, synth  # noqa: E402
from paper_2401_01728_b200.plan import LocalRingGroup  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "bert"
c = int(sys.argv[2]) if len(sys.argv) > 2 else 8
acc = sys.argv[3] if len(sys.argv) > 3 else "f64"
lens = WORKLOADS[wl]
total = sum(lens)
xs = [synth(total, m, torch.device("cuda:0")) for m in range(c)]
g = LocalRingGroup(ring_starts(lens), lens, total, [0] * c, torch.float32, acc=acc)
g.bind_tensors(xs)
for _ in range(5):
    g.run()
torch.cuda.synchronize()
g.check()
print("profile_n1 done", wl, c, acc)
