"""Single process, 2 GPUs (one cluster each, BERT-base rings): a few pull
cycles for ncu.  Device 0's kernel is launched before device 1's, so when
ncu profiles device 1 (--devices 1) its peer kernel is already running.
Stalls are reported, not raised (so a profiling pass can finish)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, ring_starts, synth  # noqa: E402
from paper_2401_01728_b200.plan import LocalRingGroup  # noqa: E402

lens = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "bert"]
proto = sys.argv[2] if len(sys.argv) > 2 else "pull"
blend = len(sys.argv) > 3 and sys.argv[3] == "blend"  # fused delayed-update blend
total = sum(lens)
xs = [synth(total, m, torch.device(f"cuda:{m}")) for m in range(2)]
g = LocalRingGroup(ring_starts(lens), lens, total, [0, 1], torch.float32, protocol=proto)
if blend:
    means = [torch.empty_like(x) for x in xs]  # held: the plan keeps raw pointers
    lives = [x + 1e-3 for x in xs]
    g.bind_tensors(xs, means)
    g.bind_live(lives)
else:
    g.bind_tensors(xs)
streams = {d: torch.cuda.Stream(device=d) for d in (0, 1)}
for _ in range(5):
    g.run(streams)
for d in (0, 1):
    torch.cuda.synchronize(d)
for plan in g.plans.values():
    rc, diag = plan.status()
    print("device", plan.device, "status", rc, diag)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with torch.cuda.device(1):
    ev[0].record(streams[1])
    for _ in range(10):
        g.run(streams)
    ev[1].record(streams[1])
for d in (0, 1):
    torch.cuda.synchronize(d)
ms = ev[0].elapsed_time(ev[1]) / 10
print(f"profile_p2p {proto}: {ms:.4f} ms per cycle, {total * 4 / ms / 1e6:.1f} GB/s busbw (C=2)")
