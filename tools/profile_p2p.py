"""Single process driving N GPUs (one cluster each, BERT-base rings): a few
cycles for ncu.  Devices launch in order, so when ncu profiles the last
device (--devices N-1, application replay) its peers' kernels are already
running.  Stalls are reported, not raised (so a profiling pass can finish).

    python tools/profile_p2p.py [workload] [pull|push|ll] [blend] [--gpus N] [--min-cb CB]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, ring_starts, synth  # noqa: E402
from paper_2401_01728_b200.plan import LocalRingGroup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="bert")
ap.add_argument("proto", nargs="?", default="pull")
ap.add_argument("blend", nargs="?", default="")
ap.add_argument("--gpus", type=int, default=2)
ap.add_argument("--min-cb", type=int, default=0)
ap.add_argument("--cycles", type=int, default=10)
args = ap.parse_args()

lens = WORKLOADS[args.workload]
n = args.gpus
total = sum(lens)
xs = [synth(total, m, torch.device(f"cuda:{m}")) for m in range(n)]
opts = {"min_cb": args.min_cb} if args.min_cb else None
g = LocalRingGroup(ring_starts(lens), lens, total, list(range(n)), torch.float32, protocol=args.proto, options=opts)
if args.blend == "blend":  # fused delayed-update blend
    means = [torch.empty_like(x) for x in xs]  # held: the plan keeps raw pointers
    lives = [x + 1e-3 for x in xs]
    g.bind_tensors(xs, means)
    g.bind_live(lives)
else:
    g.bind_tensors(xs)
streams = {d: torch.cuda.Stream(device=d) for d in range(n)}
for _ in range(5):
    g.run(streams)
for d in range(n):
    torch.cuda.synchronize(d)
for plan in g.plans.values():
    rc, diag = plan.status()
    print("device", plan.device, "status", rc, diag)
last = n - 1
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with torch.cuda.device(last):
    ev[0].record(streams[last])
    for _ in range(args.cycles):
        g.run(streams)
    ev[1].record(streams[last])
for d in range(n):
    torch.cuda.synchronize(d)
ms = ev[0].elapsed_time(ev[1]) / args.cycles
bus = total * 4 / ms / 1e6 * 2 * (n - 1) / n
print(f"profile_p2p {args.proto} C={n} min_cb={args.min_cb}: {ms:.4f} ms per cycle, {bus:.1f} GB/s busbw")
