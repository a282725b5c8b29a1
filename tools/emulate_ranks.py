"""C rank plans spread over the box's GPUs in ONE process (LoopbackGroup
with devices=...): e.g. the 8-rank push cycle an 8-GPU job runs, with its
real CB = 8 kernel at C = 8 and real NVLink traffic, on a 4-GPU box (two
ranks per GPU).  Checks every element of every rank against the C oracle,
then times cycles with CUDA events on rank 0's device.

Per GPU the NVLink bytes are NOT those of a C-GPU job: two ranks share a
GPU, so its links carry both ranks' remote traffic (scatter + means to the
ranks on other GPUs) and the local pairs move through HBM.  The line reports
the per-GPU link bytes actually moved.

    python tools/emulate_ranks.py [--ranks 8] [--workload bert] [--proto push]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, ring_starts  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_2401_01728_b200.loopback import LoopbackGroup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--workload", default="bert")
ap.add_argument("--proto", default="push")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--check", type=int, default=1)
ap.add_argument("--blend", type=int, default=0, help="config 4: average snapshots into means, fused tau=4 blend")
args = ap.parse_args()

ng = torch.cuda.device_count()
c = args.ranks
lens = WORKLOADS[args.workload]
starts = ring_starts(lens)
total = sum(lens)
devices = [m * ng // c for m in range(c)]
xs = []
for m in range(c):
    g = torch.Generator(device=f"cuda:{devices[m]}").manual_seed(20241018 * 1000 + m)
    xs.append(torch.randn(total, device=f"cuda:{devices[m]}", generator=g) * 0.02)
grp = LoopbackGroup(starts, lens, total, c, torch.float32, protocol=args.proto, devices=devices, timeout_s=20.0)
means = lives = None
if args.blend:
    means = [torch.empty_like(x) for x in xs]
    lives = []
    for m, x in enumerate(xs):  # live = snap - 1e-3 * (4 stale N(0,1) updates)
        g = torch.Generator(device=x.device).manual_seed(7919 + m)
        lives.append(x - 1e-3 * torch.randn(total, device=x.device, generator=g) * 2.0)
    grp.bind_tensors(xs, means)
    grp.bind_live(lives)
else:
    grp.bind_tensors(xs)
ok = None
if args.check and not args.blend:
    rows = [x.cpu().numpy() for x in xs]
    want = np.empty_like(rows[0])
    c_oracle.ring_mean_into(c_oracle.MODE_F32_ACC64, starts, lens, rows, None, [want] * c,
                            threads=len(os.sched_getaffinity(0)))
    del rows
    grp.run()
    for d in set(devices):
        torch.cuda.synchronize(d)
    grp.check()
    ok = all(np.array_equal(x.cpu().numpy().view(np.uint32), want.view(np.uint32)) for x in xs)
for _ in range(5):
    grp.run()
for d in set(devices):
    torch.cuda.synchronize(d)
cur = torch.cuda.current_stream(devices[0])
times = []
for _ in range(args.steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    grp.run()
    b.record(cur)
    b.synchronize()
    times.append(a.elapsed_time(b))
grp.check()
ms = statistics.median(times)
S = total * 4
# per GPU, per direction: each of its ranks sends its chunk to every rank on
# another GPU (scatter) and its mean chunk to the same ranks (all-gather)
per_gpu = {}
for m in range(c):
    remote = sum(1 for q in range(c) if devices[q] != devices[m])
    per_gpu[devices[m]] = per_gpu.get(devices[m], 0) + 2 * remote * S / c
link = max(per_gpu.values())
print(json.dumps({"ranks": c, "gpus": ng, "ranks_per_gpu": c // ng, "workload": args.workload, "proto": args.proto,
                  "blend": bool(args.blend),
                  "bitwise_vs_oracle": ok, "ms_per_cycle_median": round(ms, 4), "ms_min": round(min(times), 4),
                  "link_bytes_per_gpu_per_direction": int(link),
                  "link_gbps_per_gpu": round(link / (ms * 1e-3) / 1e9, 1),
                  "busbw_equiv_c_gpus": round(S * 2 * (c - 1) / c / (ms * 1e-3) / 1e9, 1)}), flush=True)
grp.close()
