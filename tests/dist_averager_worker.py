"""Multi-process check of AsyncAverager (launched by tests/test_dist_gpu.py):
live training updates, averaging every kappa updates on a side stream, tau
stale updates blended back.  Every rank also replays all ranks' updates on a
shadow copy and applies the oracle mean + oracle blend at the same points;
its live parameters must match its shadow bit for bit."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ring_oracle  # noqa: E402
from paper_2401_01728_b200.averager import AsyncAverager  # noqa: E402


def grad(rank, t, n, dev):
    g = torch.Generator(device=dev).manual_seed(1000 * rank + t)
    return torch.randn(n, device=dev, generator=g)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    lens = [70001, 3, 33333, 2 * world + 1]
    starts = list(np.cumsum([0] + lens[:-1]))
    n = sum(lens)
    eta = 1e-2
    failures = 0
    for kappa, tau, graph, proto in ((3, 0, False, "pull"), (4, 2, False, "push"), (5, 3, True, "auto"),
                                     (2, 1, True, "ll")):
        init = [torch.randn(n, device=dev, generator=torch.Generator(device=dev).manual_seed(7 + m))
                for m in range(world)]
        live = init[rank].clone()
        avg = AsyncAverager(live, starts=starts, lens=lens, kappa=kappa, tau=tau, protocol=proto, graph=graph,
                            sm_budget=(8 if graph else 0))
        shadow = [x.clone() for x in init]
        snap = None
        pending = None
        steps = 4 * kappa + tau + 1
        for t in range(1, steps + 1):
            g_t = grad(rank, t, n, dev)
            avg.before_update()
            live.sub_(g_t, alpha=eta)
            avg.step()
            for m in range(world):
                shadow[m].sub_(grad(m, t, n, dev), alpha=eta)
            # reference semantics on the shadow
            if pending is not None and t >= pending + tau:
                mean = ring_oracle.ring_mean(starts, lens, [s.cpu().numpy() for s in snap])
                for m in range(world):
                    b = ring_oracle.blend(mean[m].astype(np.float32), shadow[m].cpu().numpy(), snap[m].cpu().numpy())
                    shadow[m] = torch.from_numpy(b).to(dev)
                pending = None
            if t % kappa == 0 and pending is None:
                snap = [s.clone() for s in shadow]
                pending = t
                if tau == 0:
                    mean = ring_oracle.ring_mean(starts, lens, [s.cpu().numpy() for s in snap])
                    for m in range(world):
                        b = ring_oracle.blend(mean[m].astype(np.float32), shadow[m].cpu().numpy(),
                                              snap[m].cpu().numpy())
                        shadow[m] = torch.from_numpy(b).to(dev)
                    pending = None
        avg.flush()
        if pending is not None:
            mean = ring_oracle.ring_mean(starts, lens, [s.cpu().numpy() for s in snap])
            for m in range(world):
                b = ring_oracle.blend(mean[m].astype(np.float32), shadow[m].cpu().numpy(), snap[m].cpu().numpy())
                shadow[m] = torch.from_numpy(b).to(dev)
        torch.cuda.synchronize()
        avg.group.check()
        got = live.cpu().numpy().view(np.uint32)
        want = shadow[rank].cpu().numpy().view(np.uint32)
        if not np.array_equal(got, want):
            print(f"rank {rank} kappa={kappa} tau={tau} graph={graph}: {int((got != want).sum())} mismatches",
                  flush=True)
            failures += 1
        if avg.cycles != (steps // kappa):
            print(f"rank {rank}: {avg.cycles} cycles, expected {steps // kappa}", flush=True)
            failures += 1
        dist.barrier()
        avg.close()
    t = torch.tensor([failures])
    dist.all_reduce(t)
    if rank == 0:
        print(f"AVERAGER {'OK' if int(t) == 0 else 'FAIL'} world={world} failures={int(t)}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(t) == 0 else 1)


if __name__ == "__main__":
    main()
