"""Asynchronous data-parallel training with multi-ring parameter averaging
(Ravnest's Algorithm 2 on B200s).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 examples/train_async.py

Every rank is one cluster: a torch MLP whose parameters are views into one
flat arena (ParamArena), trained with SGD on its own synthetic data shard.
Every kappa updates the arena is snapshotted and averaged across ranks on a
side stream (one NVLink kernel per rank); training keeps going, and the
tau updates made meanwhile are blended onto the average.  The script times
three regimes on the same model and prints one JSON line (rank 0):

  * no averaging        -- the training step alone
  * synchronous, tau=0  -- averaging on the critical path every kappa steps
  * asynchronous, tau   -- averaging overlapped with tau training steps
"""

import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_01728_b200.arena import ParamArena  # noqa: E402
from paper_2401_01728_b200.averager import AsyncAverager  # noqa: E402


def build(width: int, depth: int, dev):
    layers = []
    for _ in range(depth):
        layers += [torch.nn.Linear(width, width), torch.nn.GELU()]
    layers.append(torch.nn.Linear(width, 10))
    return torch.nn.Sequential(*layers).to(dev)


def run(regime: str, args, rank: int, dev, sm_budget: int = 0):
    torch.manual_seed(1234)  # same init on every rank (as the reference's clusters)
    model = build(args.width, args.depth, dev)
    arena = ParamArena(model, grads=True)
    lengths = arena.ring_lengths(args.rings)
    starts = [sum(lengths[:i]) for i in range(len(lengths))]
    avg = None
    if regime != "none":
        tau = 0 if regime == "sync" else args.tau
        avg = AsyncAverager(arena.flat, starts=starts, lens=lengths, kappa=args.kappa, tau=tau,
                            graph=args.graph, sm_budget=sm_budget)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn(args.batch, args.width, device=dev, generator=g)
    y = torch.randint(0, 10, (args.batch,), device=dev, generator=g)
    loss_fn = torch.nn.CrossEntropyLoss()

    def step():
        arena.grad.zero_()
        loss = loss_fn(model(x), y)
        loss.backward()
        if avg is not None:
            avg.before_update()
        arena.flat.add_(arena.grad, alpha=-args.lr)  # one fused SGD update on the arena
        if avg is not None:
            avg.step()
        return loss

    for _ in range(args.kappa * 2):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        loss = step()
    b.record()
    if avg is not None:
        avg.flush()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    t = torch.tensor([ms])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = {"ms_per_step": round(float(t), 4), "loss": round(float(loss), 4),
           "cycles": avg.cycles if avg else 0, "params": arena.numel}
    if avg is not None:
        avg.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=4096)
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--rings", type=int, default=4)
    ap.add_argument("--kappa", type=int, default=8)
    ap.add_argument("--tau", type=int, default=4)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--graph", type=int, default=0)
    ap.add_argument("--sm-budgets", default="16,32,64,0", help="SM budgets of the async cycle (0 = all)")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    budgets = [int(b) for b in args.sm_budgets.split(",")]
    res = {"none": run("none", args, rank, dev), "sync": run("sync", args, rank, dev, 0)}
    for b in budgets:
        res[f"async_sm{b}"] = run("async", args, rank, dev, b)
    if rank == 0:
        base, sync = res["none"]["ms_per_step"], res["sync"]["ms_per_step"]
        cycle_cost = (sync - base) * args.kappa  # ms a cycle adds when it is on the critical path
        hidden = {b: round(1.0 - (res[f"async_sm{b}"]["ms_per_step"] - base) / max(sync - base, 1e-9), 3)
                  for b in budgets}
        print(json.dumps({
            "example": "train_async", "n_gpus": world, "params_per_cluster": res["none"]["params"],
            "kappa": args.kappa, "tau": args.tau, "rings": args.rings, "results": res,
            "cycle_ms_on_critical_path": round(cycle_cost, 4),
            "fraction_of_averaging_hidden_by_async": hidden,
        }), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
