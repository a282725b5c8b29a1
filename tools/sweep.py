"""Config 5 of BASELINE.json: ring-count x shard-size sweep at N GPUs against
the NCCL comparison path.  Run under torchrun (one process per GPU):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/sweep.py [--out F]

For each (R rings of `shard` MiB each, equal rings) it times one averaging
cycle of our kernel (pull and push protocols, replayed from a CUDA graph of
`--graph-steps` cycles so launch latency is amortised as a training loop
would), and NCCL ncclAllReduce(avg) per ring, all with CUDA events, max over
ranks.  Prints one JSON line per configuration (rank 0).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_01728_b200.dist import DistRingGroup  # noqa: E402
from tools.nccl_compare import NcclRings  # noqa: E402


def busbw(total, c, sec):
    return total * 4 / sec * 2 * (c - 1) / c / 1e9


def timed(fn, steps, stream):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", default="1,4,16,64,256,1024")
    ap.add_argument("--rings", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--graph-steps", type=int, default=10)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device(f"cuda:{local}"))
    rank, world = dist.get_rank(), dist.get_world_size()
    stream = torch.cuda.Stream()
    lines = []
    for mib in [int(x) for x in args.shards.split(",")]:
        for r in [int(x) for x in args.rings.split(",")]:
            n = mib * (1 << 20) // 4
            lens = [n] * r
            starts = [i * n for i in range(r)]
            total = n * r
            x = torch.randn(total, device="cuda") * 0.02
            row = {"n_gpus": world, "shard_mib": mib, "rings": r, "bytes_per_cluster": total * 4}
            with torch.cuda.stream(stream):
                protos = ("pull", "push", "ll") if total * 4 <= (16 << 20) else ("pull", "push")
                for proto in protos:
                    g = DistRingGroup(src=x, starts=starts, lens=lens, protocol=proto)
                    for _ in range(3):
                        g.average([stream])
                    torch.cuda.synchronize()
                    ms = timed(lambda: g.average([stream]), args.steps, stream)
                    # CUDA graph of graph_steps cycles (device-side epochs make it replayable)
                    graph = torch.cuda.CUDAGraph()
                    dist.barrier()
                    with torch.cuda.graph(graph, stream=stream):
                        for _ in range(args.graph_steps):
                            g.average([stream])
                    torch.cuda.synchronize()
                    dist.barrier()
                    gms = timed(graph.replay, max(2, args.steps // args.graph_steps), stream) / args.graph_steps
                    g.check()
                    # device-side phase trace of a few isolated cycles (max over ranks)
                    g.plan.set_trace(True)
                    acc = None
                    for _ in range(5):
                        dist.barrier()
                        g.average([stream])
                        torch.cuda.synchronize()
                        tr = g.plan.read_trace(0)
                        v = torch.tensor([tr["ready_us"], tr["data_us"], tr["depart_us"], tr["total_us"]],
                                         dtype=torch.float64)
                        acc = v if acc is None else acc + v
                    g.plan.set_trace(False)
                    acc /= 5
                    dist.all_reduce(acc, op=dist.ReduceOp.MAX)
                    row[proto] = {"ms": round(ms, 5), "bus_gbps": round(busbw(total, world, ms * 1e-3), 2),
                                  "graph_ms": round(gms, 5),
                                  "graph_bus_gbps": round(busbw(total, world, gms * 1e-3), 2),
                                  "phases_us": {k: round(float(x), 2) for k, x in
                                                zip(("ready", "data", "depart", "total"), acc)}}
                    del graph
                    g.close()
                rep = NcclRings(x, lens).report(args.steps)
                row["nccl"] = {"ms": rep["ms_per_step"], "bus_gbps": rep["bus_gbps_per_gpu"], "best": rep["best"],
                               "sequential_ms": rep["sequential"]["ms_per_step"],
                               "coalesced_ms": rep["coalesced"]["ms_per_step"]}
            if rank == 0:
                print(json.dumps(row), flush=True)
                lines.append(row)
            del x
            torch.cuda.empty_cache()
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            for row in lines:
                f.write(json.dumps(row) + "\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
