"""Fixed cost of one averaging cycle: back-to-back cycles on tiny vectors
(torchrun, one process per GPU), per transport, plus torch's own empty-kernel
launch rate for scale.  Prints one JSON line (rank 0)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_01728_b200.dist import DistRingGroup  # noqa: E402


def timed(fn, n):
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) * 1e3 / n])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(float(t), 2)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    out = {"n_gpus": dist.get_world_size()}
    z = torch.zeros(1, device="cuda")
    out["torch_add_us"] = timed(lambda: z.add_(1.0), 2000)
    for n in (1024, 1 << 18):
        for proto in ("pull", "push", "ll"):
            x = torch.randn(n, device="cuda")
            g = DistRingGroup(src=x, starts=[0], lens=[n], protocol=proto)
            for _ in range(10):
                g.average()
            out[f"{proto}_{n * 4 // 1024}KiB_us"] = timed(g.average, 1000)
            g.check()
            g.close()
    if dist.get_rank() == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
