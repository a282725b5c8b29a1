"""Pinned host<->device copy rates with 1/2/4 concurrent streams, per
direction and both directions at once (the e2e path's ceiling)."""
import json
import time

import torch

n = 512 << 20  # 512 MiB per stream
res = {}
for ns in (1, 2, 4):
    hs = [torch.empty(n // 4, dtype=torch.float32).pin_memory() for _ in range(ns)]
    ds = [torch.empty(n // 4, dtype=torch.float32, device="cuda") for _ in range(ns)]
    hs2 = [torch.empty(n // 4, dtype=torch.float32).pin_memory() for _ in range(ns)]
    ds2 = [torch.empty(n // 4, dtype=torch.float32, device="cuda") for _ in range(ns)]
    sts = [torch.cuda.Stream() for _ in range(2 * ns)]
    for mode in ("h2d", "d2h", "both"):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(ns):
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(sts[i]):
                        ds[i].copy_(hs[i], non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(sts[ns + i]):
                        hs2[i].copy_(ds2[i], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        res[f"{mode}_{ns}streams_GBps_per_direction"] = round(ns * n / dt / 1e9, 1)
print(json.dumps(res))
