"""Multi-process parity worker (one process per GPU), launched by
tests/test_dist_gpu.py through torchrun.  Every rank builds the same seeded
inputs for all C = world clusters, averages its own through DistRingGroup,
and checks its result bitwise against the oracle."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ring_oracle  # noqa: E402
from paper_2401_01728_b200.dist import DistRingGroup  # noqa: E402

# test harness knob: force the CB = 8 / 16 kernel buckets through the plan option
OPTIONS = {"min_cb": int(os.environ.get("RAVNEST_TEST_MIN_CB", "0"))}


def bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def stall_phase(rank, world, local):
    """Failure detection: only rank 0 launches a cycle; its kernel must give
    up after the timeout with a StallError naming a missing peer (no GPU
    hang).  Afterwards a fresh group must work normally."""
    from paper_2401_01728_b200.errors import StallError

    failures = 0
    lens = [4097, 333]
    total = sum(lens)
    for proto in ("pull", "push", "ll", "push+blend"):
        blend = proto.endswith("+blend")
        proto = proto.split("+")[0]
        x = torch.full((total,), float(rank), device=f"cuda:{local}")
        mean = torch.empty_like(x) if blend else None
        live = torch.zeros_like(x) if blend else None
        g = DistRingGroup(src=x, dst=mean, starts=[0, lens[0]], lens=lens, protocol=proto, timeout_s=0.5, live=live,
                          options=OPTIONS)
        if rank == 0:
            g.average()
            torch.cuda.synchronize()
            try:
                g.check()
                print(f"rank 0 {proto}: expected a StallError", flush=True)
                failures += 1
            except StallError as e:
                if "rank" not in str(e):
                    print(f"rank 0 {proto}: stall message lacks the rank: {e}", flush=True)
                    failures += 1
        dist.barrier()
        g.close()
        # a fresh group works
        x.fill_(float(rank))
        g = DistRingGroup(src=x, starts=[0, lens[0]], lens=lens, protocol=proto, options=OPTIONS)
        g.average()
        torch.cuda.synchronize()
        g.check()
        want = np.float32(sum(range(world)) / world)
        if not (x.cpu().numpy() == want).all():
            print(f"rank {rank} {proto}: fresh group after a stall is wrong", flush=True)
            failures += 1
        dist.barrier()
        g.close()
    return failures


def blend_phase(rank, world, local):
    """Delayed-update blend inside the cycle (DistRingGroup(live=...)):
    mean = ring mean of the snapshots, live <- mean + (live - snap), bitwise
    against the oracle, over three back-to-back cycles without host syncs
    (the fused push path has no depart barrier).  Guard bands on all three
    buffers."""
    failures = 0
    lens = [200003, 5, 77777, 2 * world + 1]
    total = sum(lens)
    starts = list(np.cumsum([0] + lens[:-1]))
    for proto in ("push", "pull", "ll"):
        for dt, lanes in ((torch.float32, 1), (torch.float32, 3), (torch.float64, 1)):
            if proto == "ll" and dt == torch.float64:
                continue
            npdt = np.float32 if dt == torch.float32 else np.float64
            snaps = [np.random.Generator(np.random.Philox(key=500 + m)).normal(0, 1, total).astype(npdt)
                     for m in range(world)]
            lives = [s + np.random.Generator(np.random.Philox(key=600 + m)).normal(0, 1e-3, total).astype(npdt)
                     for m, s in enumerate(snaps)]
            for m in range(world):  # some entries untouched since the snapshot: exactly the mean there
                lives[m][::7] = snaps[m][::7]
            bufs = [torch.full((total + 16,), -1234.5, dtype=dt, device=f"cuda:{local}") for _ in range(3)]
            x, mean, live = (b[8:8 + total] for b in bufs)
            x.copy_(torch.from_numpy(snaps[rank]))
            live.copy_(torch.from_numpy(lives[rank]))
            g = DistRingGroup(src=x, dst=mean, starts=starts, lens=lens, lanes=lanes, protocol=proto, live=live,
                              options=OPTIONS)
            streams = [torch.cuda.Stream() for _ in range(lanes)]
            for st in streams:
                st.wait_stream(torch.cuda.current_stream())
            if lanes == 1 and dt == torch.float32:
                # one cycle, then two CUDA-graph replays of a captured cycle
                # (device-side epochs, work counters and flags are graph-safe)
                g.average(streams)
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=streams[0]):
                    g.average(streams)
                dist.barrier()
                for _ in range(2):
                    graph.replay()
            else:
                for _ in range(3):
                    g.average(streams)
            torch.cuda.synchronize()
            g.check()
            want_mean = ring_oracle.ring_mean(starts, lens, snaps)[rank].astype(npdt)
            want_live = lives[rank]
            for _ in range(3):
                want_live = ring_oracle.blend(want_mean, want_live, snaps[rank])
            ok = np.array_equal(bits(mean.cpu().numpy()), bits(want_mean))
            ok = ok and np.array_equal(bits(live.cpu().numpy()), bits(want_live))
            ok = ok and np.array_equal(bits(x.cpu().numpy()), bits(snaps[rank]))  # snapshot untouched
            for b in bufs:
                h = b.cpu().numpy()
                ok = ok and (h[:8] == -1234.5).all() and (h[8 + total:] == -1234.5).all()
            if not ok:
                print(f"rank {rank} blend {proto} {dt} lanes={lanes}: mismatch", flush=True)
                failures += 1
            dist.barrier()
            g.close()
    return failures


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    os.environ.setdefault("RAVNEST_B200_TIMEOUT_S", "10")
    cases = []
    rng = np.random.Generator(np.random.Philox(key=77))
    for i in range(6):
        n_rings = int(rng.integers(1, 9))
        lens = [int(x) for x in rng.integers(0, 200000, n_rings)]
        lens[0] += world - 1
        cases.append(lens)
    cases.append([1, 0, 2, world + 1, 3 * world - 1])      # tiny and zero-length rings
    quick = os.environ.get("RAVNEST_DIST_QUICK") == "1"  # kernel-bucket / world-size variants
    if not quick:
        cases.append([26201088, 27168768, 27170304, 28942080])  # BERT-base rings
    failures = 0
    for ci, lens in enumerate(cases):
        total = sum(lens)
        starts = list(np.cumsum([0] + lens[:-1]))
        big = total > 10_000_000
        base = [("f64", torch.float32, 1, False, False)] if big else [
            ("f64", torch.float32, 1, False, False),
            ("native", torch.float32, 1, True, False),
            ("f64", torch.float64, 1, False, True),
            ("f64", torch.float32, len(lens), False, False),
            ("f64", torch.float32, 2 * len(lens) + 1, False, False),
            ("f64", torch.float32, 1, False, True),
        ]
        variants = [v + (proto,) for proto in ("pull", "push", "ll") for v in base
                    if not (proto == "ll" and v[1] == torch.float64)]
        for acc, dt, lanes, reverse_ids, src_ne_dst, proto in variants:
            npdt = np.float32 if dt == torch.float32 else np.float64
            xs = [np.random.Generator(np.random.Philox(key=1000 * ci + m)).normal(0, 1, total).astype(npdt)
                  for m in range(world)]
            cid = (world - 1 - rank) if reverse_ids else rank
            order = sorted(range(world), key=lambda r: (world - 1 - r) if reverse_ids else r)
            vals = [xs[r] for r in order]  # ascending cluster id
            want = ring_oracle.ring_mean(starts, lens, vals, acc=acc)[order.index(rank)].astype(npdt)
            off = 8 + (1 if src_ne_dst else 0)
            buf = torch.full((total + off + 8,), -1234.5, dtype=dt, device=f"cuda:{local}")  # guard bands
            x = buf[off:off + total]
            x.copy_(torch.from_numpy(xs[rank]))
            dbuf = torch.full((total + 16,), -1234.5, dtype=dt, device=f"cuda:{local}") if src_ne_dst else None
            dst = None
            if src_ne_dst:
                dst = dbuf[8:8 + total]
                dst.fill_(float("nan"))
            g = DistRingGroup(src=x, dst=dst, starts=starts, lens=lens, cluster_id=cid, acc=acc, lanes=lanes,
                              protocol=proto, options=OPTIONS)
            streams = [torch.cuda.Stream() for _ in range(lanes)]
            for s in streams:
                s.wait_stream(torch.cuda.current_stream())
            g.average(streams)
            torch.cuda.synchronize()
            g.check()
            hb = buf.cpu().numpy()
            guards_ok = (hb[:off] == -1234.5).all() and (hb[off + total:] == -1234.5).all()
            if dbuf is not None:
                hd = dbuf.cpu().numpy()
                guards_ok = guards_ok and (hd[:8] == -1234.5).all() and (hd[8 + total:] == -1234.5).all()
            if not guards_ok:
                print(f"rank {rank} case {ci} {proto}: write outside the member vector", flush=True)
                failures += 1
            got = (dst if dst is not None else x).cpu().numpy()
            if not np.array_equal(bits(got), bits(want)):
                bad = int(np.sum(bits(got) != bits(want)))
                print(f"rank {rank} case {ci} {proto} {acc} {dt} lanes={lanes} rev={reverse_ids}: {bad} mismatches",
                      flush=True)
                failures += 1
            if not big and not src_ne_dst and lanes == 1:
                # host-buffer path, twice in a row (epochs advance consistently)
                h_in = torch.from_numpy(xs[rank]).pin_memory()
                h_out = torch.empty_like(h_in).pin_memory()
                for _ in range(2):
                    g.average_host(h_in, h_out)
                    torch.cuda.synchronize()
                g.check()
                if not np.array_equal(bits(h_out.numpy()), bits(want)):
                    print(f"rank {rank} case {ci} {proto} host path mismatch", flush=True)
                    failures += 1
            if not big and not src_ne_dst and lanes == 1 and acc == "f64" and dt == torch.float32:
                # three cycles back to back, no host sync in between (epoch handling)
                x.copy_(torch.from_numpy(xs[rank]))
                torch.cuda.synchronize()
                dist.barrier()
                for _ in range(3):
                    g.average()
                torch.cuda.synchronize()
                g.check()
                cur = vals
                for _ in range(3):
                    cur = [v.astype(npdt) for v in ring_oracle.ring_mean(starts, lens, cur, acc=acc)]
                if not np.array_equal(bits(x.cpu().numpy()), bits(cur[order.index(rank)])):
                    print(f"rank {rank} case {ci} {proto} back-to-back mismatch", flush=True)
                    failures += 1
            dist.barrier()
            g.close()
    failures += blend_phase(rank, world, local)
    if not quick:
        failures += stall_phase(rank, world, local)
    t = torch.tensor([failures])
    dist.all_reduce(t)
    if rank == 0:
        print(f"DIST {'OK' if int(t) == 0 else 'FAIL'} world={world} cases={len(cases)} failures={int(t)}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(t) == 0 else 1)


if __name__ == "__main__":
    main()
