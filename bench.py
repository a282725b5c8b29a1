#!/usr/bin/env python
"""Benchmark of the B200 multi-ring parameter average (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload bert|resnet50|gpt2] [--acc f64|native] [--lanes 1|R]

Metric (BASELINE.json): param-averaging bus GB/s and ms/round.  A step is
one averaging cycle over the whole parameter set of every cluster (all
rings).  bus GB/s follows the NCCL convention per GPU,
busbw = S/t * 2(C-1)/C with S the fp32 bytes of one cluster's parameters;
``value`` is the whole-job aggregate, N_gpus * busbw.

N = 1 : C = 8 clusters co-resident on cuda:0 (one kernel, HBM-bound).
N > 1 : torchrun, one process per GPU, one cluster per GPU (C = N),
        DistRingGroup: one kernel per rank, peer loads/stores over NVLink.

``--impl reference`` times the CPU oracle port (oracle/ring_oracle.c, all
host threads) on a bounded sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# per-lane streams of one cycle must not share hardware queues (set before CUDA starts)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

# tensor-boundary ring lengths (torchvision / transformers shapes)
WORKLOADS = {
    "resnet50": [6308928, 6172672, 5511168, 7564264],
    "bert": [26201088, 27168768, 27170304, 28942080],
    "gpt2": [51463168, 43039744, 41987072, 41986048, 41989120, 41987072, 41986048, 50384896],
}
WORKLOAD_NAMES = {
    "resnet50": "ResNet-50 parameter set (25,557,032 fp32), 4 rings",
    "bert": "BERT-base parameter set (109,482,240 fp32), 4 submodel rings",
    "gpt2": "GPT-2 medium parameter set (354,823,168 fp32), 8 rings",
}
METRIC = "param-averaging bus GB/s and ms/round at 1/2/4/8 B200 vs NVLink roofline"
NVLINK_PEAK_GBS = 900.0  # NVLink 5 per direction per GPU: the roofline north_star / BASELINE.md name
NVLINK_PEER_COPY_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md), secondary
# user-data ceilings of each transport's traffic pattern: ~840 GB/s raw per
# direction / (1 + protocol overhead), ncu-measured (profiles/r01/ncu_nvlink.md)
PATTERN_CEILING_GBS = {"push": 706.0, "pull": 656.0}
SEED = 20241018
SIGMA = 0.02


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(workload: str, c: int, n_gpus: int, acc: str):
    """Per-launch DRAM bytes of the dominant kernel from a committed ncu
    capture of the same configuration (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            entry = json.load(f).get(f"{workload}/c{c}/n{n_gpus}/{acc}")
        return entry["bytes"] if entry else None
    except Exception:
        return None


def bind_to_gpu_numa(device: int) -> str:
    """Pin this process to the CPUs local to `device`'s PCIe root (sysfs
    local_cpulist) so pinned host buffers for the e2e leg are allocated on
    the GPU's own NUMA node.  Returns the cpulist used ('' if unknown)."""
    import torch

    try:
        props = torch.cuda.get_device_properties(device)
        bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        os.sched_setaffinity(0, cpus)
        return spec
    except Exception:
        return ""


def ring_starts(lens):
    out, s = [], 0
    for n in lens:
        out.append(s)
        s += n
    return out


def busbw(total_params: int, c: int, seconds: float) -> float:
    return total_params * 4 / seconds * 2 * (c - 1) / c / 1e9


# ---------------------------------------------------------------------------
# CPU legs (oracle port; only bench.py's cpu_baseline / --impl reference use it)


class CpuSample:
    """A bounded sample of the workload for the CPU legs: the first `frac` of
    every ring (same C, same ring structure), fp32 N(0, 0.02)."""

    def __init__(self, lens, c: int, budget_params: int):
        import numpy as np

        total = sum(lens)
        frac = min(1.0, budget_params / total)
        self.lens = [max(1, int(n * frac)) for n in lens]
        self.total = sum(self.lens)
        self.c = c
        rng = np.random.Generator(np.random.Philox(key=SEED))
        self.xs = [rng.standard_normal(self.total, dtype=np.float32) * np.float32(SIGMA) for _ in range(c)]
        self.outs = [np.empty_like(x) for x in self.xs]

    def run_port(self) -> float:
        """One cycle of the reference's own algorithm, ported faithfully: the
        round-by-round ring of apply_ring_mean (multiring.py:302-333) in numpy
        float64 with its copy-in and payload copies (oracle/ring_oracle.py
        ring_mean_rounds).  numpy ufuncs are single-threaded, like the
        reference.  Returns seconds."""
        import numpy as np

        from oracle import ring_oracle

        t0 = time.perf_counter()
        ring_oracle.ring_mean_rounds(ring_starts(self.lens), self.lens, self.xs, dtype=np.float64)
        return time.perf_counter() - t0

    def run_threaded(self, threads: int) -> float:
        """One cycle of the closed-form C oracle on `threads` host threads
        (f32 in, f64 fold, f32 out -- the product contract); seconds."""
        from oracle import c_oracle

        t0 = time.perf_counter()
        c_oracle.ring_mean_into(c_oracle.MODE_F32_ACC64, ring_starts(self.lens), self.lens, self.xs, None,
                                self.outs, threads=threads)
        return time.perf_counter() - t0


def cpu_legs(lens, c: int, port_params: int, threaded_params: int, threads: int):
    """(reference-port record, threaded-oracle record) for cpu_baseline."""
    port = CpuSample(lens, c, port_params)
    port.run_port()
    tp = min(port.run_port() for _ in range(2))
    thr = CpuSample(lens, c, threaded_params)
    thr.run_threaded(threads)
    tt = min(thr.run_threaded(threads) for _ in range(3))
    total = sum(lens)
    return (
        {"value": round(busbw(port.total, c, tp), 4), "unit": "GB/s", "cores": 1, "kind": "port",
         "sample": f"first {port.total} of {total} params per cluster (every ring scaled), C={c}; "
                   f"reference algorithm ported round by round (numpy fp64, single-threaded like the "
                   f"reference), best of 2, {cpu_model()}"},
        {"value": round(busbw(thr.total, c, tt), 3), "unit": "GB/s", "cores": threads, "kind": "oracle-c",
         "sample": f"first {thr.total} of {total} params per cluster, C={c}; closed-form C oracle, "
                   f"{threads} threads, best of 3"},
    )


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def import_reference():
    """The UNMODIFIED reference package: baseline/_ref (the offline install,
    travels to the GPU box), else the read-only tree of the dev container.
    Returns (ravnest module, where) or (None, why)."""
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "ravnest")):
            sys.dont_write_bytecode = True  # /root/reference is read-only
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                import ravnest
                import ravnest.multiring  # noqa: F401
            except Exception as e:  # pragma: no cover - broken install
                return None, f"import from {path} failed: {e!r}"
            return ravnest, path
    return None, "baseline/_ref not installed (see DESIGN.md, reference install)"


def host_inputs(total: int, c: int):
    """Per-cluster fp32 N(0, 0.02) vectors, Philox-seeded."""
    import numpy as np

    return [np.random.Generator(np.random.Philox(key=SEED * 1000 + m)).standard_normal(total, dtype=np.float32)
            * np.float32(SIGMA) for m in range(c)]


def mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


def run_reference(args, n_gpus: int, rank: int):
    """--impl reference: the reference's own CPU implementation of the path --
    the unmodified ``ravnest.multiring.apply_ring_mean`` (multiring.py:302-333)
    imported from baseline/_ref -- on the FULL workload of our arm (same rings,
    same C, fp32 N(0, 0.02) inputs that it widens to float64 itself), rank 0
    only.  One full-size cycle takes seconds, so the step count is capped to
    keep the arm within a few minutes (``steps`` reports what was timed).
    Without the install (or the RAM for a full cycle) it falls back to the
    faithful port on a bounded sample and says so."""
    if rank != 0:
        return
    import numpy as np

    lens = WORKLOADS[args.workload]
    c = args.clusters or (8 if n_gpus == 1 else n_gpus)
    total = sum(lens)
    starts = ring_starts(lens)
    ravnest, where = import_reference()
    need = total * c * (4 + 3 * 8)  # fp32 inputs + the reference's float64 working set
    full = ravnest is not None and args.ref_sample_params <= 0 and (mem_available() == 0 or need < 0.8 * mem_available())
    base = {
        "impl": "reference", "metric": METRIC, "unit": "GB/s", "n_gpus": n_gpus,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (reference arithmetic)",
        "data": "synthetic N(0,0.02) fp32 per cluster (Philox seeded), widened to fp64 by the reference",
        "config": {"workload": WORKLOAD_NAMES[args.workload], "clusters": c, "rings": len(lens),
                   "parallelism": "1 host thread (numpy ufuncs, as the reference)"},
    }
    if full:
        mr = ravnest.multiring
        sched = mr.build_ring_schedule({m: [mr.ParamRange(st, n) for st, n in zip(starts, lens)] for m in range(c)})
        xs = host_inputs(total, c)
        vals = {m: xs[m] for m in range(c)}
        t0 = time.perf_counter()
        out = mr.apply_ring_mean(sched, vals)  # warm-up (and the step-count estimate)
        first = time.perf_counter() - t0
        del out
        warm = 1
        for _ in range(min(args.warmup, 2) - 1):
            if first * (warm + 1) > args.ref_budget_s / 2:
                break
            mr.apply_ring_mean(sched, vals)
            warm += 1
        steps = max(1, min(args.steps, int(args.ref_budget_s // max(first, 1e-3))))
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            out = mr.apply_ring_mean(sched, vals)
            times.append(time.perf_counter() - t0)
            del out
        t = statistics.median(times)
        value = busbw(total, c, t) * n_gpus
        sample = (f"FULL workload: {c} clusters x {total} params, unmodified ravnest.multiring.apply_ring_mean "
                  f"from {os.path.relpath(where, ROOT) if where.startswith(ROOT) else where}; "
                  f"{warm} warm-up + {steps} timed cycle(s) of the {args.steps} requested (one cycle takes "
                  f"{first:.1f} s; capped at ~{args.ref_budget_s:.0f} s), median; {cpu_model()}")
        line = dict(base, value=round(value, 4), steps=steps, warmup=warm, steps_requested=args.steps,
                    ms_per_step=round(t * 1e3, 3), ms_per_round=round(t * 1e3 / (2 * (c - 1)), 3),
                    ms_per_step_min=round(min(times) * 1e3, 3))
        line["cpu_baseline"] = {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
                                "sample": sample}
    else:
        why = where if ravnest is None else ("--ref-sample-params set" if args.ref_sample_params > 0 else
                                             f"full cycle needs ~{need / 1e9:.0f} GB of host RAM")
        smp = CpuSample(lens, c, args.ref_sample_params if args.ref_sample_params > 0 else 2_000_000)
        for _ in range(args.warmup):
            smp.run_port()
        times = [smp.run_port() for _ in range(args.steps)]
        t = statistics.median(times)
        value = busbw(smp.total, c, t) * n_gpus
        line = dict(base, value=round(value, 4), steps=args.steps, warmup=args.warmup,
                    ms_per_step=round(t * 1e3 * total / smp.total, 3), ms_per_step_extrapolated=True)
        line["cpu_baseline"] = {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "port",
                                "sample": f"first {smp.total} of {total} params per cluster (every ring scaled), "
                                          f"C={c}, round-by-round numpy port of multiring.apply_ring_mean "
                                          f"(oracle/ring_oracle.ring_mean_rounds); not the full workload: {why}; "
                                          f"{cpu_model()}"}
    line["e2e"] = {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU legs


def synth(total: int, key: int, device):
    import torch

    g = torch.Generator(device=device).manual_seed(SEED * 1000 + key)
    return torch.randn(total, device=device, generator=g, dtype=torch.float32) * SIGMA


def warm_under_load(step, warmup: int, seconds: float = 0.6, lockstep: bool = False):
    """W untimed warm-up steps, extended until ~`seconds` of load so the clock
    sampler (started just before) has samples under load.  With `lockstep`
    (multi-rank) the step count is agreed across ranks: each rank runs the
    same number of collective cycles."""
    import torch

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    per = max(time.perf_counter() - t0, 1e-5)
    extra = int(min(5000, seconds / per))
    if lockstep:
        import torch.distributed as dist

        t = torch.tensor([extra])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        extra = int(t)
    for _ in range(extra):
        step()
    torch.cuda.synchronize()


def stale_live(snap, key: int, tau: int, eta: float = 1e-3):
    """live = snap - eta * sum_{j=1..tau} g_j, g_j ~ N(0,1) seeded per (cluster, j)
    (the tau updates that landed after the snapshot)."""
    import torch

    live = snap.clone()
    for j in range(1, tau + 1):
        g = torch.Generator(device=snap.device).manual_seed(SEED * 7919 + key * 31 + j)
        live.sub_(torch.randn(snap.numel(), device=snap.device, generator=g), alpha=eta)
    return live


L2_BYTES = 126 * 1024 * 1024  # B200 L2


class L2Flush:
    """Between timed steps, overwrite a buffer twice the L2 size so that no
    step starts with its inputs cached.  Used when the per-GPU input set does
    not exceed L2 by itself (ResNet-50 at one cluster per GPU); the flush runs
    outside each step's events."""

    def __init__(self, device):
        import torch

        self.buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=device)
        self.n = 0

    def __call__(self, stream):
        import torch

        with torch.cuda.stream(stream):
            self.n += 1
            self.buf.fill_(float(self.n))


def l2_policy(mode: str, input_bytes: int, device):
    """(flusher or None, config text) for the per-GPU input bytes of a step."""
    big = input_bytes > 2 * L2_BYTES
    if mode == "off" or (mode == "auto" and big):
        return None, f"inputs larger than L2 ({input_bytes / 1e6:.0f} MB per GPU vs {L2_BYTES / 1e6:.0f} MB L2)"
    return L2Flush(device), (f"L2 flushed before every timed step ({2 * L2_BYTES / 1e6:.0f} MB write, outside the "
                             f"step's events; inputs {input_bytes / 1e6:.0f} MB per GPU); ms_per_step = mean of the "
                             f"per-step event intervals")


def launches_per_step(args, grp, total: int) -> int:
    """Our kernels per rank per step at N > 1: one cycle kernel per lane,
    plus the blend when it is not fused into the push kernel (rv_blend: one
    vector launch, one more for a tail that is not a whole 16-byte vector)."""
    n = args.lanes
    if args.blend:
        per_blend = 1 + (1 if total % 4 else 0)
        if not args.fused_blend:
            n += per_blend
        elif grp.protocol != "push":
            n += args.lanes * per_blend
    return n


def time_steps(fn, stream, steps: int, flush=None):
    """Per-step CUDA events on `stream`: (start, after-averaging, end).  The
    first interval is the averaging launch(es) alone -- the roofline basis.
    With `flush`, the L2 flush runs before each step's start event."""
    import torch

    evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(steps)]
    for a, m, b in evs:
        if flush is not None:
            flush(stream)
        a.record(stream)
        fn(m)
        b.record(stream)
    return evs


def run_single(args):
    """N = 1: C clusters co-resident on cuda:0."""
    import torch

    from paper_2401_01728_b200.blend import blend_
    from paper_2401_01728_b200.plan import LocalRingGroup

    lens = WORKLOADS[args.workload]
    c = args.clusters or 8
    total = sum(lens)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    xs = [synth(total, m, dev) for m in range(c)]
    lives = means = None
    if args.blend:
        lives = [stale_live(x, m, args.tau) for m, x in enumerate(xs)]
        means = [torch.empty_like(x) for x in xs]
    g = LocalRingGroup(ring_starts(lens), lens, total, [0] * c, torch.float32, acc=args.acc, lanes=args.lanes)
    g.bind_tensors(xs, means)
    in_cycle_blend = bool(args.blend and args.fused_blend)
    if in_cycle_blend:
        g.bind_live(lives)  # fused into the co-resident TMA kernel
    stream = torch.cuda.current_stream()
    lane_streams = [torch.cuda.Stream() for _ in range(args.lanes)] if args.lanes > 1 else None

    def step(mid=None):
        if lane_streams:
            for s in lane_streams:
                s.wait_stream(stream)
            g.run({0: lane_streams})
            for s in lane_streams:
                stream.wait_stream(s)
        else:
            g.run({0: [stream]})
        if mid is not None:
            mid.record(stream)
        if args.blend and not in_cycle_blend:
            for m in range(c):
                blend_(lives[m], xs[m], means[m], stream)

    clocks = ClockSampler(0)
    clocks.start()
    warm_under_load(step, args.warmup)
    g.check()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    flush, l2_text = l2_policy(args.l2_flush, c * total * 4, dev)
    t_start.record(stream)
    evs = time_steps(step, stream, args.steps, flush)
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    g.check()
    total_ms = t_start.elapsed_time(t_end)
    kernel_ms = statistics.mean(a.elapsed_time(m) for a, m, _ in evs)
    per_step = [a.elapsed_time(b) for a, _, b in evs]
    ms = total_ms / args.steps if flush is None else statistics.mean(per_step)
    step_median, step_min = statistics.median(per_step), min(per_step)

    # e2e: host (pinned) buffers -> device -> average -> host, via the C ABI
    hsrc = [x.cpu().pin_memory() for x in xs]
    hdst = [torch.empty_like(h).pin_memory() for h in hsrc]
    e2e_streams = [torch.cuda.Stream() for _ in range(args.e2e_lanes)]
    plan_e2e = LocalRingGroup(ring_starts(lens), lens, total, [0] * c, torch.float32, acc=args.acc,
                              lanes=args.e2e_lanes)
    plan_e2e.bind_tensors(xs)
    pe = plan_e2e.plans[0]

    def e2e_step():
        pe.run_host([h.data_ptr() for h in hsrc], [h.data_ptr() for h in hdst], e2e_streams)
        for s in e2e_streams:
            stream.wait_stream(s)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e_steps = max(3, min(args.steps, 10))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    for s in e2e_streams:
        s.wait_stream(stream)
    a.record(stream)
    for _ in range(e_steps):
        for s in e2e_streams:
            s.wait_stream(stream)
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    plan_e2e.check()
    e2e_ms = a.elapsed_time(b) / e_steps

    seam = optional_leg("e2e_seam", lambda: e2e_seam(lens, c, xs, args.e2e_seam_steps)) if args.e2e_seam else None

    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # the fused blend also reads and writes every live vector
    hbm_bytes = (4 if in_cycle_blend else 2) * c * total * 4
    achieved = hbm_bytes / (kernel_ms * 1e-3) / 1e9
    bw = busbw(total, c, ms * 1e-3)

    # CPU baselines on bounded samples: the reference algorithm (faithful
    # port, 1 thread) and the closed-form C oracle on every host thread
    threads = host_threads()
    cpu_port, cpu_threaded = cpu_legs(lens, c, args.cpu_port_params, args.cpu_sample_params, threads)

    line = {
        "metric": METRIC, "value": round(bw, 3), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "ms_per_round": round(ms / (2 * (c - 1)), 5),
        "avg_kernel_ms": round(kernel_ms, 4),
        "ms_per_step_median": round(step_median, 4), "ms_per_step_min": round(step_min, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" + (" (f64 fold)" if args.acc == "f64" else " (f32 fold)"),
        "data": "synthetic N(0,0.02) fp32 per cluster, torch Philox seeded",
        "config": {"workload": WORKLOAD_NAMES[args.workload], "clusters": c, "rings": len(lens),
                   "placement": "co-resident on cuda:0", "lanes": args.lanes, "parallelism": "replicas only",
                   "blend": (f"snapshot average + delayed-update blend, tau={args.tau}, "
                             + ("fused into the cycle kernel" if in_cycle_blend else "separate launches"))
                   if args.blend else None,
                   "l2": l2_text},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4),
                     "traffic": ncu_traffic(args.workload, c, 1, args.acc) if not args.blend else None,
                     "basis": (f"4*C*S = {hbm_bytes} B per launch (read C snapshots and C live vectors, "
                               f"write C means and C live vectors)" if in_cycle_blend else
                               f"2*C*S = {hbm_bytes} B per launch (read C, write C vectors)"),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"},
        "cpu_baseline": cpu_port,
        "cpu_threaded": cpu_threaded,
        "e2e": {"value": round(busbw(total, c, e2e_ms * 1e-3), 3), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": c * total * 4, "d2h_bytes_per_step": c * total * 4,
                "path": f"rv_allreduce_mean_host (pinned host fp32, {args.e2e_lanes} pipelined lanes)"},
        "e2e_seam": seam,
        "gpu_launches": args.steps * (args.lanes + (0 if in_cycle_blend or not args.blend
                                                     else c * (1 + (1 if total % 4 else 0)))),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def plan_options(args) -> dict:
    """rv_plan_set_option values from the command line (kernel-bucket and
    push-layout experiments; defaults are the library's)."""
    opts = {}
    if args.min_cb:
        opts["min_cb"] = args.min_cb
    if args.push_items:
        opts["push_items"] = args.push_items
    if args.blend_lag >= 0:
        opts["blend_lag"] = args.blend_lag
    return opts


def e2e_seam(lens, c: int, xs, steps: int):
    """The reference user's call, end to end: after ``plugin.install`` on the
    unmodified reference, ``ravnest.multiring.apply_ring_mean(schedule,
    {cid: float64 numpy})`` (multiring.py:302-333) -- float64 copy-in into
    pinned staging, H2D, the float64 kernel, D2H, new float64 arrays out,
    pipelined by lane.  Host wall time per call (the call is synchronous)."""
    import numpy as np

    ravnest, where = import_reference()
    if ravnest is None:
        return {"unavailable": where}
    from paper_2401_01728_b200 import plugin

    mr = ravnest.multiring
    total = sum(lens)
    starts = ring_starts(lens)
    sched = mr.build_ring_schedule({m: [mr.ParamRange(st, n) for st, n in zip(starts, lens)] for m in range(c)})
    vals = {m: xs[m].cpu().numpy().astype(np.float64) for m in range(c)}
    plugin.install(ravnest)
    try:
        out = mr.apply_ring_mean(sched, vals)  # warm-up: plan, device buffers, pinned staging
        ok = bool(np.array_equal(out[0][:4096], out[c - 1][:4096]))
        del out
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            out = mr.apply_ring_mean(sched, vals)
            times.append(time.perf_counter() - t0)
            del out
    finally:
        plugin.uninstall(ravnest)
    t = statistics.median(times)
    return {"value": round(busbw(total, c, t), 3), "unit": "GB/s", "ms_per_step": round(t * 1e3, 2),
            "ms_per_step_min": round(min(times) * 1e3, 2), "steps": steps,
            "h2d_bytes_per_step": c * total * 8, "d2h_bytes_per_step": c * total * 8, "members_agree": ok,
            "path": "ravnest.multiring.apply_ring_mean after plugin.install (unmodified reference, numpy float64 "
                    "in/out, float64 kernel bitwise the reference)"}


def run_multi(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_2401_01728_b200.blend import blend_
    from paper_2401_01728_b200.dist import DistRingGroup

    lens = WORKLOADS[args.workload]
    total = sum(lens)
    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    x = synth(total, rank, dev)
    live = mean = None
    if args.blend:
        # config 4: average a snapshot x into `mean`, then blend the tau
        # pending updates of `live` onto it (live <- mean + (live - snap))
        live = stale_live(x, rank, args.tau)
        mean = torch.empty_like(x)
    # the blend rides in the cycle (rv_plan_bind_live): fused into the push
    # kernel, or launched per lane by the C ABI for the other transports
    in_cycle_blend = bool(args.blend and args.fused_blend)
    grp = DistRingGroup(src=x, dst=mean, starts=ring_starts(lens), lens=lens, acc=args.acc, lanes=args.lanes,
                        protocol=args.protocol, max_blocks=args.max_blocks, live=live if in_cycle_blend else None,
                        options=plan_options(args))
    stream = torch.cuda.current_stream()
    lane_streams = [torch.cuda.Stream() for _ in range(args.lanes)] if args.lanes > 1 else None

    def step(mid=None):
        if lane_streams:
            for s in lane_streams:
                s.wait_stream(stream)
            grp.average(lane_streams)
            for s in lane_streams:
                stream.wait_stream(s)
        else:
            grp.average([stream])
        if mid is not None:
            mid.record(stream)
        if args.blend and not in_cycle_blend:
            blend_(live, x, mean, stream)

    clocks = ClockSampler(local_rank) if rank == 0 else None
    if clocks:
        clocks.start()
    warm_under_load(step, args.warmup, lockstep=True)
    grp.check()
    dist.barrier()
    torch.cuda.synchronize()
    flush, l2_text = l2_policy(args.l2_flush, total * 4 * (3 if args.blend else 1), dev)
    # every timed step starts from a rank-aligned point: a one-element NCCL
    # all-reduce on the step's stream (it completes on all ranks together)
    # right before the step's start event, after the optional L2 flush.  A
    # step is then timed per rank from that point, and each step's duration
    # is the max over ranks.
    align = torch.zeros(1, device=dev)
    evs = []
    for _ in range(args.steps):
        if flush is not None:
            flush(stream)
        dist.all_reduce(align)
        e = tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
        e[0].record(stream)
        step(e[1])
        e[2].record(stream)
        evs.append(e)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop() if clocks else None
    grp.check()
    per = torch.tensor([[ea.elapsed_time(eb) for ea, _, eb in evs], [ea.elapsed_time(em) for ea, em, _ in evs]],
                       dtype=torch.float64)
    dist.all_reduce(per, op=dist.ReduceOp.MAX)  # per step, max over ranks (gloo, outside the timed region)
    per_step, per_kernel = per[0].tolist(), per[1].tolist()
    ms, kernel_ms = statistics.mean(per_step), statistics.mean(per_kernel)
    step_median, step_min = statistics.median(per_step), min(per_step)
    kernel_median = statistics.median(per_kernel)

    # e2e through the host-buffer C ABI: pinned host -> GPU -> average -> host
    numa_cpus = bind_to_gpu_numa(local_rank) if args.numa_bind else ""
    hsrc = x.cpu().pin_memory()
    hdst = torch.empty_like(hsrc).pin_memory()
    grp_e2e = DistRingGroup(src=x, starts=ring_starts(lens), lens=lens, acc=args.acc, lanes=args.e2e_lanes,
                            protocol=args.protocol, options=plan_options(args))
    e2e_streams = [torch.cuda.Stream() for _ in range(args.e2e_lanes)]

    def e2e_step():
        for s in e2e_streams:
            s.wait_stream(stream)
        grp_e2e.average_host(hsrc, hdst, e2e_streams)
        for s in e2e_streams:
            stream.wait_stream(s)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    e_steps = max(3, min(args.steps, 10))
    ea = torch.cuda.Event(enable_timing=True)
    eb = torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(e_steps):
        e2e_step()
    eb.record(stream)
    torch.cuda.synchronize()
    grp_e2e.check()
    te = torch.tensor([ea.elapsed_time(eb) / e_steps], dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te[0])

    phases = None
    if args.trace:
        phases = optional_leg("trace", lambda: trace_phases(grp, step))
    nccl = None
    if args.nccl:
        nccl = optional_leg("nccl_compare", lambda: nccl_compare(lens, x, world, min(args.steps, 20), flush))

    if rank == 0:
        c = world
        bw = busbw(total, c, ms * 1e-3)
        alg_bytes = 2 * (c - 1) / c * total * 4
        achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": round(bw * world, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "ms_per_round": round(ms / (2 * (c - 1)), 5),
            "avg_kernel_ms": round(kernel_ms, 4),
            "ms_per_step_median": round(step_median, 4), "ms_per_step_min": round(step_min, 4),
            "bus_gbps_per_gpu": round(bw, 3), "bus_gbps_per_gpu_median": round(busbw(total, c, step_median * 1e-3), 3),
            "timing": "each step starts after a rank-aligning NCCL all-reduce; per-step max over ranks, "
                      "mean (ms_per_step) and median reported",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" + (" (f64 fold)" if args.acc == "f64" else " (f32 fold)"),
            "data": "synthetic N(0,0.02) fp32 per cluster, torch Philox seeded",
            "config": {"workload": WORKLOAD_NAMES[args.workload], "clusters": c, "rings": len(lens),
                       "placement": "one cluster per GPU", "lanes": args.lanes, "protocol": grp.protocol,
                       "plan_options": plan_options(args) or None,
                       "max_blocks": args.max_blocks or None,
                       "blend": (f"snapshot average + delayed-update blend, tau={args.tau}, "
                                 + ("in the cycle (push: fused per unit)" if in_cycle_blend else "separate launch")) if args.blend else None,
                       "parallelism": f"multi-ring all-reduce over {world} GPUs (NVLink P2P)",
                       "l2": l2_text},
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK_GBS,
                         "unit": "GB/s", "frac": round(achieved / NVLINK_PEAK_GBS, 4),
                         "achieved_median": round(alg_bytes / (kernel_median * 1e-3) / 1e9, 1),
                         "traffic": ncu_traffic(args.workload, c, world, args.acc) if grp.protocol == "push" else None,
                         "measured_peer_copy": NVLINK_PEER_COPY_GBS,
                         "frac_of_measured_peer_copy": round(achieved / NVLINK_PEER_COPY_GBS, 4),
                         "pattern_ceiling": PATTERN_CEILING_GBS.get(grp.protocol),
                         "frac_of_pattern_ceiling": round(achieved / PATTERN_CEILING_GBS[grp.protocol], 4)
                         if grp.protocol in PATTERN_CEILING_GBS else None,
                         "basis": f"2(C-1)/C*S = {int(alg_bytes)} B per GPU per launch, each direction; "
                                  f"mean over steps of the per-step max over ranks",
                         "peak_source": "NVLink 5 nominal 900 GB/s per direction per GPU (north_star, BASELINE.md); "
                                        "secondary: 770 measured peer copy (B200_PROFILING.md), pattern ceiling "
                                        "from ncu protocol overheads (profiles/r01/ncu_nvlink.md)"},
            "e2e": {"value": round(busbw(total, c, e2e_ms * 1e-3) * world, 3), "unit": "GB/s",
                    "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": world * total * 4, "d2h_bytes_per_step": world * total * 4,
                    "path": f"rv_allreduce_mean_host (pinned host fp32, {args.e2e_lanes} pipelined lanes)",
                    "host_cpus_rank0": numa_cpus or None},
            "gpu_launches": args.steps * world * launches_per_step(args, grp, total),
            "clocks": clk,
        }
        if nccl:
            line["nccl_compare"] = nccl
        if phases:
            line["phases_us"] = phases
        print(json.dumps(line), flush=True)
    grp_e2e.close()
    grp.close()


def optional_leg(name: str, fn):
    """Informational legs (NCCL comparison, phase trace) must never suppress
    the headline line: report a failure in the JSON instead of raising."""
    try:
        return fn()
    except Exception as e:  # pragma: no cover - diagnostic path
        print(f"[bench] optional leg {name} failed: {e!r}", file=sys.stderr, flush=True)
        return {"error": repr(e)[:200]}


def trace_phases(grp, step):
    """Device-side phase split of a few isolated cycles, max over ranks."""
    import torch
    import torch.distributed as dist

    grp.plan.set_trace(True)
    acc = torch.zeros(4, dtype=torch.float64)
    for _ in range(5):
        dist.barrier()
        step()
        torch.cuda.synchronize()
        tr = grp.plan.read_trace(0)
        acc += torch.tensor([tr["ready_us"], tr["data_us"], tr["depart_us"], tr["total_us"]], dtype=torch.float64)
    grp.plan.set_trace(False)
    acc /= 5
    dist.all_reduce(acc, op=dist.ReduceOp.MAX)
    return {k: round(float(v), 2) for k, v in zip(("ready", "data", "depart", "total"), acc)}


def nccl_compare(lens, x, world: int, steps: int, flush=None):
    """NCCL comparison (tools/nccl_compare.py): ncclAllReduce(avg) per ring,
    issued back to back and coalesced into one NCCL group; the faster one is
    the headline comparison.  Same L2 policy as our timed steps."""
    from tools.nccl_compare import NcclRings

    return NcclRings(x, lens).report(steps, flush)


def spawn_ranks(n: int) -> int:
    """``python bench.py --gpus N`` without a launcher: start the N ranks
    (one process per GPU) with torch.distributed.run on 127.0.0.1 and pass
    rank 0's JSON line through.  Returns the launcher's exit code."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="bert")
    ap.add_argument("--acc", choices=["f64", "native"], default="f64")
    ap.add_argument("--lanes", type=int, default=1)
    ap.add_argument("--l2-flush", choices=["auto", "on", "off"], default="auto",
                    help="flush L2 between timed steps (auto: when the per-GPU inputs are < 2x L2)")
    ap.add_argument("--max-blocks", type=int, default=0, help="cap resident blocks of the cycle (0 = all SMs)")
    ap.add_argument("--protocol", choices=["auto", "pull", "push"], default="auto")
    ap.add_argument("--clusters", type=int, default=0, help="N=1 only: co-resident cluster count (default 8)")
    ap.add_argument("--cpu-sample-params", type=int, default=8_000_000)
    ap.add_argument("--ref-sample-params", type=int, default=0,
                    help="--impl reference: time the port on this many params per cluster instead of the "
                         "unmodified reference on the full workload (0 = full)")
    ap.add_argument("--ref-budget-s", type=float, default=60.0,
                    help="--impl reference: cap on the timed full-size cycles (seconds)")
    ap.add_argument("--cpu-port-params", type=int, default=2_000_000,
                    help="cpu_baseline: params per cluster of the port sample")
    ap.add_argument("--nccl", type=int, default=1)
    ap.add_argument("--min-cb", type=int, default=0, help="N>1: force the member-count kernel bucket (8: the 8-GPU kernel)")
    ap.add_argument("--push-items", type=int, default=0, help="N>1: push work items per resident block (0: default)")
    ap.add_argument("--blend-lag", type=int, default=-1, help="N>1: fused-blend lag in groups of C items (-1: default)")
    ap.add_argument("--e2e-seam", type=int, default=1, help="N=1: time apply_ring_mean through the reference's seam")
    ap.add_argument("--e2e-seam-steps", type=int, default=3)
    ap.add_argument("--blend", type=int, default=0, help="config 4: snapshot average + delayed-update blend")
    ap.add_argument("--tau", type=int, default=4)
    ap.add_argument("--fused-blend", type=int, default=1,
                    help="blend inside the cycle (rv_plan_bind_live) instead of separate launches")
    ap.add_argument("--trace", type=int, default=1, help="N>1: add a device-side phase trace")
    ap.add_argument("--numa-bind", type=int, default=1, help="bind ranks to their GPU's NUMA-local CPUs for e2e")
    ap.add_argument("--e2e-lanes", type=int, default=0,
                    help="pipeline stages of the host-buffer path (0: 32 on one GPU, one per ring across GPUs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = max(world, 1) if world > 1 else args.gpus
    if args.e2e_lanes <= 0:
        # measured: finer pipelining helps the single-GPU host path (BERT C=8
        # per step: 8 / 16 / 32 / 64 lanes 79.1 / 76.1-83.8 / 75.8 / 80.4 ms,
        # profiles/r02/e2e_lanes_n1.txt); across GPUs every extra lane adds
        # its own barriers
        args.e2e_lanes = 32 if world <= 1 else len(WORKLOADS[args.workload])

    if args.impl == "reference":
        run_reference(args, n_gpus, rank)
        return
    if world <= 1 and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device(f"cuda:{local_rank}"))
        try:
            run_multi(args, rank, world, local_rank)
        finally:
            dist.destroy_process_group()
        return
    run_single(args)


if __name__ == "__main__":
    main()
