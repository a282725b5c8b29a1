"""Build profiles/<round>/SUMMARY.md from the bench lines of tools/gpu_final.sh.

    python tools/summarize_final.py profiles/r01/final profiles/r01/SUMMARY.md
"""

import glob
import json
import os
import sys


def last_json(path):
    line = None
    with open(path) as f:
        for raw in f:
            if raw.startswith("{"):
                line = raw
    return json.loads(line) if line else None


def key(name):
    # n1 before n2 before n4; reference lines last
    ref = name.startswith("ref")
    n = int("".join(ch for ch in name.split("_")[0 if not ref else 1] if ch.isdigit()) or 0)
    return (ref, n, name)


def main(src, out):
    rows = []
    for path in sorted(glob.glob(os.path.join(src, "*.jsonl")), key=lambda p: key(os.path.basename(p)[:-6])):
        name = os.path.basename(path)[:-6]
        d = last_json(path)
        if not d or "value" not in d:
            continue
        if d.get("impl") == "reference":
            rows.append(f"| {name} (reference arm: {d['cpu_baseline']['kind']}, {d['cpu_baseline']['cores']} core) "
                        f"| {d['value']} | {d['ms_per_step']} | | | | | | |")
            continue
        rf = d.get("roofline", {})
        cfg = d.get("config", {})
        nccl = (d.get("nccl_compare") or {}).get("bus_gbps_per_gpu", "—")
        transport = "co-resident TMA" if d["n_gpus"] == 1 else cfg.get("protocol")
        blend = cfg.get("blend")
        rows.append(
            f"| {name} | {d['value']} | {d['ms_per_step']} | {d.get('bus_gbps_per_gpu', '—')} | {rf.get('frac')} "
            f"| {rf.get('frac_of_pattern_ceiling', '—')} | {d['e2e']['value']} | {nccl} "
            f"| {transport} (lanes {cfg.get('lanes')}){'; ' + blend if blend else ''} |")
    head = """# Final measurements (`tools/gpu_final.sh`, one box)

All lines are `bench.py` output; raw JSON in `final/*.jsonl`.
- `value` is the whole-job aggregate: N × busbw (NCCL convention, fp32 bytes).
- Roofline fractions are against:
  - the measured HBM copy (N=1; the fused-blend line counts 4·C·S bytes);
  - the 770 GB/s measured peer copy (N>1, `frac`);
  - the 706 GB/s push-pattern ceiling derived from ncu NVLink counters (`pattern`).
- NCCL is the better of sequential and coalesced `AllReduce(avg)` per ring.

| run | value GB/s | ms/step | bus GB/s per GPU | roofline frac | pattern | e2e GB/s | NCCL bus GB/s | transport |
|---|---|---|---|---|---|---|---|---|
"""
    notes = """
Notes:
- `*_gpt2_blend` is config 4: snapshot average + τ=4 delayed-update blend per step, the blend fused into the
  cycle (`rv_plan_bind_live`). Its value uses the whole step; at N=1 the roofline counts the fused kernel's
  4·C·S bytes, at N>1 the NVLink bytes of the cycle.
- `lanes 4` is one launch and stream per ring (the north star's layout).
- `pytest_gpu.log`: the GPU test suite of the same session.
- `*_rerun*`: a configuration run again in a separate call. When the timed steps are separated by L2 flushes
  (ResNet-50 at N>1), `ms_per_step` is the mean of the per-step intervals, so one slow step (a rank whose host
  queued its step late) raises the mean; the line's `ms_per_step_median` / `ms_per_step_min` show it.
"""
    with open(out, "w") as f:
        f.write(head + "\n".join(rows) + "\n" + notes)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
