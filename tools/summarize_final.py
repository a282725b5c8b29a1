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
            cb = d["cpu_baseline"]
            rows.append(f"| {name} (reference arm: {cb['kind']}, {cb['cores']} core, "
                        f"{d.get('steps')} of {d.get('steps_requested', d.get('steps'))} steps) "
                        f"| {d['value']} | {d['ms_per_step']} | | | | | | | |")
            continue
        rf = d.get("roofline", {})
        cfg = d.get("config", {})
        nccl = (d.get("nccl_compare") or {}).get("bus_gbps_per_gpu", "—")
        transport = "co-resident TMA" if d["n_gpus"] == 1 else cfg.get("protocol")
        blend = cfg.get("blend")
        opts = cfg.get("plan_options")
        seam = (d.get("e2e_seam") or {}).get("ms_per_step")
        rows.append(
            f"| {name} | {d['value']} | {d['ms_per_step']} / {d.get('ms_per_step_median', '—')} "
            f"| {d.get('bus_gbps_per_gpu', '—')} | {rf.get('frac')} "
            f"| {rf.get('frac_of_pattern_ceiling', '—')} | {d['e2e']['value']} "
            f"| {f'{seam} ms' if seam else '—'} | {nccl} "
            f"| {transport} (lanes {cfg.get('lanes')}){'; ' + blend if blend else ''}{f'; {opts}' if opts else ''} |")
    head = """# Final measurements (`tools/gpu_final.sh`, one box)

All lines are `bench.py` output; raw JSON in `final/*.jsonl`.
- `value` is the whole-job aggregate: N × busbw (NCCL convention, fp32 bytes).
- Roofline fractions are against:
  - the measured HBM copy (N=1; the fused-blend line counts 4·C·S bytes);
  - 900 GB/s, NVLink 5 per direction per GPU (N>1, `frac`);
  - the 706 GB/s push-pattern ceiling derived from ncu NVLink counters (`pattern`).
- N>1: every step starts after a rank-aligning barrier; ms/step is the mean / median of the per-step max over ranks.
- NCCL is the better of sequential and coalesced `AllReduce(avg)` per ring.
- seam: `ravnest.multiring.apply_ring_mean` after `plugin.install` (numpy float64 in/out), ms per call.
- The reference arm runs the unmodified `apply_ring_mean` on the full workload (`kind: reference`).

| run | value GB/s | ms/step mean / median | bus GB/s per GPU | roofline frac | pattern | e2e GB/s | seam | NCCL bus GB/s | transport |
|---|---|---|---|---|---|---|---|---|---|
"""
    notes = """
Notes:
- `*_gpt2_blend` is config 4: snapshot average + τ=4 delayed-update blend per step, the blend fused into the
  cycle (`rv_plan_bind_live`). Its value uses the whole step; at N=1 the roofline counts the fused kernel's
  4·C·S bytes, at N>1 the NVLink bytes of the cycle.
- `lanes 4` is one launch and stream per ring (the north star's layout).
- `pytest_gpu.log`: the GPU test suite of the same session.
- `*_cb8`: the CB = 8 push kernel (what every rank of an 8-GPU job runs) forced with the `min_cb` plan option.
"""
    with open(out, "w") as f:
        f.write(head + "\n".join(rows) + "\n" + notes)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
