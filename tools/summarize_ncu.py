"""Summarise ncu outputs into profiles/ (run in the dev container).

    python tools/summarize_ncu.py launches <launches.csv> <out.md>
    python tools/summarize_ncu.py full <report.ncu-rep> <out.md> [algorithmic_bytes]
"""

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.search(r"(ring_\w+_kernel<[^>]*>|blend_kernel\w*<[^>]*>)", name)
    if m:
        return m.group(1)
    return name.split("(")[0][-90:]


def launches(path: str, out: str) -> None:
    rows = []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            unit = r["Metric Unit"]
            v = float(r["Metric Value"].replace(",", ""))
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
            rows.append((int(r["ID"]), short(r["Kernel Name"]), r["Grid Size"], ns))
    agg = defaultdict(lambda: [0, 0.0])
    for _, k, _, ns in rows:
        agg[k][0] += 1
        agg[k][1] += ns
    total = sum(v[1] for v in agg.values())
    ours = sum(v[1] for k, v in agg.items() if k.startswith("ring_") or "blend" in k)
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({path})\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole program "
                "(setup + timed steps + e2e); per-launch times are cold-cache and serialised.\n\n")
        f.write(f"launches: {len(rows)}; our kernels' share of all GPU time: {100 * ours / total:.1f}%\n\n")
        f.write("| kernel | launches | total ms | mean us |\n|---|---|---|---|\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} |\n")
        ring = [r for r in rows if r[1].startswith("ring_")]
        if ring:
            f.write("\nring kernel launches (in order): " + ", ".join(f"{r[3] / 1e3:.1f}us" for r in ring) + "\n")
    print(open(out).read())


METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__waves_per_multiprocessor", "smsp__inst_executed.sum", "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
]


def full(path: str, out: str, alg_bytes: float | None) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({path.split('/')[-1]})\n\n")
        for vals in rows[2:]:
            name = vals[hdr.index("Kernel Name")]
            f.write(f"## `{short(name)}`\n\n| metric | value | unit |\n|---|---|---|\n")
            got = {}
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    f.write(f"| {m} | {vals[i]} | {units[i]} |\n")
                    got[m] = (vals[i], units[i])
            if alg_bytes and "dram__bytes_read.sum" in got:
                def gb(v):
                    x, u = v
                    x = float(x.replace(",", ""))
                    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
                traffic = gb(got["dram__bytes_read.sum"]) + gb(got["dram__bytes_write.sum"])
                f.write(f"\ntraffic (dram read+write) = {traffic:.4e} B; algorithmic = {alg_bytes:.4e} B; "
                        f"ratio = {traffic / alg_bytes:.4f}\n\n")
    print(open(out).read())


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
