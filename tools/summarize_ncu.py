"""Summaries of ncu captures for profiles/: launch-list shares and key metrics
of the full captures (read here, on the CPU box, from gpurun_out/)."""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) > vi:
            agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k[:70]}` | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/len(v)/1e3:.2f} | "
                   f"{sum(v)/tot:.3f} |")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__block_size", "launch__cluster_dim_x",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_barrier",
           "smsp__pcsamp_warps_issue_stalled_no_instructions"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        out.append(f"### `{name}`")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"- {m}: {row[i]} {u[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
