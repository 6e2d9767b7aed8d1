"""Summarise ncu evidence for profiles/: the per-kernel launch list of a
`--metrics gpu__time_duration.sum` run and key metrics of `--set full` reports.
usage: python scripts/ncu_summary.py launches.csv [report.ncu-rep ...]"""
import collections
import csv
import subprocess
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = r[h.index("Kernel Name")].split("(")[0]
        v = float(r[h.index("Metric Value")].replace(",", "")) * SCALE[r[h.index("Metric Unit")]]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | µs (sum) | share |\n|---|---|---|---|")
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {v:.1f} | {100 * v / tot:.1f}% |")
    print(f"\ntotal {tot:.1f} µs")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print(f"\n{path}: {name[:80]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k} = {v[i]} {u[i]}")


if __name__ == "__main__":
    launches(sys.argv[1])
    for p in sys.argv[2:]:
        report(p)
