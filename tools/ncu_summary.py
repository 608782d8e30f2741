#!/usr/bin/env python3
"""Summarise ncu output for profiles/: the launch list (share of device time per
kernel) and the key counters of a `--set full` capture.

  python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN/launch_share.md
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep     > profiles/rNN/full_key_metrics.csv
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = OrderedDict([
    ("duration_ms", ("gpu__time_duration.sum", 1e-6)),          # ns -> ms (unit-checked below)
    ("dram_read_GB", ("dram__bytes_read.sum", None)),
    ("dram_write_GB", ("dram__bytes_write.sum", None)),
    ("dram_pct_peak", ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None)),
    ("l2_pct_peak", ("lts__throughput.avg.pct_of_peak_sustained_elapsed", None)),
    ("l1_wavefronts_pct", ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", None)),
    ("l1_hit_pct", ("l1tex__t_sector_hit_rate.pct", None)),
    ("l2_sectors", ("lts__t_sectors.sum", None)),
    ("occupancy_pct", ("sm__warps_active.avg.pct_of_peak_sustained_active", None)),
    ("regs", ("launch__registers_per_thread", None)),
])
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3}


def short(name):
    return name.split("(")[0].replace("void ", "").strip()


def launches(path):
    tot, cnt = OrderedDict(), OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(io.StringIO("".join(lines))):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(row["Kernel Name"])
        v = float(row["Metric Value"].replace(",", "")) * SCALE.get(row["Metric Unit"], 1e-6)
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] = cnt.get(k, 0) + 1
    all_ms = sum(tot.values())
    print("| kernel | launches | total ms | mean ms | share |")
    print("|---|---:|---:|---:|---:|")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"| `{k}` | {cnt[k]} | {tot[k]:.3f} | {tot[k] / cnt[k]:.4f} | {100 * tot[k] / all_ms:.1f} % |")
    print(f"\nTotal device time in the list: {all_ms:.3f} ms over {sum(cnt.values())} launches.")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]

    def col(metric):
        if metric in hdr:
            return hdr.index(metric)
        for i, h in enumerate(hdr):
            if h.endswith("." + metric):
                return i
        return None

    w = csv.writer(sys.stdout)
    w.writerow(["id", "kernel", "grid", "block"] + list(KEYS))
    for r in data:
        vals = []
        for key, (metric, _) in KEYS.items():
            i = col(metric)
            if i is None or not r[i]:
                vals.append("")
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                vals.append("")
                continue
            u = units[i]
            if key == "duration_ms" or key.endswith("_GB"):
                v *= SCALE.get(u, 1.0)
            vals.append(f"{v:.6g}")
        w.writerow([r[0], short(r[hdr.index("Kernel Name")]), r[hdr.index("Grid Size")],
                    r[hdr.index("Block Size")]] + vals)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
