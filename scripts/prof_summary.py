#!/usr/bin/env python
"""Summaries for profiles/ (committed evidence):

  prof_summary.py launches LAUNCHES.csv      per-kernel launch count, mean / total
                                             gpu__time_duration and share of the
                                             profiled time (ncu launch list)
  prof_summary.py full REPORT.ncu-rep        per-kernel headline metrics of an
                                             `ncu --set full` capture (duration,
                                             DRAM bytes read + written, throughput,
                                             occupancy, registers, instructions)
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("emb::", "")


def launches(path):
    rows = [ln for ln in open(path) if ln.startswith('"')]
    r = list(csv.DictReader(io.StringIO("".join(rows))))
    agg = collections.OrderedDict()
    for x in r:
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(x["Kernel Name"])
        v = float(x["Metric Value"].replace(",", "")) / 1e3  # ns -> us
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'mean us':>9s} {'total us':>10s} {'share':>6s}")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {s / n:9.2f} {s:10.1f} {100 * s / tot:5.1f}%")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    idx = {m: h.index(m) for m in METRICS if m in h}
    ki, gi = h.index("Kernel Name"), h.index("Grid Size")

    def val(x, m):
        if m not in idx or not x[idx[m]]:
            return None
        return float(x[idx[m]].replace(",", "")) * SCALE.get(units[idx[m]], 1.0)

    print("| kernel | grid | us | DRAM read MB | DRAM write MB | DRAM GB/s | warps active % | regs | warp instr | L2 hit % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for x in r[2:]:
        us, rd, wr = val(x, "gpu__time_duration.sum"), val(x, "dram__bytes_read.sum"), val(x, "dram__bytes_write.sum")
        gbs = (rd + wr) / us * 1e3 if us and rd is not None else None
        f = lambda v, fmt="{:.1f}": "-" if v is None else fmt.format(v)
        print(f"| {short(x[ki])} | {x[gi]} | {f(us, '{:.2f}')} | {f(rd, '{:.2f}')} | {f(wr, '{:.2f}')} | {f(gbs, '{:.0f}')} "
              f"| {f(val(x, 'sm__warps_active.avg.pct_of_peak_sustained_active'))} "
              f"| {f(val(x, 'launch__registers_per_thread'), '{:.0f}')} | {f(val(x, 'smsp__inst_executed.sum'), '{:.0f}')} "
              f"| {f(val(x, 'lts__t_sector_hit_rate.pct'))} |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
