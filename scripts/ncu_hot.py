#!/usr/bin/env python
"""Summarise an ncu report: per-kernel headline metrics and the hottest source
lines by warp-stall samples.

  python scripts/ncu_hot.py REPORT.ncu-rep [kernel-regex] [--src cuda|sass] [--top N]
"""

import csv
import io
import subprocess
import sys

HEAD = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Compute (SM) Throughput", "L2 Hit Rate", "Grid Size", "Block Size", "Warp Cycles Per Issued Instruction",
        "Executed Instructions"]


def run(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def details(rep, kre):
    out = run(["-i", rep, "--page", "details", "--csv"] + (["--kernel-name", f"regex:{kre}"] if kre else []))
    r = list(csv.reader(io.StringIO(out)))
    if not r:
        return
    h = r[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    for x in r[1:]:
        if x[mi] in HEAD:
            print(f"{x[ii]:>3} {x[ki][:40]:40} {x[mi]:36} {x[vi]} {x[ui]}")


def hot(rep, kre, src, top):
    out = run(["-i", rep, "--page", "source", "--csv", "--print-source", src] +
              (["--kernel-name", f"regex:{kre}"] if kre else []))
    lines = out.splitlines()
    blocks, cur = [], []
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            if cur:
                blocks.append(cur)
            cur = [ln]
        else:
            cur.append(ln)
    if cur:
        blocks.append(cur)
    for b in blocks[:1]:
        print(b[0][:160])
        r = list(csv.reader(io.StringIO("\n".join(b[1:]))))
        while r and "Warp Stall Sampling (All Samples)" not in r[0]:
            r = r[1:]
        if not r:
            print("(no per-line stall metrics in this view; try --src sass)")
            return
        h = r[0]
        si = h.index("Warp Stall Sampling (All Samples)")
        srci = h.index("Source")
        stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        rows = [x for x in r[1:] if len(x) > si and x[si] not in ("", "0")]
        tot = sum(float(x[si]) for x in rows) or 1
        rows.sort(key=lambda x: -float(x[si]))
        for x in rows[:top]:
            st = sorted(((float(x[i]) if x[i] else 0, h[i][6:]) for i in stall_cols), reverse=True)[:3]
            lab = ", ".join(f"{n}={v:.0f}" for v, n in st if v > 0)
            loc = x[0] if src == "cuda" else ""
            print(f"{100 * float(x[si]) / tot:5.1f}%  {loc[:6]:6} {x[srci].strip()[:90]:90} [{lab}]")


def by_line(rep, kre, top):
    """Aggregate executed instructions and stall samples per CUDA source line
    (cuda,sass view: a line row carries the totals of the SASS rows below it)."""
    out = run(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] +
              (["--kernel-name", f"regex:{kre}"] if kre else []))
    fname, rows = None, []
    hdr = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr[4:], rec[4:]))
        try:
            ins = float(d.get("Instructions Executed", "0") or 0)
            smp = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        rows.append((ins, smp, f"{fname}:{rec[0]}", rec[1].strip()[:80]))
    ti = sum(r[0] for r in rows) or 1
    ts = sum(r[1] for r in rows) or 1
    print(f"total instructions {ti:.0f}, samples {ts:.0f}")
    for ins, smp, loc, src in sorted(rows, key=lambda r: -r[0])[:top]:
        print(f"{100 * ins / ti:5.1f}% ins {100 * smp / ts:5.1f}% smp  {loc:18} {src}")


if __name__ == "__main__":
    if "--lines" in sys.argv:
        a = [x for x in sys.argv[1:] if x != "--lines"]
        by_line(a[0], a[1] if len(a) > 1 else None, int(a[a.index("--top") + 1]) if "--top" in a else 30)
        sys.exit(0)
    a = sys.argv[1:]
    rep = a[0]
    kre = a[1] if len(a) > 1 and not a[1].startswith("--") else None
    src = a[a.index("--src") + 1] if "--src" in a else "cuda"
    top = int(a[a.index("--top") + 1]) if "--top" in a else 25
    details(rep, kre)
    hot(rep, kre, src, top)
