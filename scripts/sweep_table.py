#!/usr/bin/env python
"""Markdown table of a bench sweep directory (scripts/sweep.sh output)."""
import glob
import json
import os
import sys

d = sys.argv[1]
print("| run | value (Mtok/s) | us/step | dominant kernel | frac | traffic MB | step frac | e2e (Mtok/s) | launches/step | SM MHz | cpu baseline |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    for line in open(f):
        if not line.startswith("{"):
            continue
        x = json.loads(line)
        if "unavailable" in x:
            print(f"| {os.path.basename(f)} | unavailable |"); continue
        rf = x.get("roofline") or {}
        sr = x.get("step_roofline") or {}
        e2e = x.get("e2e") or {}
        cb = x.get("cpu_baseline") or {}
        ck = x.get("clocks") or {}
        tr = rf.get("traffic")
        cbs = f"{cb.get('value'):.0f} {cb.get('unit', '')} ({cb.get('cores')} core)" if cb.get("value") else ""
        print(f"| {os.path.basename(f)[:-5]} | {x['value'] / 1e6:.2f} | {x['ms_per_step'] * 1e3:.1f} | {rf.get('kernel', '')} "
              f"| {rf.get('frac', '')} | {'' if tr is None else round(tr / 1e6, 1)} | {sr.get('frac', '')} "
              f"| {(e2e.get('value') or 0) / 1e6:.2f} | {x.get('gpu_launches_per_step', '')} | {ck.get('sm_mhz', '')} | {cbs} |")
