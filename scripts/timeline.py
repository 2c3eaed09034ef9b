#!/usr/bin/env python
"""Summarise an EMB_PROF_TIMELINE dump (kind start_us dur_us per launch, one
file per rank): mean start offset / duration of each kernel relative to the
step's forward launch, over the steps after the first few."""
import sys
from collections import defaultdict

NAMES = ["fwd", "sort", "mark", "coal", "merge0", "defpush", "merge1", "rawpush", "rawcoal", "tables"]
for path in sys.argv[1:]:
    rows = [tuple(map(float, ln.split())) for ln in open(path) if ln.strip()]
    steps, cur = [], []
    for k, s, d in rows:
        if int(k) == 0 and cur:
            steps.append(cur)
            cur = []
        cur.append((int(k), s, d))
    steps.append(cur)
    steps = steps[4:-1]
    acc = defaultdict(lambda: [0.0, 0.0, 0])
    per = []
    for st in steps:
        t0 = st[0][1]
        for k, s, d in st:
            a = acc[k]
            a[0] += s - t0
            a[1] += d
            a[2] += 1
    for i in range(len(steps) - 1):
        per.append(steps[i + 1][0][1] - steps[i][0][1])
    print(f"{path}: {len(steps)} steps, mean step {sum(per) / max(1, len(per)):.1f} us")
    for k, (s, d, n) in sorted(acc.items(), key=lambda kv: kv[1][0] / kv[1][2]):
        print(f"  {NAMES[k]:8s} start {s / n:7.1f}  dur {d / n:6.1f}  ({n / len(steps):.0f}/step)")
