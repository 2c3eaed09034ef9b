#!/usr/bin/env python
"""Summarise kernel trace rings dumped by `EMB_TRACE_OUT=<prefix> bench.py`
from an EMB_TRACE build (EMB_NVCC_EXTRA=-DEMB_TRACE):  per kernel, the mean
entry / past-waits / finish time in us relative to the forward entry of the
same iteration, over the iterations in the ring, for every rank's file.
Cross-rank offsets use the raw globaltimer (same node)."""
import sys

import numpy as np

NAMES = ["fwd", "sort", "mark", "coal", "merge0", "defpush", "merge1", "rawpush", "rawcoal", "tables",
         "gate_fwd", "gate_sort", "gate_pub0", "gate_pub1", "gate_sorted", "gate_marked", "apply", "k17", "k18", "k19"]
files = sys.argv[1:]
rings = [np.load(f).view(np.uint64).astype(np.int64).reshape(16, 20, 8) for f in files]
base_rank = rings[0]
for f, ring in zip(files, rings):
    print(f)
    # order iterations by their fwd entry; skip the oldest (partially overwritten)
    order = np.argsort(ring[:, 0, 0])
    its = [i for i in order if ring[i, 0, 0] > 0][2:-1]
    steps = np.diff(sorted(ring[its, 0, 0])) / 1e3
    print(f"  iterations {len(its)}  mean fwd-to-fwd {steps.mean():.1f} us  (min {steps.min():.1f} max {steps.max():.1f})")
    for k in range(20):
        rel = []
        for i in its:
            e = ring[i, k]
            if e[0] == 0:
                continue
            t0 = base_rank[i, 0, 0] if base_rank[i, 0, 0] > 0 else ring[i, 0, 0]
            w = e[1] if e[1] > 0 else e[0]
            m = e[3] if e[3] > 0 else e[0]
            rel.append(((e[0] - t0) / 1e3, (m - t0) / 1e3, (w - t0) / 1e3, (e[2] - t0) / 1e3))
        if rel:
            r = np.array(rel).mean(0)
            extra = "  ".join(f"s{j}:{(np.mean([ring[i, k, j] for i in its]) - np.mean([base_rank[i, 0, 0] for i in its])) / 1e3:6.1f}"
                              for j in range(4, 8) if all(ring[i, k, j] > 0 for i in its))
            print(f"  {NAMES[k]:8s} enter {r[0]:7.1f}  mid {r[1]:7.1f}  waited {r[2]:7.1f}  done {r[3]:7.1f}"
                  f"   (span {r[3]-r[0]:5.1f})  {extra}")
