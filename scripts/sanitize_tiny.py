#!/usr/bin/env python
"""Small runs of the exchange for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per invocation): tiny config, N = 1, RAW / COAL / SPLIT,
SGD and Adam, with and without emb_prefetch, each checked against the oracle.
  compute-sanitizer --tool memcheck python scripts/sanitize_tiny.py"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
sys.path.insert(0, os.path.dirname(HERE))

from _harness import parity_run  # noqa: E402
from synthetic import get_config  # noqa: E402

cfg = get_config("tiny")
for mode in ("raw", "coal", "split"):
    parity_run(cfg, N=1, mode=mode, iters=3)
parity_run(cfg, N=1, mode="split", iters=3, optim="adam", lr=1e-2, prefetch=True)
parity_run(cfg, N=1, mode="split", iters=4, pipelined=True, null_at=(1,))
print("SANITIZE RUN OK")
