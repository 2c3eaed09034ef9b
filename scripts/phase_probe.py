#!/usr/bin/env python
"""Print device phase timestamps of the route kernel (needs a build with
EMB_NVCC_EXTRA=-DEMB_PHASE_TIMING).  Runs a few LM-shaped iterations at N=1."""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_09132_b200 import embrace as E  # noqa: E402
from paper_2110_09132_b200.runtime import EmbraceExchange  # noqa: E402
from synthetic import get_config, make_workload  # noqa: E402
from synthetic.workloads import gen_table  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "lstm_lm")
mode = sys.argv[2] if len(sys.argv) > 2 else "split"
wl = make_workload(cfg, 1, 6)
W = torch.from_numpy(gen_table(cfg)).cuda()
if cfg.dtype == "bf16":
    W = W.to(torch.bfloat16)
ex = EmbraceExchange(cfg.L, cfg.D, W, max_tokens=cfg.max_tokens, mode=mode, optim=cfg.optim, lr=cfg.lr,
                     dtype=cfg.dtype)
tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
for k in range(5):
    ids = torch.from_numpy(wl.ids[k][0]).cuda()
    ex.forward(ids)
    ex.backward(torch.from_numpy(wl.dY[k][0]).cuda().to(tdt), torch.from_numpy(wl.ids[k + 1][0]).cuda())
    ex.flush()
    ts = E.emb_debug_copy(ex.ctx, E.EMB_DBG_TIMESTAMPS).view(np.uint64).astype(np.int64)
    base = ts[0]
    marks = {i: (ts[i] - base) / 1e3 for i in range(16) if ts[i] >= base and ts[i] > 0}
    print(f"iter {k}: " + "  ".join(f"{i}:{v:.2f}us" for i, v in sorted(marks.items())))
ex.close()
