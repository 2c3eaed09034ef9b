#!/usr/bin/env python
"""NVLink peer-memory bandwidth of SM-issued 16-byte loads / stores between
GPU 0 and GPU 1 of this box (one process, peer access enabled) — the
achievable rate for the exchange's forward pull (loads from the peer's shard)
and backward push (stores into the owner's receive rows); SURVEY §8(d)
"measure achievable P2P store bandwidth".  Kernel: scripts/p2p_bw.cu.

  python scripts/p2p_bw.py [out.json]

Per size and grid: pull (GPU 0 reads GPU 1's memory), push (GPU 0 writes
GPU 1's memory), local (same-device copy, HBM reference), and both GPUs
pulling from each other at once (both link directions loaded).  GB/s = bytes
moved over the link per second (copy bytes / time).  CUDA events, average of
`iters` back-to-back copies after 3 warm-ups.
"""

import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def build():
    so = os.path.join(ROOT, "build", "p2p_bw.so")
    os.makedirs(os.path.dirname(so), exist_ok=True)
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                    os.path.join(HERE, "p2p_bw.cu"), "-o", so], check=True)
    return ctypes.CDLL(so)


def main():
    assert torch.cuda.device_count() >= 2, "needs two GPUs"
    lib = build()
    f = ctypes.c_float
    lib.p2p_copy.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                             ctypes.c_int, ctypes.POINTER(f)]
    lib.p2p_copy2.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                                      ctypes.POINTER(f), ctypes.POINTER(f)]
    assert lib.p2p_enable(0, 1) == 0 and lib.p2p_enable(1, 0) == 0, "peer access"
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    out = {"gpu": torch.cuda.get_device_name(0), "nsm": nsm, "rows": []}
    big = 256 << 20
    a0 = torch.empty(big, dtype=torch.uint8, device="cuda:0")
    b0 = torch.empty(big, dtype=torch.uint8, device="cuda:0")
    a1 = torch.empty(big, dtype=torch.uint8, device="cuda:1")
    b1 = torch.empty(big, dtype=torch.uint8, device="cuda:1")
    for d in (0, 1):
        torch.cuda.synchronize(d)
    for mb in (1, 4, 16, 64, 256):
        nb = mb << 20
        iters = max(5, min(200, (2048 << 20) // nb))
        for per_sm in (2, 4, 8):
            grid = nsm * per_sm
            row = {"mbytes": mb, "grid": grid}
            for name, dev, dst, src in (("pull", 0, b0, a1), ("push", 0, b1, a0), ("local", 0, b0, a0)):
                ms = f()
                rc = lib.p2p_copy(dev, dst.data_ptr(), src.data_ptr(), nb, grid, iters, ctypes.byref(ms))
                assert rc == 0, (name, rc)
                row[name + "_gbs"] = round(nb / (ms.value * 1e-3) / 1e9, 1)
            m0, m1 = f(), f()
            rc = lib.p2p_copy2(b0.data_ptr(), a1.data_ptr(), b1.data_ptr(), a0.data_ptr(), nb, grid, iters,
                               ctypes.byref(m0), ctypes.byref(m1))
            assert rc == 0, ("pull2", rc)
            row["pull_both_gbs_per_gpu"] = round(nb / (max(m0.value, m1.value) * 1e-3) / 1e9, 1)
            out["rows"].append(row)
            print(json.dumps(row), flush=True)
    best = {k: max(r[k] for r in out["rows"]) for k in ("pull_gbs", "push_gbs", "local_gbs", "pull_both_gbs_per_gpu")}
    out["best"] = best
    out["note"] = ("SM-issued 16-byte copies over NVLink 5 between two B200s of one box; nominal 900 GB/s per "
                   "direction.  pull = loads from the peer (the forward pull-gather's pattern), push = stores to "
                   "the peer (the gradient push's pattern), pull_both = both GPUs pulling at once.")
    print(json.dumps({"best": best}), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
