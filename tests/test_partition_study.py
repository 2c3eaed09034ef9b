"""NEXT-4: the row-wise vs column-wise partition load study
(PAPER.md:271-274 — "some parts will be accessed much more frequently under
the row-wise situation, leading to an unbalancing communication cost ... [with
column-wise] each partition will get the same amount of requests"; PAPER.md:
472-475, Parallax's row-wise PS vs CPPS).  On the synthetic paper-shaped Zipf
batches at N = 2, 4, 8, the NVLink bytes each owner must SEND in one forward
exchange (oracle.partition.forward_bytes_out) under column-wise, row-wise
(contiguous rows of a frequency-sorted vocabulary) and row-wise hashed (id mod
N) partitions; the exchange is bound by the busiest owner.  Run with -s to
print the table (profiles/r02_partition/study.txt)."""

import numpy as np
import pytest

from oracle import partition
from synthetic import get_config, make_workload

NVL = 770e9  # B/s, the guide's measured peer-copy rate per direction


@pytest.mark.parametrize("name", ["lstm_lm", "gnmt", "transformer", "bert_large"])
def test_partition_load_study(name):
    cfg = get_config(name)
    esz = 2 if cfg.dtype == "bf16" else 4
    rows = []
    for N in (2, 4, 8):
        wl = make_workload(cfg, N, 2, with_dY=False)
        out = {}
        for scheme in ("column", "row", "hash"):
            per_it = [partition.forward_bytes_out(wl.ids[k], cfg.L, cfg.D, N, scheme, esz) for k in range(2)]
            b = np.mean(per_it, axis=0)
            out[scheme] = (b.max(), b.mean())
        rows.append((N, out))
        col_max, col_mean = out["column"]
        row_max, row_mean = out["row"]
        hash_max, hash_mean = out["hash"]
        assert col_max / col_mean < 1.01                      # balanced
        assert row_max / row_mean > 1.5                       # frequency-sorted rows: a hot owner
        assert row_max > col_max                              # the busiest owner sends more
    print(f"\n{name} (L={cfg.L}, D={cfg.D} {cfg.dtype}): forward NVLink bytes sent by the busiest owner "
          f"(max/mean over owners) and its time at 770 GB/s")
    for N, out in rows:
        cells = "  ".join(f"{s}: {out[s][0] / 2**20:7.2f} MiB ({out[s][0] / out[s][1]:4.2f}x) "
                          f"{out[s][0] / NVL * 1e6:6.1f} us" for s in ("column", "row", "hash"))
        print(f"  N={N}  {cells}")
