#!/usr/bin/env python
"""NVLink reference bandwidths on the box the exchange runs on (SURVEY §8(d):
"measure achievable P2P store bandwidth and NCCL AlltoAll bus bandwidth").

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      scripts/nvlink_bench.py

Per message size (bytes per peer pair, the exchange's range):
  * NCCL all_to_all_single (the library AlltoAll the paper uses):
    algorithm bandwidth per rank = bytes sent to peers / time, and the
    per-direction NVLink rate of one GPU;
Device time with CUDA events, max over ranks.  One JSON line on rank 0.
"""

import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    out = {"n_gpus": world, "alltoall": []}
    for per_pair in (256 << 10, 1 << 20, 4 << 20, 16 << 20):
        n = per_pair * world // 4
        x = torch.ones(n, dtype=torch.float32, device=dev)
        y = torch.empty_like(x)
        for _ in range(5):
            dist.all_to_all_single(y, x)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 50
        e0.record()
        for _ in range(it):
            dist.all_to_all_single(y, x)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / it], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms.item())
        sent = per_pair * (world - 1)
        out["alltoall"].append({"bytes_per_pair": per_pair, "us": round(ms * 1e3, 2),
                                "gbs_per_rank_out": round(sent / (ms * 1e-3) / 1e9, 1)})
    # NCCL all_reduce of one dense block (bf16), the a13 queue's collective
    out["allreduce"] = []
    for mib in (4, 25, 100):
        x = torch.ones((mib << 20) // 2, dtype=torch.bfloat16, device=dev)
        for _ in range(5):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 20
        e0.record()
        for _ in range(it):
            dist.all_reduce(x)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / it], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms.item())
        algbw = (mib << 20) / (ms * 1e-3) / 1e9
        out["allreduce"].append({"mib_bf16": mib, "us": round(ms * 1e3, 1), "algbw_gbs": round(algbw, 1),
                                 "busbw_gbs": round(algbw * 2 * (world - 1) / world, 1)})
    if rank == 0:
        out["note"] = ("alltoall gbs_per_rank_out = bytes each rank sends to its N-1 peers / time (the exchange's "
                       "per-GPU NVLink injection); nominal 900 GB/s per direction, guide-measured peer copy 770")
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
