"""torchrun worker: multi-GPU parity of the exchange against the oracle.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tests/dist_worker.py --config tiny --mode split --iters 3

Every rank generates every rank's inputs, runs its own part through the C ABI
(NVLink P2P exchange between the N processes), runs the oracle for all N
simulated workers and asserts parity of its own outputs (tests/_harness.py).
Prints one line "PARITY OK rank=r ..." per rank on success; exits non-zero on
failure.
"""

import argparse
import dataclasses
import os
import sys
import traceback

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--mode", default="split")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0, help="override sequences per rank (0 = config's)")
    ap.add_argument("--pad-id", type=int, default=-1)
    ap.add_argument("--optim", default=None)
    ap.add_argument("--prefetch", action="store_true", help="call emb_prefetch before every forward")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")  # bootstrap only (handles, resync); the exchange is NVLink P2P
    from synthetic import get_config
    from _harness import parity_run

    cfg = get_config(args.config)
    if args.batch:
        cfg = dataclasses.replace(cfg, batch=args.batch) if not cfg.packed else dataclasses.replace(
            cfg, seq_len=args.batch)
    try:
        errs = parity_run(cfg, N=world, rank=rank, mode=args.mode, iters=args.iters, device=local,
                          pad_id=args.pad_id, optim=args.optim, prefetch=args.prefetch)
        print(f"PARITY OK rank={rank} world={world} config={args.config} mode={args.mode} errs={errs}", flush=True)
        code = 0
    except Exception:
        traceback.print_exc()
        print(f"PARITY FAIL rank={rank}", flush=True)
        code = 1
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(code)


if __name__ == "__main__":
    main()
