"""torchrun worker: the dense-gradient AllReduce priority queue (SURVEY §8(a)
a13) on N GPUs — values against the oracle's all-reduce mean, issue order
against the oracle's window rule (reading R16)."""

import argparse
import os
import sys
import traceback

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--window", type=int, default=1)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from oracle import collectives, schedule
    from paper_2110_09132_b200 import embrace as E
    from paper_2110_09132_b200.runtime import EmbraceExchange
    from synthetic import get_config
    from synthetic.workloads import gen_table

    code = 1
    try:
        cfg = get_config("tiny")
        d = cfg.D // world
        W = gen_table(cfg)
        shard = torch.from_numpy(np.ascontiguousarray(W[:, rank * d:(rank + 1) * d])).cuda()
        ex = EmbraceExchange(cfg.L, cfg.D, shard, world=world, rank=rank, device=local, dtype="fp32",
                             max_tokens=cfg.max_tokens, mode="split", optim="sgd", lr=0.1, dense_queue=True,
                             queue_window=args.window)
        # blocks in BP order with FP-order priorities (lower = sooner); sizes and dtypes mixed
        prios = [5, 1, 4, 0, 3, 2, 1]
        sizes = [1, 4099, 1 << 16, 3, 1 << 20, 777, 2048]
        dts = [torch.float32, torch.bfloat16, torch.float32, torch.bfloat16, torch.bfloat16, torch.float32,
               torch.float32]
        stream = torch.cuda.current_stream()
        host, bufs, tickets, events = [], [], [], []
        for k, (pr, n, dt) in enumerate(zip(prios, sizes, dts)):
            g = np.random.default_rng([0x21100913, k, rank]).uniform(-1, 1, n)
            # every rank's contribution, for the oracle (same seeds)
            allr = [np.random.default_rng([0x21100913, k, s]).uniform(-1, 1, n) for s in range(world)]
            t = torch.from_numpy(g).to(dt).cuda()
            allr = [torch.from_numpy(a).to(dt).double().numpy() for a in allr]  # what each rank put in
            ev = torch.cuda.Event()
            ev.record(stream)
            events.append(ev)  # borrowed by the queue until issued (embrace.h)
            tickets.append(E.dense_allreduce_enqueue(ex.ctx, t, pr, ev))
            host.append((allr, dt))
            bufs.append(t)
        E.dense_queue_flush(ex.ctx)
        for tk in tickets:
            E.dense_wait(ex.ctx, tk, stream)
        torch.cuda.synchronize()
        for k, (t, (allr, dt)) in enumerate(zip(bufs, host)):
            ref = collectives.all_reduce(allr)[0] / world
            sig = np.sum(np.abs(np.stack(allr)), axis=0) / world
            got = t.double().cpu().numpy()
            err = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), sig)) if got.size else 0.0
            tol = 2e-2 if dt == torch.bfloat16 else 1e-5
            assert err <= tol, f"block {k}: err {err:.3e} > {tol}"
        log = ex.debug(E.EMB_DBG_ISSUE_LOG)
        want = schedule.issue_order(prios, args.window)
        assert [int(x) for x in log] == [int(tickets[i]) for i in want], (list(log), want, tickets)
        print(f"DENSE OK rank={rank} world={world} window={args.window}", flush=True)
        code = 0
        ex.close()
    except Exception:
        traceback.print_exc()
        print(f"DENSE FAIL rank={rank}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(code)


if __name__ == "__main__":
    main()
