"""Debug: LM-shaped N=2 eager iterations, then print the kernel trace of t=1..5 (EMB_TRACE build)."""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2110_09132_b200 import embrace as E
from paper_2110_09132_b200.runtime import EmbraceExchange
from synthetic import get_config, make_workload
from synthetic.workloads import gen_table
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl")
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "lstm_lm")
wl = make_workload(cfg, world, 6)
W = gen_table(cfg)
d = cfg.D // world
shard = torch.from_numpy(np.ascontiguousarray(W[:, rank * d:(rank + 1) * d])).cuda()
ex = EmbraceExchange(cfg.L, cfg.D, shard, world=world, rank=rank, device=rank, dtype=cfg.dtype,
                     max_tokens=cfg.max_tokens, mode="split", optim=cfg.optim, lr=cfg.lr, timeout_ms=500)
tdt = torch.float32
for k in range(5):
    ids = torch.from_numpy(wl.ids[k][rank]).cuda()
    Y = torch.empty(len(ids), cfg.D, device="cuda")
    E.emb_forward_exchange(ex.ctx, ids, Y, torch.cuda.current_stream())
    E.emb_backward_exchange(ex.ctx, torch.from_numpy(wl.dY[k][rank]).cuda(), torch.from_numpy(wl.ids[k + 1][rank]).cuda(),
                            torch.cuda.current_stream())
E.emb_join(ex.ctx, torch.cuda.current_stream())
torch.cuda.synchronize()
info = E.emb_debug_copy(ex.ctx, E.EMB_DBG_ERRINFO).reshape(8, 4)
print(rank, "err", ex.stats()["err_flags"], [tuple(int(v) for v in r[:3]) for r in info if r[3]], flush=True)
ts = E.emb_debug_copy(ex.ctx, E.EMB_DBG_TIMESTAMPS).view(np.uint64).astype(np.int64).reshape(16, 20, 8)
names = ["fwd","sort","mpush","coal","m0","defp","m1","rp","rc","tab","g_fwd","g_sort","g_pub0","g_pub1","g_sorted","g_marked","apply","mtag","g_seq","plan"]
base = ts[1, 0, 0]
for t in range(1, 6):
    row = ts[t]
    ev = sorted((row[k, 0], names[k], row[k, 2]) for k in range(20) if row[k, 0] > 0)
    print(rank, t, " ".join(f"{n}:{(a-base)/1e3:.0f}-{(b-base)/1e3:.0f}" for a, n, b in ev), flush=True)
dist.barrier()
