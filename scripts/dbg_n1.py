import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2110_09132_b200 import embrace as E
from paper_2110_09132_b200.runtime import EmbraceExchange
from synthetic import get_config, make_workload
from synthetic.workloads import gen_table
cfg = get_config("tiny")
wl = make_workload(cfg, 1, 4)
W = torch.from_numpy(gen_table(cfg)).cuda()
ex = EmbraceExchange(cfg.L, cfg.D, W, max_tokens=cfg.max_tokens, mode="split", optim=cfg.optim, lr=cfg.lr, dtype=cfg.dtype, timeout_ms=1000)
for k in range(3):
    ids = torch.from_numpy(wl.ids[k][0]).cuda()
    ex.forward(ids)
    ex.backward(torch.from_numpy(wl.dY[k][0]).cuda(), torch.from_numpy(wl.ids[k + 1][0]).cuda())
    torch.cuda.synchronize()
    print("iter", k, "err", ex.stats()["err_flags"], flush=True)
print("errinfo", E.emb_debug_copy(ex.ctx, E.EMB_DBG_ERRINFO))
ts = E.emb_debug_copy(ex.ctx, E.EMB_DBG_TIMESTAMPS).view(np.uint64).astype(np.int64).reshape(16, 20, 8)
names = ["fwd","sort","mark","coal","m0","defp","m1","rp","rc","tab","g_fwd","g_sort","g_pub0","g_pub1","g_sorted","g_marked","apply","g_defdone","g_seq","k19"]
base = ts[1, 0, 0]
for t in range(1, 4):
    row = ts[t]
    print(t, {names[k]: (round((row[k,0]-base)/1e3, 1), round((row[k,2]-base)/1e3, 1)) for k in range(20) if row[k,0] > 0})
