"""Debug: eager LM-shaped N=1 loop with per-step H2D/D2H copies (bench e2e pattern)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2110_09132_b200 import embrace as E
from paper_2110_09132_b200.runtime import EmbraceExchange
from synthetic import get_config, make_workload
from synthetic.workloads import gen_table
variant = sys.argv[1]
cfg = get_config("lstm_lm")
wl = make_workload(cfg, 1, 8)
W = torch.from_numpy(gen_table(cfg)).cuda()
ex = EmbraceExchange(cfg.L, cfg.D, W, max_tokens=cfg.max_tokens, mode="split", optim=cfg.optim, lr=cfg.lr,
                     dtype=cfg.dtype, timeout_ms=300)
stream = torch.cuda.Stream() if variant == "stream" else torch.cuda.current_stream()
h_ids = [torch.from_numpy(x[0].astype(np.int32)).pin_memory() for x in wl.ids]
h_dY = [torch.from_numpy(x[0]).pin_memory() for x in wl.dY]
ids_buf = [torch.empty(cfg.max_tokens, dtype=torch.int32, device="cuda") for _ in range(3)]
dY_buf = torch.empty((cfg.max_tokens, cfg.D), device="cuda")
Y_buf = torch.empty((cfg.max_tokens, cfg.D), device="cuda")
h_Y = torch.empty((cfg.max_tokens, cfg.D)).pin_memory()
with torch.cuda.stream(stream):
    for j in range(60):
        b, bn = j % 7, (j + 1) % 7
        n, nn = h_ids[b].numel(), h_ids[bn].numel()
        cur, nxt = ids_buf[j % 3][:n], ids_buf[(j + 1) % 3][:nn]
        if j == 0:
            cur.copy_(h_ids[b], non_blocking=True)
        nxt.copy_(h_ids[bn], non_blocking=True)
        dY_buf[:n].copy_(h_dY[b], non_blocking=True)
        if variant != "noprefetch":
            E.emb_prefetch(ex.ctx, nxt, stream)
        E.emb_forward_exchange(ex.ctx, cur, Y_buf[:n], stream)
        E.emb_backward_exchange(ex.ctx, dY_buf[:n], nxt, stream)
        if variant != "nod2h":
            h_Y[:n].copy_(Y_buf[:n], non_blocking=True)
    E.emb_join(ex.ctx, stream)
torch.cuda.synchronize()
info = E.emb_debug_copy(ex.ctx, E.EMB_DBG_ERRINFO).reshape(8, 4)
print(variant, "err", ex.stats()["err_flags"], [tuple(int(v) for v in r[:3]) for r in info if r[3]], flush=True)
