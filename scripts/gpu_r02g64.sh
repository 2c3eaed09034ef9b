#!/bin/bash
# bench graphs of >= 64 steps (one pipeline drain per graph): N = 1 / 2 / 4, K = 2000 and 20
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02g64; mkdir -p $O
for cfg in lstm_lm bert_large gnmt; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline > $O/n1_$cfg.json 2> $O/n1_$cfg.err
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/n1_k20.json 2> $O/n1_k20.err
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $n --no-cpu-baseline > $O/n${n}_lstm_lm.json 2> $O/n${n}_lstm_lm.err
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline > $O/n${n}_k20.json 2> $O/n${n}_k20.err
done
for f in $O/*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1].split('/')[-1], d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s; graph_steps", d["config"].get("graph_steps"), "graph med", d["step_time"]["graph"]["median_us"], "roof", d["roofline"]["frac"], "err", d.get("device_errors"))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
