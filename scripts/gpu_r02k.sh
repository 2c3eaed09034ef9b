#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02k; mkdir -p $O
for k in 16 20 32 36 200; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --config lstm_lm --steps $k --warmup 3 --no-cpu-baseline > $O/k$k.json 2> $O/k$k.err
done
for f in $O/k*.json; do python - $f <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
print(sys.argv[1].split('/')[-1], d["steps"], round(d["ms_per_step"]*1e3,2), "us; graph med", d["step_time"]["graph"]["median_us"])
PY
done
