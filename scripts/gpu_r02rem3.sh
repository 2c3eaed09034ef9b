#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02rem3; mkdir -p $O
i=0
for rep in 1 2 3; do
  i=$((i+1))
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/n2_k20_$rep.json 2> $O/n2_k20_$rep.err
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 2 --steps 16 --warmup 3 --no-cpu-baseline > $O/n2_k16.json 2> $O/n2_k16.err
timeout 300 python bench.py --steps 20 --warmup 3 > $O/n1_k20.json 2> $O/n1_k20.err
for f in $O/*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1], d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s", "graph med", d["step_time"]["graph"]["median_us"], "e2e", round(d["e2e"]["value"]/1e6,2))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
