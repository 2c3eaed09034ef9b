#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02rem2; mkdir -p $O
i=0
for rep in 1 2 3; do for gr in 1 0; do
  i=$((i+1))
  BENCH_GRAPH_REM=$gr timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/n2_gr${gr}_$rep.json 2> $O/n2_gr${gr}_$rep.err
done; done
for rep in 1 2; do for gr in 1 0; do
  BENCH_GRAPH_REM=$gr timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/n1_gr${gr}_$rep.json 2> $O/n1_gr${gr}_$rep.err
done; done
for f in $O/*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1], d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s", "graph med", d["step_time"]["graph"]["median_us"])
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
