#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02rem; mkdir -p $O
for k in 20 7 33; do
  timeout 300 python bench.py --steps $k --warmup 3 > $O/n1_k$k.json 2> $O/n1_k$k.err; echo "n1 k$k rc=$?" >> $O/rc.txt
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 20 --warmup 3 > $O/n2_k20.json 2> $O/n2_k20.err; echo "n2 k20 rc=$?" >> $O/rc.txt
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 37 --warmup 3 > $O/n2_k37.json 2> $O/n2_k37.err; echo "n2 k37 rc=$?" >> $O/rc.txt
cat $O/rc.txt
for f in $O/*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1], d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s", d.get("device_errors"))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
