#!/bin/bash
# N = 4 stress with the sort stream default (every vocabulary at N >= 4): 40k steps, device errors checked
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02stress2; mkdir -p $O
for cfg in bert_large gnmt transformer lstm_lm; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus 4 --config $cfg --steps 40000 --warmup 20 --no-cpu-baseline > $O/s4_$cfg.json 2> $O/s4_$cfg.err
  echo "$cfg rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
for f in $O/s*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1].split('/')[-1], d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s errors", d.get("device_errors"))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
