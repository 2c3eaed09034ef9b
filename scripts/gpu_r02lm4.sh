#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02lm4; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 600 > $O/multi_tests.log 2>&1; echo "multi rc=$?" >> $O/rc.txt
tail -n 2 $O/multi_tests.log
run() { local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?" >> $O/rc.txt; }
run main_lstm_lm_n4 4 bench.py --gpus 4 --config lstm_lm --steps 1000 --warmup 20
run main_lm_tables2_n4 4 bench.py --gpus 4 --config lstm_lm --tables 2 --steps 1000 --warmup 20
run main_lm_x4_n4 4 bench.py --gpus 4 --config lstm_lm --batch-mult 4 --steps 500 --warmup 20
run main_lstm_lm_n4_k20 4 bench.py --gpus 4 --config lstm_lm --steps 20 --warmup 3
cat $O/rc.txt
for f in $O/main*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1].split('/')[-1], d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s frac", d["step_roofline"]["frac"], d["step_roofline"]["plain_alltoall"]["frac"], "err", d.get("device_errors"))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
