#!/bin/bash
# multi-GPU stress: long runs of every config (device error flags checked after the timed region)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02stress; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
for n in $NG 2; do for cfg in lstm_lm bert_large gnmt transformer; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $n --config $cfg --steps 40000 --warmup 20 --no-cpu-baseline > $O/s${n}_$cfg.json 2> $O/s${n}_$cfg.err
  echo "n$n $cfg rc=$?" >> $O/rc.txt
done; done
for n in $NG 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $n --config lstm_lm --mode coal --steps 20000 --warmup 20 --no-cpu-baseline > $O/s${n}_coal.json 2> $O/s${n}_coal.err
  echo "n$n coal rc=$?" >> $O/rc.txt
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $n --config gnmt --optim adagrad --tables 2 --steps 20000 --warmup 20 --no-cpu-baseline > $O/s${n}_adagrad2t.json 2> $O/s${n}_adagrad2t.err
  echo "n$n adagrad2t rc=$?" >> $O/rc.txt
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
