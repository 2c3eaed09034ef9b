#!/bin/bash
# epoch-tagged id all-gather: multi-GPU tests + N = 2 / 4 benches (compare: profiles/r02_multi_final/stress)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02tag4; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 600 -x > $O/multi.log 2>&1; echo "multi rc=$?" >> $O/rc.txt
tail -n 2 $O/multi.log
for n in 4 2; do
  for cfg in lstm_lm bert_large gnmt transformer; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $n --config $cfg --steps 4000 --warmup 20 --no-cpu-baseline > $O/b${n}_$cfg.json 2> $O/b${n}_$cfg.err
  done
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $n --config lstm_lm --mode coal --steps 4000 --warmup 20 --no-cpu-baseline > $O/b${n}_coal.json 2> $O/b${n}_coal.err
done
for f in $O/b*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1].split('/')[-1], d["n_gpus"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,1), "M/s", d["config"]["mode"], "err", d.get("device_errors"), "step_frac", d["step_roofline"]["frac"])
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
cat $O/rc.txt
