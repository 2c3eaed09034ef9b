#!/bin/bash
# final numbers on the final code: N = 1 (all configs, K = 20, reference arm) and N = 2 / 4 sweep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02_sf; mkdir -p $O
timeout 600 python bench.py > $O/n1_lstm_lm.json 2> $O/n1_lstm_lm.err
for cfg in gnmt transformer bert_large; do
  timeout 600 python bench.py --config $cfg > $O/n1_$cfg.json 2> $O/n1_$cfg.err
done
timeout 300 python bench.py --steps 20 --warmup 3 > $O/n1_k20.json 2> $O/n1_k20.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/n1_ref.json 2> $O/n1_ref.err
run() { local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?" >> $O/rc.txt; }
for n in 2 4; do
  for cfg in lstm_lm bert_large gnmt transformer; do run main_${cfg}_n$n $n bench.py --gpus $n --config $cfg --steps 1000 --warmup 20; done
  run main_lm_tables2_n$n $n bench.py --gpus $n --config lstm_lm --tables 2 --steps 1000 --warmup 20
  run main_lm_x4_n$n $n bench.py --gpus $n --config lstm_lm --batch-mult 4 --steps 500 --warmup 20
  run main_gnmt_x8_n$n $n bench.py --gpus $n --config gnmt --batch-mult 8 --steps 500 --warmup 20
  run main_lstm_lm_k20_n$n $n bench.py --gpus $n --config lstm_lm --steps 20 --warmup 3
done
cat $O/rc.txt
for f in $O/*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    sr=d.get("step_roofline") or {}
    print(sys.argv[1].split('/')[-1], d.get("impl","ours"), d["n_gpus"], d["steps"], round(d["ms_per_step"]*1e3,2), "us", round(d["value"]/1e6,3), "M/s frac", sr.get("frac"), (sr.get("plain_alltoall") or {}).get("frac"), "roof", (d.get("roofline") or {}).get("frac"), "e2e", round(d["e2e"]["value"]/1e6,2), "err", d.get("device_errors"))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
