#!/bin/bash
# Bench sweep on one box: every paper config at N = 1, 2, 4 (as many GPUs as visible),
# plus the default invocation (cpu_baseline leg) and the reference (oracle) arm.
# Usage (on a GPU box): bash scripts/sweep.sh <tag>
tag=${1:-sweep}
out=gpurun_out/$tag
mkdir -p $out
ngpu=$(nvidia-smi -L | wc -l)
timeout 300 python bench.py > $out/default_n1.json 2> $out/default_n1.err
python bench.py --impl reference --steps 3 --warmup 1 > $out/reference_n1.json 2> $out/reference_n1.err
for cfg in lstm_lm gnmt transformer bert_large; do
  CUDA_VISIBLE_DEVICES=0 EMB_TIMEOUT_MS=2000 timeout 240 python bench.py --config $cfg --no-cpu-baseline > $out/${cfg}_n1.json 2> $out/${cfg}_n1.err
  for n in 2 4 8; do
    [ $n -le $ngpu ] || continue
    EMB_TIMEOUT_MS=2000 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --config $cfg --no-cpu-baseline > $out/${cfg}_n$n.json 2> $out/${cfg}_n$n.err
  done
done
for f in $out/*.json; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
for line in open(f):
    if line.startswith("{"):
        d = json.loads(line)
        if "unavailable" in d:
            print(f, "unavailable"); continue
        rf = d.get("roofline", {})
        print(f"{f.split('/')[-1]:24s} {d['value']/1e6:9.2f} M{d['unit']}  {d['ms_per_step']*1e3:8.1f} us/step  "
              f"roof {rf.get('kernel','')}:{rf.get('frac')}  step_frac {d.get('step_roofline',{}).get('frac')}  "
              f"e2e {d.get('e2e',{}).get('value',0)/1e6:.2f}M  cpu {d.get('cpu_baseline',{}).get('value')}")
PY
done
