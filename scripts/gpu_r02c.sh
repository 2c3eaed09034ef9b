#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02c
mkdir -p $O
for cfg in lstm_lm bert_large gnmt transformer; do
  for v in "" "--graph-no-prefetch"; do
    timeout 300 python bench.py --config $cfg --steps 1000 --warmup 20 --no-cpu-baseline $v > $O/b_${cfg}${v}.json 2> $O/b_${cfg}${v}.err
    python -c "import json,sys; d=json.loads(open('$O/b_${cfg}${v}.json').read().strip().splitlines()[-1]); print('$cfg $v', round(d['ms_per_step']*1e3,2), d['step_time']['graph'], d['roofline']['frac'])" >> $O/summary.txt 2>&1
  done
done
cat $O/summary.txt
