#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_colocated.py -q -m gpu --timeout 300 -x -k "two_tables or tiny or pipelined" > $O/coloc.log 2>&1; echo "coloc rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/parity.log $O/coloc.log | cat
bash scripts/gpu_exp.sh $O "lstm_lm gnmt bert_large" "EMB_FWD_DEDUP1=0" "EMB_FWD_DEDUP1=1"
for cfg in lstm_lm gnmt; do timeout 300 python bench.py --config $cfg --tables 2 --steps 1000 --warmup 20 --no-cpu-baseline > $O/t2_$cfg.json 2> $O/t2_$cfg.err; python -c "import json; d=json.loads(open('$O/t2_$cfg.json').read().strip().splitlines()[-1]); print('$cfg tables=2', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,1), 'Mtok/s')"; done
