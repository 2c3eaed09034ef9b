#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02cap; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py -q -m gpu --timeout 600 -x -k "16k or bf16_configs or tiny_sgd or lm_fp32" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/parity.log
# bandwidth-regime sweep: tokens per rank x1 x2 x4 x8 (where the cap allows), N = 1
for cfg in lstm_lm gnmt bert_large; do for m in 1 2 4 8; do
  timeout 300 python bench.py --config $cfg --batch-mult $m --steps 500 --no-cpu-baseline > $O/b_${cfg}_x$m.json 2> $O/b_${cfg}_x$m.err
  python -c "import json; d=json.loads(open('$O/b_${cfg}_x$m.json').read().strip().splitlines()[-1]); print('$cfg x$m', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,1), 'Mtok/s step_frac', d['step_roofline']['frac'], 'roof', d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null || echo "$cfg x$m failed: $(tail -n 1 $O/b_${cfg}_x$m.err)"
done; done
