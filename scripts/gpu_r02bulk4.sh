#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bulk4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 2 $O/parity.log
for w in lstm_lm gnmt transformer bert_large; do
  timeout 300 python bench.py --config $w --steps 2000 --warmup 20 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02bulk4/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["ms_per_step"]*1e3, d["value"], d["roofline"]["frac"])
    except Exception as e: print(f, e)
PY
