#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02gs; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py -q -m gpu --timeout 400 -k "graph" > $O/graph.log 2>&1; echo "graph rc=$?" >> $O/rc.txt
tail -n 3 $O/graph.log
for k in 17 33 7; do timeout 300 python bench.py --steps $k --warmup 3 --no-cpu-baseline > $O/k$k.json 2> $O/k$k.err; echo "k$k rc=$?" >> $O/rc.txt; grep -i "capture failed" $O/k$k.err; done
for f in $O/k*.json; do python - $f <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
print(sys.argv[1], d["steps"], round(d["ms_per_step"]*1e3,2), "us", d["config"]["cuda_graph"], d.get("device_errors"))
PY
done
cat $O/rc.txt
for cfg in gnmt transformer; do
  CMD2="python bench.py --config $cfg --steps 30 --warmup 5 --no-graph --no-cpu-baseline --profile-steps 4"
  $CMD2 > $O/plain2_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|fwd_bulk|coal_reduce|coal_apply" -s 12 -c 6 -o $O/full_$cfg $CMD2 > $O/ncu_f_$cfg.log 2>&1
  echo "full $cfg rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
