#!/bin/bash
# N > 1: prefetched sort on its own stream (EMB_SORT_STREAM) A/B + multi-GPU parity
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 400 -x > $O/multi.log 2>&1; echo "multi rc=$?" >> $O/rc.txt
tail -n 3 $O/multi.log
bash scripts/gpu_multi_exp.sh $O 2 "lstm_lm bert_large gnmt transformer" "EMB_SORT_STREAM=0" "EMB_SORT_STREAM=1" "EMB_SORT_STREAM=0" "EMB_SORT_STREAM=1"
for f in $O/b2_*.json; do python - $f <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
print(sys.argv[1], d["nvlink_measured"]["library_counters_per_step"])
PY
done
cat $O/rc.txt
