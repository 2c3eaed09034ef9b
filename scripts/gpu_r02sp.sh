#!/bin/bash
# sort: keys spread over all warps (EMB_SORT_SPREAD) — parity + A/B with traces
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02sp; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py -q -m gpu --timeout 400 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 2 $O/parity.log
bash scripts/gpu_variants.sh $O "lstm_lm gnmt bert_large" "-DEMB_SORT_SPREAD=0" "-DEMB_SORT_SPREAD=1" "-DEMB_SORT_SPREAD=0" "-DEMB_SORT_SPREAD=1" | grep -v "^  [a-z]" | head -40
grep -A3 "== \|sort " $O/traces.txt | grep "==\|sort " 
cat $O/rc.txt
