#!/bin/bash
# sort: 10-bit digits when they save a radix pass (LM: 3 -> 2 passes) — parity + A/B with traces
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02db; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py -q -m gpu --timeout 600 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 2 $O/parity.log
bash scripts/gpu_variants.sh $O "lstm_lm" "-DEMB_SORT_DB10=0" "-DEMB_SORT_DB10=1" "-DEMB_SORT_DB10=0" "-DEMB_SORT_DB10=1" | grep step
grep "== \|sort \|apply " $O/traces.txt
cat $O/rc.txt
