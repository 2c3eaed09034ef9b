#!/bin/bash
# N == 1 joined prefetch sorts without the flag fences (EMB_SORT_QUIET): parity + A/B with traces
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02quiet; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 2 $O/parity.log
bash scripts/gpu_variants.sh $O "lstm_lm bert_large gnmt" "-DEMB_SORT_QUIET=0" "-DEMB_SORT_QUIET=1" "-DEMB_SORT_QUIET=0" "-DEMB_SORT_QUIET=1" | grep step
grep "== \|sort " $O/traces.txt
cat $O/rc.txt
