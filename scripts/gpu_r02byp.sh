#!/bin/bash
# single-row uniques bypass coal_reduce (EMB_SINGLE_BYPASS) A/B + parity
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02byp; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py -q -m gpu --timeout 400 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 3 $O/parity.log
bash scripts/gpu_exp.sh $O "lstm_lm gnmt transformer bert_large" "EMB_SINGLE_BYPASS=0" "EMB_SINGLE_BYPASS=1" "EMB_SINGLE_BYPASS=0" "EMB_SINGLE_BYPASS=1"
cat $O/rc.txt
