#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bulk; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/parity.log
bash scripts/gpu_exp.sh $O "lstm_lm gnmt transformer bert_large" "EMB_FWD_BULK=0" "EMB_FWD_BULK=1"
bash scripts/gpu_trace.sh $O/trace "lstm_lm bert_large"
