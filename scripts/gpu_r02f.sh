#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/parity.log
bash scripts/gpu_exp.sh $O "lstm_lm bert_large gnmt transformer" "EMB_SORT_JOIN=0" "EMB_SORT_JOIN=1" "EMB_FWD_GRID_PER_SM=2" "EMB_FWD_GRID_PER_SM=1"
