#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02e; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x -k "not slow" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
timeout 600 python -m pytest tests/test_gpu_colocated.py -q -m gpu --timeout 300 -x -k "tiny or pipelined" > $O/coloc.log 2>&1; echo "coloc rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -2 $O/parity.log $O/coloc.log
bash scripts/gpu_exp.sh $O "lstm_lm bert_large gnmt" "EMB_FOLD_SORTED=0" "EMB_FOLD_SORTED=1" "EMB_FWD_GRID_PER_SM=1" "EMB_FWD_GRID_PER_SM=2" "EMB_FWD_GRID_PER_SM=8"
