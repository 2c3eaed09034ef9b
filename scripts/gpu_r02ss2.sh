#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ss2; mkdir -p $O
bash scripts/gpu_multi_exp.sh $O 2 "lstm_lm gnmt transformer" "EMB_SORT_STREAM=0" "EMB_SORT_STREAM=1" "EMB_SORT_STREAM=0" "EMB_SORT_STREAM=1" > /dev/null
cat $O/summary.txt
