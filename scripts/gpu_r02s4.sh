#!/bin/bash
# N = 4 / 2: sort of t+1 on its own stream (EMB_SORT_STREAM) A/B, two reps
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s4; mkdir -p $O
bash scripts/gpu_multi_exp.sh $O 4 "lstm_lm bert_large gnmt transformer" "EMB_SORT_STREAM=0" "EMB_SORT_STREAM=1" "EMB_SORT_STREAM=0" "EMB_SORT_STREAM=1" | grep "N="
EMB_SORT_STREAM=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 600 -x -k "tiny or prefetch" > $O/multi.log 2>&1; echo "multi rc=$?"; tail -n 2 $O/multi.log
