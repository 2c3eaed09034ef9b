#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02sp3; mkdir -p $O
bash scripts/gpu_multi_exp.sh $O 4 "bert_large gnmt lstm_lm" "EMB_SIDE_PRIO=0" "EMB_SIDE_PRIO=1" "EMB_SIDE_PRIO=0 BENCH_GRAPH_MIN_STEPS=1" "EMB_SIDE_PRIO=1 BENCH_GRAPH_MIN_STEPS=1" > /dev/null
bash scripts/gpu_multi_exp.sh $O 2 "bert_large lstm_lm" "EMB_SIDE_PRIO=0" "EMB_SIDE_PRIO=1" > /dev/null
cat $O/summary.txt
