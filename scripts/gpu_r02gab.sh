#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02gab; mkdir -p $O
bash scripts/gpu_multi_exp.sh $O 4 "bert_large lstm_lm gnmt" "BENCH_GRAPH_MIN_STEPS=1" "BENCH_GRAPH_MIN_STEPS=64" "BENCH_GRAPH_MIN_STEPS=1" "BENCH_GRAPH_MIN_STEPS=64" > /dev/null
bash scripts/gpu_multi_exp.sh $O 2 "bert_large lstm_lm" "BENCH_GRAPH_MIN_STEPS=1" "BENCH_GRAPH_MIN_STEPS=64" > /dev/null
bash scripts/gpu_exp.sh $O "bert_large lstm_lm" "BENCH_GRAPH_MIN_STEPS=1" "BENCH_GRAPH_MIN_STEPS=64" > /dev/null
cat $O/summary.txt
