#!/bin/bash
# coal_reduce grid cap after the single-row bypass
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02rg; mkdir -p $O
bash scripts/gpu_exp.sh $O "lstm_lm gnmt transformer bert_large" "EMB_REDUCE_GRID_PER_SM=12" "EMB_REDUCE_GRID_PER_SM=1" "EMB_REDUCE_GRID_PER_SM=2" "EMB_REDUCE_GRID_PER_SM=4" "EMB_REDUCE_GRID_PER_SM=12" "EMB_REDUCE_GRID_PER_SM=2"
