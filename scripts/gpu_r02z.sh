#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z; mkdir -p $O
bash scripts/gpu_exp.sh $O "lstm_lm bert_large gnmt" "EMB_REDUCE_GRID_PER_SM=12" "EMB_REDUCE_GRID_PER_SM=2" "EMB_REDUCE_GRID_PER_SM=4" "EMB_FWD_GRID_PER_SM=2"
EMB_REDUCE_GRID_PER_SM=3 bash scripts/gpu_variants.sh $O/rb2 "lstm_lm bert_large gnmt" "-DEMB_RB=2"
