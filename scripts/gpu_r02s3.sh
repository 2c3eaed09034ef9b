#!/bin/bash
# N = 2: sort stream x forward dedup matrix
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s3; mkdir -p $O
bash scripts/gpu_multi_exp.sh $O 2 "lstm_lm gnmt bert_large" "EMB_SORT_STREAM=0 EMB_FWD_DEDUPN=1" "EMB_SORT_STREAM=0 EMB_FWD_DEDUPN=0" "EMB_SORT_STREAM=1 EMB_FWD_DEDUPN=1" "EMB_SORT_STREAM=1 EMB_FWD_DEDUPN=0" "EMB_SORT_STREAM=0 EMB_FWD_DEDUPN=1" "EMB_SORT_STREAM=0 EMB_FWD_DEDUPN=0"
EMB_TRACE=1 true
