#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ag; mkdir -p $O
bash scripts/gpu_variants.sh $O "lstm_lm gnmt transformer bert_large" "-DEMB_APPLY_GRID_PER_SM=8" "-DEMB_APPLY_GRID_PER_SM=4" "-DEMB_APPLY_GRID_PER_SM=4 -DEMB_APPLY_EA_BF16=2" "-DEMB_APPLY_GRID_PER_SM=8" "-DEMB_APPLY_GRID_PER_SM=4" | grep "step" 
grep "== \|apply " $O/traces.txt
