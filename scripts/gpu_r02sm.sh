#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02sm; mkdir -p $O
bash scripts/gpu_variants.sh $O "lstm_lm gnmt transformer bert_large" "-DEMB_APPLY_SMALL=1" "-DEMB_APPLY_SMALL=2" "-DEMB_APPLY_SMALL=4" "-DEMB_APPLY_SMALL=8" "-DEMB_APPLY_SMALL=1" "-DEMB_APPLY_SMALL=4" | grep "step"
grep "== \|apply " $O/traces.txt
