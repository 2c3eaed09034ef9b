#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02fb2; mkdir -p $O
bash scripts/gpu_variants.sh $O "lstm_lm" "-DEMB_FWD_BULK_ROWS=16 -DEMB_FWD_BULK_PER_SM=3" "-DEMB_FWD_BULK_ROWS=4 -DEMB_FWD_BULK_PER_SM=8" "-DEMB_FWD_BULK_ROWS=16 -DEMB_FWD_BULK_PER_SM=3" "-DEMB_FWD_BULK_ROWS=4 -DEMB_FWD_BULK_PER_SM=8" | grep step
grep "== \|fwd \|coal \|apply " $O/traces.txt
