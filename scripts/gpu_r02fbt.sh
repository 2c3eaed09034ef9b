#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02fbt; mkdir -p $O
bash scripts/gpu_variants.sh $O "lstm_lm" "-DEMB_FWD_BULK_THREADS=128" "-DEMB_FWD_BULK_THREADS=32" "-DEMB_FWD_BULK_THREADS=128" "-DEMB_FWD_BULK_THREADS=32" | grep step
grep "== \|fwd " $O/traces.txt
