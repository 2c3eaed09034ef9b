#!/bin/bash
# EMB_PDL_EARLY A/B (compute kernels trigger their dependents right after griddepcontrol.wait)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02pdl; mkdir -p $O
EMB_PDL_EARLY=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py tests/test_gpu_multi.py -q -m gpu --timeout 400 -x > $O/parity_early.log 2>&1; echo "parity early rc=$?" >> $O/rc.txt
tail -n 3 $O/parity_early.log
bash scripts/gpu_exp.sh $O "lstm_lm gnmt transformer bert_large" "EMB_PDL_EARLY=0" "EMB_PDL_EARLY=1" "EMB_PDL_EARLY=0" "EMB_PDL_EARLY=1"
bash scripts/gpu_multi_exp.sh $O 2 "lstm_lm bert_large gnmt" "EMB_PDL_EARLY=0" "EMB_PDL_EARLY=1" "EMB_PDL_EARLY=0" "EMB_PDL_EARLY=1"
cat $O/rc.txt
