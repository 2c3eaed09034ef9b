#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_colocated.py -q -m gpu --timeout 300 -x -k "tiny or pipelined or modes or lm_colocated or bert" > $O/coloc.log 2>&1; echo "coloc rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 3 $O/parity.log; tail -n 3 $O/coloc.log
bash scripts/gpu_exp.sh $O "lstm_lm bert_large gnmt transformer" "EMB_FUSED=0" "EMB_FUSED=1"
bash scripts/gpu_trace.sh $O/trace "lstm_lm bert_large"
