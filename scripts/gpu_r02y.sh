#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x -k "not slow" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_colocated.py -q -m gpu --timeout 300 -x -k "tiny or modes or lm" > $O/coloc.log 2>&1; echo "coloc rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/parity.log $O/coloc.log | cat
bash scripts/gpu_exp.sh $O "lstm_lm gnmt transformer bert_large" ""
bash scripts/gpu_trace.sh $O/trace "lstm_lm"
