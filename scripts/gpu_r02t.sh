#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_colocated.py -q -m gpu --timeout 300 -x > $O/coloc.log 2>&1; echo "coloc rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 300 -x -k "tiny or prefetch or dense" > $O/multi.log 2>&1; echo "multi rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/multi.log $O/coloc.log 2>/dev/null | cat
bash scripts/gpu_multi_exp.sh $O 2 "lstm_lm bert_large gnmt transformer" ""
bash scripts/gpu_trace_multi.sh $O 2 "lstm_lm"
