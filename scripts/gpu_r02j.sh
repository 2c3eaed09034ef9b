#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x -k "not slow" > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 2 $O/parity.log
bash scripts/gpu_variants.sh $O "lstm_lm bert_large gnmt" "" "-DEMB_FUSED_MINB=3 -DEMB_FUSED_EB_F32=1"
