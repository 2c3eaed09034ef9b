#!/bin/bash
# N == 1 split apply (EMB_FUSE_SINGLE): single-row updates beside coal_reduce; A/B + parity
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02fs; mkdir -p $O
EMB_FUSE_SINGLE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 400 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 3 $O/parity.log
bash scripts/gpu_exp.sh $O "lstm_lm gnmt transformer bert_large" "EMB_FUSE_SINGLE=0" "EMB_FUSE_SINGLE=1" "EMB_FUSE_SINGLE=0" "EMB_FUSE_SINGLE=1"
cat $O/rc.txt
