#!/bin/bash
# final-code ncu evidence (one GPU): launch lists (LM, BERT, N=1) + ncu --set full of the hot kernels
cd "$GRAFT_REPO_ROOT"
O=${1:-gpurun_out/r02_ncu}; mkdir -p $O
for cfg in lstm_lm bert_large; do
  CMD="python bench.py --config $cfg --steps 64 --warmup 8 --no-cpu-baseline"
  $CMD > $O/plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 400 --csv --log-file $O/launches_$cfg.csv $CMD > $O/ncu_l_$cfg.log 2>&1
  echo "launches $cfg rc=$?" >> $O/rc.txt
  CMD2="python bench.py --config $cfg --steps 30 --warmup 5 --no-graph --no-cpu-baseline --profile-steps 4"
  $CMD2 > $O/plain2_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|fwd_bulk|coal_reduce|coal_apply" -s 12 -c 6 -o $O/full_$cfg $CMD2 > $O/ncu_f_$cfg.log 2>&1
  echo "full $cfg rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
