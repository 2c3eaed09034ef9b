#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02_ncu3; mkdir -p $O
cfg=lstm_lm
CMD="python bench.py --config $cfg --steps 64 --warmup 8 --no-cpu-baseline"
$CMD > $O/plain_$cfg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 400 --csv --log-file $O/launches_$cfg.csv $CMD > $O/ncu_l_$cfg.log 2>&1
echo "launches rc=$?"
CMD2="python bench.py --config $cfg --steps 30 --warmup 5 --no-graph --no-cpu-baseline --profile-steps 4"
$CMD2 > $O/plain2_$cfg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|fwd_bulk|coal_reduce|coal_apply" -s 12 -c 6 -o $O/full_$cfg $CMD2 > $O/ncu_f_$cfg.log 2>&1
echo "full rc=$?"
