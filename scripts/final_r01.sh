#!/bin/bash
# End-of-round evidence on one 4-GPU box: the bench sweep (scripts/sweep.sh),
# the a13 dense-queue measurement at N = 1, 2, 4, the ncu launch lists of the
# default bench (LM N = 1) and BERT N = 1, and one `ncu --set full` capture of
# the dominant kernel (coal_apply) of each.
# Usage (on a GPU box): bash scripts/final_r01.sh <tag> [sweep|ncu|all]
tag=${1:-final}
what=${2:-all}
out=gpurun_out/$tag
mkdir -p $out
if [ $what != ncu ]; then
bash scripts/sweep.sh $tag > $out/sweep_table.txt 2>&1
ngpu=$(nvidia-smi -L | wc -l)
for c in "gnmt 1" "gnmt 16" "bert_large 1" "bert_large 24"; do
  set -- $c
  CUDA_VISIBLE_DEVICES=0 timeout 240 python bench.py --config $1 --dense-queue $2 --steps 20 --warmup 12 \
    > $out/dq_$1_n1_w$2.json 2> $out/dq_$1_n1_w$2.err
  for n in 2 4; do
    [ $n -le $ngpu ] || continue
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n --config $1 --dense-queue $2 --steps 20 --warmup 12 \
      > $out/dq_$1_n${n}_w$2.json 2> $out/dq_$1_n${n}_w$2.err
  done
done
fi
[ $what != sweep ] || exit 0
export CUDA_VISIBLE_DEVICES=0
for cfg in lstm_lm bert_large; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_${cfg}_n1.csv python bench.py --config $cfg --steps 48 --warmup 3 --no-graph \
    --no-cpu-baseline --profile-steps 1 > $out/ncu_launch_${cfg}.log 2>&1
  python scripts/prof_summary.py launches $out/launches_${cfg}_n1.csv > $out/launches_${cfg}_n1.txt 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:coal_apply -s 20 -c 1 \
    -o $out/full_${cfg}_n1 python bench.py --config $cfg --steps 24 --warmup 3 --no-graph --no-cpu-baseline \
    --profile-steps 1 > $out/ncu_full_${cfg}.log 2>&1
  python scripts/prof_summary.py full $out/full_${cfg}_n1.ncu-rep > $out/full_${cfg}_n1.md 2>&1
done
