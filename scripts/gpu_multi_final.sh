#!/bin/bash
# round-2 final multi-GPU sweep: bash scripts/gpu_multi_final.sh OUTDIR "2 4"
cd "$GRAFT_REPO_ROOT"
O=$1; NS=$2
mkdir -p $O
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
     --master-port $((29500 + RANDOM % 2000)) "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?" >> $O/rc.txt
}
for n in $NS; do
  for cfg in lstm_lm bert_large gnmt transformer; do
    run main_${cfg}_n$n $n bench.py --gpus $n --config $cfg --steps 1000 --warmup 20
  done
  run main_lm_tables2_n$n $n bench.py --gpus $n --config lstm_lm --tables 2 --steps 1000 --warmup 20
  run main_lm_x4_n$n $n bench.py --gpus $n --config lstm_lm --batch-mult 4 --steps 500 --warmup 20
  run main_gnmt_x8_n$n $n bench.py --gpus $n --config gnmt --batch-mult 8 --steps 500 --warmup 20
  run main_bert_raw_n$n $n bench.py --gpus $n --config bert_large --mode raw --steps 1000 --warmup 20
  run sched_gnmt_n$n $n bench.py --gpus $n --config gnmt --schedule --steps 20 --warmup 5
  run dq_bert_n$n $n bench.py --gpus $n --config bert_large --dense-queue 24 --steps 20 --warmup 5
done
cat $O/rc.txt
