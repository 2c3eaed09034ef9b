#!/bin/bash
# round-2 multi-GPU sweep: bash scripts/gpu_multi_sweep.sh OUTDIR "2 4"
cd "$GRAFT_REPO_ROOT"
O=$1; NS=$2
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
     --master-port $((29500 + RANDOM % 2000)) "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?" >> $O/rc.txt
}
for n in $NS; do
  run nvlink_n$n $n scripts/nvlink_bench.py
  for cfg in lstm_lm bert_large gnmt transformer; do
    run main_${cfg}_n$n $n bench.py --gpus $n --config $cfg --steps 1000 --warmup 20
  done
  for cfg in gnmt bert_large; do run sched_${cfg}_n$n $n bench.py --gpus $n --config $cfg --schedule --steps 20 --warmup 5; done
  for b in allgather allreduce; do
    for cfg in lstm_lm bert_large gnmt; do run base_${b}_${cfg}_n$n $n bench.py --gpus $n --config $cfg --baseline $b --steps 100 --warmup 5; done
  done
  run main_lm_tables2_n$n $n bench.py --gpus $n --config lstm_lm --tables 2 --steps 1000 --warmup 20
done
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 600 > $O/multi_tests.log 2>&1; echo "multi tests rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 3 $O/multi_tests.log
