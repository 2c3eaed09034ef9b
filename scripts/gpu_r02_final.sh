#!/bin/bash
# round-2 final evidence on one GPU: round-end validation, per-config benches, ncu of the final code
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02_end2; mkdir -p $O
bash scripts/gpu_roundend.sh $O
for cfg in gnmt transformer bert_large; do
  timeout 600 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err; echo "bench $cfg rc=$?" >> $O/rc.txt
done
timeout 300 python bench.py --steps 20 --warmup 3 > $O/bench_k20.json 2> $O/bench_k20.err; echo "bench k20 rc=$?" >> $O/rc.txt
bash scripts/gpu_ncu_final.sh gpurun_out/r02_ncu2
cat $O/rc.txt
