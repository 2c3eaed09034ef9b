#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=${1:-gpurun_out/r02_end3}; mkdir -p $O
bash scripts/gpu_roundend.sh $O
timeout 300 python bench.py --steps 20 --warmup 3 > $O/bench_k20.json 2> $O/bench_k20.err; echo "bench k20 rc=$?" >> $O/rc.txt
cat $O/rc.txt
