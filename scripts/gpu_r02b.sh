#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02b
mkdir -p $O
timeout 600 python -m pytest tests -q -m gpu --timeout 300 -k "graph" > $O/graph.log 2>&1; echo "graph rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 400 --warmup 20 > $O/bench_lm.json 2> $O/bench_lm.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --config bert_large --steps 400 --warmup 20 --no-cpu-baseline > $O/bench_bert.json 2> $O/bench_bert.err; echo "bench bert rc=$?" >> $O/rc.txt
cat $O/rc.txt
