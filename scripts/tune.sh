#!/bin/bash
# Compile-time variant sweep (N = 1): each variant rebuilds libembrace.so with
# EMB_NVCC_EXTRA and runs the LM and BERT benches.  Usage: bash scripts/tune.sh "<flags1>" "<flags2>" ...
for v in "$@"; do
  export EMB_NVCC_EXTRA="$v"
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for cfg in lstm_lm bert_large; do
    r=$(EMB_TIMEOUT_MS=2000 timeout 120 python bench.py --config $cfg --steps 1000 --warmup 10 --no-cpu-baseline 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')
    echo "[$v] $cfg $r"
  done
done
