#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02pt; mkdir -p $O
echo "== phase stamps"; bash scripts/gpu_trace.sh $O/phase "lstm_lm bert_large" | grep "sort"
EMB_NVCC_EXTRA="-DEMB_TRACE -DEMB_SORT_PASS_TRACE" python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build.log 2>&1
for cfg in lstm_lm bert_large; do
  EMB_TRACE_OUT=$O/tr_$cfg timeout 300 python bench.py --config $cfg --steps 400 --warmup 20 --no-cpu-baseline > /dev/null 2>&1
  echo "== first-pass stamps $cfg (s4 ranked, s5 cluster.sync 1, s6 offsets, s7 scatter+sync)"; python scripts/trace.py $O/tr_$cfg.*.npy | grep sort
done
python -c "from paper_2110_09132_b200.build import build; build(force=True)" >> $O/build.log 2>&1
