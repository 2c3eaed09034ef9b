#!/bin/bash
# kernel-trace run: EMB_TRACE build, bench with the trace ring dumped, summary (scripts/trace.py)
# usage: bash scripts/gpu_trace.sh OUTDIR "config list" [extra bench args]
cd "$GRAFT_REPO_ROOT"
O=$1; CFGS=$2; shift 2
mkdir -p $O
EMB_NVCC_EXTRA=-DEMB_TRACE python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build.log 2>&1
for cfg in $CFGS; do
  EMB_TRACE_OUT=$O/tr_$cfg timeout 300 python bench.py --config $cfg --steps 400 --warmup 20 --no-cpu-baseline "$@" > $O/b_$cfg.json 2> $O/b_$cfg.err
  python scripts/trace.py $O/tr_$cfg.*.npy > $O/trace_$cfg.txt 2>&1
  cat $O/trace_$cfg.txt
done
python -c "from paper_2110_09132_b200.build import build; build(force=True)" >> $O/build.log 2>&1
